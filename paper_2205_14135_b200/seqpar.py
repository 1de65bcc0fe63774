"""Sequence-parallel attention over key shards (the paper's multi-GPU
extension).

One long sequence, R ranks (one process per GPU). Rank r holds every query and the key /
value shard [k0_r, k1_r) (tile-aligned, ``shard_range``). Forward: each rank runs the sm_100a
forward on its shard with ``k_offset = k0_r`` (global key indices for causal / padding /
custom masks and the dropout hash) and fp32 partial outputs. The exchange is an all-gather of
the partial LSE_r only (R x B x H x Nq floats) and an all-reduce (sum) of fp32 O-sized shares:
with LSE_rest = logsumexp of the other ranks' LSE, ``tatn_merge_partials`` over the pair
(O_r, LSE_r), (0, LSE_rest) — the reference's merge_stats algebra (softmax.hpp:48-59,
softmax.cpp:62-83) — gives rank r's share O_r exp(LSE_r - LSE) and the global LSE, and the shares
sum to O. Memory and traffic stay at one O per rank (an all-gather of the partial O would move R
of them). Backward: each rank
runs the backward on its shard against the merged (O, LSE) — D = rowsum(dO * O) and P are
then global — which yields the shard's dK, dV exactly and a partial dQ over the shard's keys;
the exchange is an all-reduce (sum) of the fp32 partial dQ.

The collectives are torch.distributed (NCCL on GPUs); the kernels are the C ABI's. The
compute steps are methods so the orchestration can be exercised on CPU with gloo and a
stand-in compute (tests/test_seqpar.py).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import torch
import torch.distributed as dist

TILE = 128


def shard_range(n_keys: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, 128-aligned key shard [k0, k1) of rank `rank` (the last shard takes the tail)."""
    tiles = -(-n_keys // TILE)
    per = -(-tiles // world)
    k0 = min(rank * per * TILE, n_keys)
    k1 = min((rank + 1) * per * TILE, n_keys)
    return k0, k1


class KeyShardedAttention:
    """Forward / backward of attention whose keys are sharded across the ranks of `group`."""

    def __init__(self, group: Optional[dist.ProcessGroup] = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    # ------------------------------------------------------------------ compute steps
    def _partial_fwd(self, q, k, v, spec, out=None):
        from . import attention as A

        spec = dataclasses.replace(spec, out_fp32=True)
        o = torch.empty(q.shape, dtype=torch.float32, device=q.device) if out is None else out
        return A.flash_fwd(q, k, v, spec, out=o)

    def _merge(self, o_parts, lse_parts, out_dtype):
        from . import attention as A

        B, H, Nq, d = o_parts.shape[1:]
        out = torch.empty((B, H, Nq, d), dtype=out_dtype, device=o_parts.device)
        return A.merge_partials(o_parts, lse_parts, out=out)

    def _partial_bwd(self, q, k, v, o32, do, lse, spec):
        from . import attention as A

        spec = dataclasses.replace(spec, out_fp32=True)
        f32 = lambda t: torch.empty(t.shape, dtype=torch.float32, device=t.device)
        return A.flash_bwd(q, k, v, o32, do, lse, spec, f32(q), f32(k), f32(v))

    # ------------------------------------------------------------------ public
    def local_keys(self, n_keys: int) -> Tuple[int, int]:
        return shard_range(n_keys, self.world, self.rank)

    def forward(self, q, k_local, v_local, spec, n_keys: int):
        """q [B,H,Nq,d] (all queries), k/v_local [B,H,k1-k0,d] = this rank's shard of n_keys keys.
        Returns (o in q's dtype, lse fp32, o fp32 for the backward)."""
        k0, k1 = self.local_keys(n_keys)
        if k_local.shape[2] != k1 - k0:
            raise ValueError(f"rank {self.rank}: key shard has {k_local.shape[2]} rows, expected {k1 - k0}")
        local = dataclasses.replace(spec, k_offset=k0)
        # [2, B, H, Nq, d] fp32: slot 0 = this shard's partial O_r, slot 1 = zeros (the "rest" partial)
        pair = torch.zeros((2,) + tuple(q.shape), dtype=torch.float32, device=q.device)
        if k1 > k0:
            _, lse_p = self._partial_fwd(q, k_local, v_local, local, out=pair[0])
        else:  # an empty shard contributes nothing (LSE = -inf)
            lse_p = torch.full(q.shape[:3], float("-inf"), dtype=torch.float32, device=q.device)
        lse_all = self._all_gather(lse_p)  # the only gather: R x B x H x Nq floats
        others = torch.cat([lse_all[:self.rank], lse_all[self.rank + 1:]])
        lse_rest = (torch.logsumexp(others, dim=0) if others.shape[0] else
                    torch.full_like(lse_p, float("-inf")))
        # this rank's share O_r exp(LSE_r - LSE) and the global LSE, then the sum over ranks
        o32, lse = self._merge(pair, torch.stack([lse_p, lse_rest]).contiguous(), torch.float32)
        if self.world > 1:
            dist.all_reduce(o32, op=dist.ReduceOp.SUM, group=self.group)
        return o32.to(q.dtype), lse, o32

    def backward(self, q, k_local, v_local, o32, do, lse, spec, n_keys: int):
        """Gradients for all queries (dq, summed over ranks) and this rank's key shard (dk, dv)."""
        k0, k1 = self.local_keys(n_keys)
        local = dataclasses.replace(spec, k_offset=k0)
        if k1 > k0:
            dq_p, dk, dv = self._partial_bwd(q, k_local, v_local, o32, do, lse, local)
        else:
            dq_p = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
            dk = torch.zeros(k_local.shape, dtype=torch.float32, device=q.device)
            dv = torch.zeros(v_local.shape, dtype=torch.float32, device=q.device)
        if self.world > 1:
            dist.all_reduce(dq_p, op=dist.ReduceOp.SUM, group=self.group)
        return dq_p.to(q.dtype), dk.to(k_local.dtype), dv.to(v_local.dtype)

    def _all_gather(self, t: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if self.world == 1:
            out[0].copy_(t)
        elif dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        else:  # gloo (CPU tests) has no all_gather_into_tensor
            dist.all_gather(list(out.unbind(0)), t.contiguous(), group=self.group)
        return out
