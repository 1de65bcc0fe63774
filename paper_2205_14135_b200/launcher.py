"""(batch, head)-sharded multi-GPU launcher (north star part 4).

The reference's only concurrency model is independent (b, h) problems, each
with its own MemoryModel, combined afterwards with
AccessCounter::merge (counters.cpp:8-13). Here one process per GPU (torchrun,
``torch.distributed``) owns a contiguous range of the flattened b*H + h slices
and runs the sm_100a kernels on them; there is no collective on the hot path.
``torch.distributed`` is used only for the bench's barrier / max-over-ranks
timing and for an optional off-path gather of results for verification.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional, Sequence, Tuple


def shard_range(n_slices: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [start, end) of n_slices for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad world/rank {world}/{rank}")
    base, extra = divmod(n_slices, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def slice_batch_index(start: int, end: int, H: int) -> list:
    """Batch index b of every flattened slice s = b*H + h in [start, end)."""
    return [s // H for s in range(start, end)]


@dataclass
class DistEnv:
    world: int = 1
    rank: int = 0
    local_rank: int = 0

    @staticmethod
    def from_env() -> "DistEnv":
        return DistEnv(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                       int(os.environ.get("LOCAL_RANK", "0")))


def init_distributed(backend: str = "nccl") -> DistEnv:
    """Initialise torch.distributed when launched by torchrun (no-op for 1 rank).

    TATN_DIST_BACKEND=gloo and TATN_SHARED_GPU=1 are test hooks: they let several
    ranks share one device (gloo for the bench's timing collectives) so the
    multi-rank path can be exercised on a single-GPU machine."""
    env = DistEnv.from_env()
    backend = os.environ.get("TATN_DIST_BACKEND", backend)
    if os.environ.get("TATN_SHARED_GPU") == "1":
        env.local_rank = 0
    if env.world > 1:
        import torch.distributed as dist

        if not dist.is_initialized():
            import torch

            if backend == "nccl":
                torch.cuda.set_device(env.local_rank)
                dist.init_process_group("nccl", device_id=torch.device("cuda", env.local_rank))
            else:
                dist.init_process_group(backend)
    return env


class BHShardedAttention:
    """Runs attention over this rank's share of the (b, h) slices.

    ``q, k, v`` are this rank's views of the global ``[B, H, N, d]`` tensors
    flattened to slices: rank r owns slices ``shard_range(B*H, world, r)`` and
    passes them as ``[S, 1, N, d]`` (B' = S slices, H' = 1). Per-batch
    ``valid_len`` is expanded per slice so key padding stays exact.
    ``compute`` is the per-device attention call (the C-ABI kernels in
    production: :func:`paper_2205_14135_b200.attention.flash_fwd`/``flash_bwd``).
    """

    def __init__(self, B: int, H: int, env: Optional[DistEnv] = None):
        self.B, self.H = B, H
        self.env = env or DistEnv.from_env()
        self.start, self.end = shard_range(B * H, self.env.world, self.env.rank)

    @property
    def n_local(self) -> int:
        return self.end - self.start

    def local_slices(self, t):
        """This rank's [S, 1, N, d] view of a contiguous global [B, H, N, d] tensor."""
        B, H, N, d = t.shape
        flat = t.reshape(B * H, N, d)
        return flat[self.start:self.end].unsqueeze(1)

    def local_valid_len(self, valid_len: Sequence[int]):
        return [int(valid_len[b]) for b in slice_batch_index(self.start, self.end, self.H)]

    def run(self, compute: Callable, *tensors, **kw):
        return compute(*[self.local_slices(t) for t in tensors], **kw)


def gather_slices(local, env: DistEnv, B: int, H: int):
    """Off-path verification gather: reassemble [B, H, ...] from every rank's
    [S, 1, ...] results (all_gather over the process group; not timed)."""
    import torch
    import torch.distributed as dist

    if env.world == 1:
        return local.reshape(B, H, *local.shape[2:])
    sizes = [shard_range(B * H, env.world, r) for r in range(env.world)]
    maxn = max(e - s for s, e in sizes)
    pad = torch.zeros((maxn,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(env.world)]
    dist.all_gather(bufs, pad)
    parts = [bufs[r][: e - s] for r, (s, e) in enumerate(sizes)]
    return torch.cat(parts, 0).reshape(B, H, *local.shape[2:])
