"""Sequence-parallel attention over key shards.

CPU: the shard partition; the merge algebra (numpy restatement of tatn_merge_partials /
merge_stats, softmax.cpp:62-83) recombines per-shard oracle results into full attention;
a 2- and 3-rank gloo run of KeyShardedAttention's orchestration (all-gather of the partial
LSEs, pairwise merge into this rank's share of O, all-reduce of the shares and of dQ) with the
oracle standing in for the kernels reproduces single-process attention. GPU: the kernels with k_offset on R virtual shards + tatn_merge_partials against
the oracle (north-star tolerance) for causal / none / key padding / custom / dropout, and the
merge kernel against its restatement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2205_14135_b200.seqpar import KeyShardedAttention, shard_range


@pytest.mark.parametrize("n", [1, 128, 300, 1024, 1025])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_tile_aligned_partition(n, world):
    spans = [shard_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
        assert e0 == s1 and s1 % 128 == 0 or s1 == n


def merge_np(o_parts, lse_parts):
    """merge_stats in log form: the restatement tatn_merge_partials is checked against."""
    m = lse_parts.max(axis=0)
    w = np.where(np.isneginf(lse_parts), 0.0, np.exp(lse_parts - np.where(np.isneginf(m), 0.0, m)))
    ws = w.sum(axis=0)
    o = (w[..., None] * o_parts).sum(axis=0) / np.where(ws > 0, ws, 1.0)[..., None]
    lse = np.where(ws > 0, m + np.log(np.where(ws > 0, ws, 1.0)), -np.inf)
    return o, lse


def _shard_keep(n, k0, k1, kind, valid_len=None):
    """Global mask of queries x shard keys as a custom keep matrix (global key = k0 + j)."""
    i = np.arange(n)[:, None]
    j = np.arange(k0, k1)[None, :]
    if kind == "causal":
        return j <= i
    if kind == "key_padding":
        return np.broadcast_to(j < valid_len, (n, k1 - k0))
    return np.ones((n, k1 - k0), bool)


@pytest.mark.parametrize("kind", ["none", "causal"])
def test_merge_of_shards_equals_full_oracle(kind):
    B, H, N, d, R = 1, 2, 300, 16, 3
    q, k, v, do = O.gaussian_inputs(B, H, N, N, d)
    o_full, lse_full = O.forward(q, k, v, mask=kind)
    dq_full, dk_full, dv_full = O.backward(q, k, v, o_full, do, lse_full, mask=kind)
    parts_o, parts_l, spans = [], [], [shard_range(N, R, r) for r in range(R)]
    for k0, k1 in spans:
        keep = _shard_keep(N, k0, k1, kind)
        o, lse = O.forward(q, k[:, :, k0:k1], v[:, :, k0:k1], mask="custom", custom=keep)
        parts_o.append(o)
        parts_l.append(lse)
    o, lse = merge_np(np.stack(parts_o), np.stack(parts_l))
    np.testing.assert_allclose(o, o_full, atol=1e-12)
    np.testing.assert_allclose(lse, lse_full, atol=1e-12)
    dq = np.zeros_like(q)
    for k0, k1 in spans:
        keep = _shard_keep(N, k0, k1, kind)
        dqp, dk, dv = O.backward(q, k[:, :, k0:k1], v[:, :, k0:k1], o, do, lse, mask="custom", custom=keep)
        dq += dqp
        np.testing.assert_allclose(dk, dk_full[:, :, k0:k1], atol=1e-10)
        np.testing.assert_allclose(dv, dv_full[:, :, k0:k1], atol=1e-10)
    np.testing.assert_allclose(dq, dq_full, atol=1e-10)


class _OracleSharded(KeyShardedAttention):
    """The orchestration under test with the oracle standing in for the kernels (CPU, fp64)."""

    kind = "causal"

    def _keep(self, q, spec, nk):
        return _shard_keep(q.shape[2], spec.k_offset, spec.k_offset + nk, self.kind)

    def _partial_fwd(self, q, k, v, spec, out=None):
        o, lse = O.forward(q.numpy(), k.numpy(), v.numpy(), mask="custom", custom=self._keep(q, spec, k.shape[2]))
        o = torch.from_numpy(o).float()
        if out is not None:
            out.copy_(o)
            o = out
        return o, torch.from_numpy(lse).float()

    def _merge(self, o_parts, lse_parts, out_dtype):
        o, lse = merge_np(o_parts.double().numpy(), lse_parts.double().numpy())
        return torch.from_numpy(o).to(out_dtype), torch.from_numpy(lse).float()

    def _partial_bwd(self, q, k, v, o32, do, lse, spec):
        dq, dk, dv = O.backward(q.numpy(), k.numpy(), v.numpy(), o32.double().numpy(), do.numpy(),
                                lse.double().numpy(), mask="custom", custom=self._keep(q, spec, k.shape[2]))
        return torch.from_numpy(dq).float(), torch.from_numpy(dk).float(), torch.from_numpy(dv).float()


def _worker(rank, world, port, N, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_14135_b200.attention import AttnSpec

    B, H, d = 1, 2, 16
    q, k, v, do = (torch.from_numpy(t) for t in O.gaussian_inputs(B, H, N, N, d))
    sp = _OracleSharded()
    k0, k1 = sp.local_keys(N)
    spec = AttnSpec(mask="causal")
    o, lse, o32 = sp.forward(q, k[:, :, k0:k1], v[:, :, k0:k1], spec, N)
    dq, dk, dv = sp.backward(q, k[:, :, k0:k1], v[:, :, k0:k1], o32, do, lse, spec, N)
    parts = [None] * world
    dist.all_gather_object(parts, (k0, k1, dk.numpy(), dv.numpy()))
    if rank == 0:
        torch.save({"o": o, "lse": lse, "dq": dq, "parts": parts}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_key_sharded_equals_single_process(tmp_path, world):
    N = 300
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "res.pt"
    mp.spawn(_worker, args=(world, port, N, str(out)), nprocs=world, join=True)
    res = torch.load(out, weights_only=False)
    q, k, v, do = O.gaussian_inputs(1, 2, N, N, 16)
    o, lse = O.forward(q, k, v, mask="causal")
    dq, dk, dv = O.backward(q, k, v, o, do, lse, mask="causal")
    np.testing.assert_allclose(res["o"].numpy(), o.astype(np.float32), atol=1e-6)
    np.testing.assert_allclose(res["lse"].numpy(), lse, atol=1e-5)
    np.testing.assert_allclose(res["dq"].numpy(), dq, atol=1e-5)
    for k0, k1, dk_r, dv_r in res["parts"]:
        np.testing.assert_allclose(dk_r, dk[:, :, k0:k1], atol=1e-5)
        np.testing.assert_allclose(dv_r, dv[:, :, k0:k1], atol=1e-5)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
@pytest.mark.parametrize("d,mask,p_drop", [(64, "causal", 0.0), (128, "none", 0.0), (64, "key_padding", 0.0),
                                           (128, "causal", 0.2), (64, "custom", 0.0)])
def test_gpu_key_shards_merge_to_full_attention(cuda_device, R, d, mask, p_drop):
    from paper_2205_14135_b200 import attention as A
    from tests import gpu_helpers as G

    B, H, N = 2, 2, 640
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")
    vl = np.array([N - 77, N - 300], dtype=np.int32) if mask == "key_padding" else None
    cm = (np.random.default_rng(5).random((N, N)) < 0.4) if mask == "custom" else None
    ref = G.oracle_full(q, k, v, do, mask=mask, valid_len=vl, p_drop=p_drop, seed=7, custom=cm)
    qd, kd, vd, dod = (G.to_dev(t, "bf16") for t in (q, k, v, do))
    spec = A.AttnSpec(mask=mask, p_drop=p_drop, seed=7)
    if vl is not None:
        spec.valid_len = torch.from_numpy(vl).cuda()
    if cm is not None:
        spec.custom = A.pack_custom_mask(torch.from_numpy(cm).cuda())

    class Virtual(KeyShardedAttention):  # R shards on one GPU, the collectives done by hand
        def __init__(self, r):
            self.group, self.world, self.rank = None, R, r

    parts = []
    for r in range(R):
        sp = Virtual(r)
        k0, k1 = sp.local_keys(N)
        local = A.AttnSpec(**{**spec.__dict__, "k_offset": k0})
        parts.append(sp._partial_fwd(qd, kd[:, :, k0:k1].contiguous(), vd[:, :, k0:k1].contiguous(), local))
    o_parts = torch.stack([p[0] for p in parts]).contiguous()
    lse_parts = torch.stack([p[1] for p in parts]).contiguous()
    o32, lse = A.merge_partials(o_parts, lse_parts)
    G.assert_close("o", o32.double().cpu().numpy(), ref["o"])
    G.assert_close("lse", lse.double().cpu().numpy(), ref["lse"])
    # the merge kernel equals its restatement on the same partials
    mo, ml = merge_np(o_parts.double().cpu().numpy(), lse_parts.double().cpu().numpy())
    np.testing.assert_allclose(o32.double().cpu().numpy(), mo, atol=2e-6)
    dq = torch.zeros(qd.shape, dtype=torch.float32, device="cuda")
    for r in range(R):
        sp = Virtual(r)
        k0, k1 = sp.local_keys(N)
        local = A.AttnSpec(**{**spec.__dict__, "k_offset": k0})
        dq_p, dk, dv = sp._partial_bwd(qd, kd[:, :, k0:k1].contiguous(), vd[:, :, k0:k1].contiguous(), o32, dod, lse,
                                       local)
        dq += dq_p
        G.assert_close("dk", dk.double().cpu().numpy(), ref["dk"][:, :, k0:k1])
        G.assert_close("dv", dv.double().cpu().numpy(), ref["dv"][:, :, k0:k1])
    G.assert_close("dq", dq.double().cpu().numpy(), ref["dq"])


@pytest.mark.gpu
def test_gpu_merge_kernel_empty_rows_and_dtypes(cuda_device):
    from paper_2205_14135_b200 import attention as A

    R, B, H, N, d = 3, 1, 2, 200, 128
    g = torch.Generator(device="cuda").manual_seed(1)
    o_parts = torch.randn((R, B, H, N, d), generator=g, device="cuda")
    lse_parts = torch.randn((R, B, H, N), generator=g, device="cuda") * 4
    lse_parts[:, :, :, 5] = float("-inf")  # no key in any shard
    lse_parts[1, :, :, 9] = float("-inf")  # shard 1 empty for row 9
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        out = torch.empty((B, H, N, d), dtype=dt, device="cuda")
        o, lse = A.merge_partials(o_parts, lse_parts, out=out)
        mo, ml = merge_np(o_parts.double().cpu().numpy(), lse_parts.double().cpu().numpy())
        tol = 2e-6 if dt == torch.float32 else 2e-2
        np.testing.assert_allclose(o.double().cpu().numpy(), mo, atol=tol, rtol=tol)
        np.testing.assert_allclose(lse.double().cpu().numpy(), ml, atol=2e-5)
        assert torch.all(o[:, :, 5] == 0) and torch.all(torch.isneginf(lse[:, :, 5]))


@pytest.mark.gpu
@pytest.mark.parametrize("R,mask", [(2, "causal"), (3, "none"), (4, "causal")])
def test_gpu_pairwise_shares_sum_to_full_attention(cuda_device, R, mask):
    """The forward exchange KeyShardedAttention uses: each shard's fp32 partial merged with
    (0, logsumexp of the other shards' LSE) by tatn_merge_partials is O_r exp(LSE_r - LSE); the
    shares sum (the all-reduce) to full attention, and every pair yields the global LSE."""
    from paper_2205_14135_b200 import attention as A
    from tests import gpu_helpers as G

    B, H, N, d = 2, 2, 700, 64
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")
    ref = G.oracle_full(q, k, v, do, mask=mask, backward=False)
    qd, kd, vd = (G.to_dev(t, "bf16") for t in (q, k, v))

    class Virtual(KeyShardedAttention):
        def __init__(self, r):
            self.group, self.world, self.rank = None, R, r

    parts = []
    for r in range(R):
        sp = Virtual(r)
        k0, k1 = sp.local_keys(N)
        local = A.AttnSpec(mask=mask, k_offset=k0)
        pair = torch.zeros((2,) + tuple(qd.shape), dtype=torch.float32, device="cuda")
        if k1 > k0:
            _, lse_r = sp._partial_fwd(qd, kd[:, :, k0:k1].contiguous(), vd[:, :, k0:k1].contiguous(), local,
                                       out=pair[0])
        else:  # R = 4 over 700 keys leaves the last shard empty: it contributes LSE = -inf, O = 0
            lse_r = torch.full(qd.shape[:3], float("-inf"), device="cuda")
        parts.append((pair, lse_r))
    lse_all = torch.stack([p[1] for p in parts])
    total = torch.zeros(qd.shape, dtype=torch.float32, device="cuda")
    for r, (pair, lse_r) in enumerate(parts):
        others = torch.cat([lse_all[:r], lse_all[r + 1:]])
        share, lse = A.merge_partials(pair, torch.stack([lse_r, torch.logsumexp(others, 0)]).contiguous())
        total += share
        G.assert_close("lse", lse.double().cpu().numpy(), ref["lse"])
    G.assert_close("o", total.double().cpu().numpy(), ref["o"])
