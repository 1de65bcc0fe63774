"""Host logic of the (b, h)-sharded launcher, including a 2-rank gloo run on CPU.

On CPU the per-device attention call is replaced by the oracle (test
infrastructure standing in for the kernels); what is under test is the shard
partition, the per-slice valid_len expansion and the off-path gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_14135_b200.launcher import BHShardedAttention, DistEnv, gather_slices, shard_range, slice_batch_index


@pytest.mark.parametrize("n", [1, 7, 96, 256, 1001])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partitions(n, world):
    spans = [shard_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (s0, e0), (s1, _) in zip(spans, spans[1:]):
        assert e0 == s1
    sizes = [e - s for s, e in spans]
    assert max(sizes) - min(sizes) <= 1


def test_bad_rank():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_slice_batch_index():
    assert slice_batch_index(3, 9, 4) == [0, 1, 1, 1, 1, 2]


def _oracle_compute(q, k, v, valid_len=None):
    from oracle import oracle as O

    o, lse = O.forward(q.numpy(), k.numpy(), v.numpy(), mask="key_padding" if valid_len is not None else "none",
                       valid_len=None if valid_len is None else np.asarray(valid_len))
    return torch.from_numpy(o), torch.from_numpy(lse)


def _worker(rank, world, port, B, H, N, d, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env = DistEnv.from_env()
    g = torch.Generator().manual_seed(0)
    q, k, v = (torch.randn(B, H, N, d, generator=g, dtype=torch.float64) for _ in range(3))
    valid_len = [N - 3 * b for b in range(B)]
    sh = BHShardedAttention(B, H, env)
    # each slice of the local shard is its own (b', h') problem: B' = S, H' = 1
    ql, kl, vl = (sh.local_slices(t) for t in (q, k, v))
    o, lse = _oracle_compute(ql, kl, vl, valid_len=sh.local_valid_len(valid_len))
    o_all = gather_slices(o.contiguous(), env, B, H)
    lse_all = gather_slices(lse.contiguous(), env, B, H)
    if rank == 0:
        torch.save({"o": o_all, "lse": lse_all, "q": q, "k": k, "v": v, "vl": valid_len}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_equals_single_process(tmp_path):
    B, H, N, d = 3, 5, 40, 8  # 15 slices: uneven split 8 / 7, shards straddle batch rows
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "res.pt"
    mp.spawn(_worker, args=(2, port, B, H, N, d, str(out)), nprocs=2, join=True)
    res = torch.load(out)
    from oracle import oracle as O

    o_ref, lse_ref = O.forward(res["q"].numpy(), res["k"].numpy(), res["v"].numpy(), mask="key_padding",
                               valid_len=np.asarray(res["vl"]))
    np.testing.assert_array_equal(res["o"].numpy(), o_ref)
    np.testing.assert_array_equal(res["lse"].numpy(), lse_ref)
