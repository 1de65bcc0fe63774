"""The (b, h)-sharded launcher driving the REAL sm_100a kernels (north star part 4): two ranks
(gloo; TATN_SHARED_GPU=1 lets both share the one GPU of the test box) each run K1-K4 on their
shard_range of the B*H slices as [S, 1, N, d] with per-slice valid_len, the results are gathered
off the hot path and compared with the fp64 oracle on the whole batch; and bench.py's multi-rank
strong-scaling path runs end to end under torchrun."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import gpu_helpers as G

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, H, N, d, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), TATN_SHARED_GPU="1", TATN_DIST_BACKEND="gloo")
    sys.path.insert(0, str(ROOT))
    from paper_2205_14135_b200 import attention as A
    from paper_2205_14135_b200.launcher import BHShardedAttention, gather_slices, init_distributed

    env = init_distributed("nccl")  # the test hooks select gloo on the shared device
    torch.cuda.set_device(0)
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")  # identical on every rank (the reference generator)
    valid_len = [N - 37 * b for b in range(B)]
    sh = BHShardedAttention(B, H, env)
    dev = [sh.local_slices(torch.from_numpy(t.astype(np.float32))).to(torch.bfloat16).cuda().contiguous()
           for t in (q, k, v, do)]
    spec = A.AttnSpec(mask="key_padding",
                      valid_len=torch.tensor(sh.local_valid_len(valid_len), dtype=torch.int32, device="cuda"))
    o, lse = A.flash_fwd(dev[0], dev[1], dev[2], spec)
    dq, dk, dv = A.flash_bwd(dev[0], dev[1], dev[2], o, dev[3], lse, spec)
    torch.cuda.synchronize()
    res = {name: gather_slices(t.double().cpu().contiguous(), env, B, H)
           for name, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv))}
    if rank == 0:
        torch.save({**res, "n_local": [sh.n_local]}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_kernels_equal_oracle(cuda_device, tmp_path):
    B, H, N, d = 3, 5, 256, 64  # 15 slices: uneven split 8 / 7, shards straddle batch rows
    out = tmp_path / "res.pt"
    mp.spawn(_worker, args=(2, _port(), B, H, N, d, str(out)), nprocs=2, join=True)
    res = torch.load(out)
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")
    ref = G.oracle_full(q, k, v, do, mask="key_padding", valid_len=np.array([N - 37 * b for b in range(B)]))
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, res[key].numpy(), ref[key])


def test_bench_two_ranks_strong_scaling(cuda_device):
    env = dict(os.environ, TATN_SHARED_GPU="1", TATN_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-sweep", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    assert line["config"]["global_batch"] == 8 and "BHShardedAttention" in line["config"]["parallelism"]
    assert line["gpu_launches"] == 4 * line["steps"]
