"""Persistent kernels (K1 d=64 / d=128, K3): dynamic item claims from self-resetting device
counters must give the same results under every launch pattern — back-to-back launches reusing
a counter, concurrent launches on different streams, far more items than CTAs, items with no
tiles, and CUDA-graph replay."""
import numpy as np
import pytest
import torch

from tests import gpu_helpers as G
from paper_2205_14135_b200 import attention as A

pytestmark = pytest.mark.gpu


def _inputs(B, H, N, d, dtype="bf16", seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = G.TORCH_DT[dtype]
    return [torch.randn((B, H, N, d), generator=g, device="cuda").to(dt) for _ in range(4)]


@pytest.mark.parametrize("d", [64, 128])
def test_repeated_and_concurrent_launches_agree(cuda_device, d):
    q, k, v, do = _inputs(4, 8, 777, d)
    spec = A.AttnSpec(mask="causal")
    o0, l0 = A.flash_fwd(q, k, v, spec)
    g0 = A.flash_bwd(q, k, v, o0, do, l0, spec)
    torch.cuda.synchronize()
    for _ in range(5):  # the counters reset themselves between launches
        o1, l1 = A.flash_fwd(q, k, v, spec)
        assert torch.equal(o1, o0) and torch.equal(l1, l0)
    # concurrent launches on two streams (distinct counter slots) over different problems
    q2, k2, v2, do2 = _inputs(2, 16, 1500, d, seed=3)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = {}
    with torch.cuda.stream(s1):
        outs["a"] = A.flash_fwd(q, k, v, spec)
    with torch.cuda.stream(s2):
        outs["b"] = A.flash_fwd(q2, k2, v2, A.AttnSpec(mask="none"))
    torch.cuda.synchronize()
    assert torch.equal(outs["a"][0], o0)
    ref_b = A.flash_fwd(q2, k2, v2, A.AttnSpec(mask="none"))
    torch.cuda.synchronize()
    assert torch.equal(outs["b"][0], ref_b[0])
    # backward: dK, dV are deterministic; dQ is an fp32 reduction (order may vary)
    g1 = A.flash_bwd(q, k, v, o0, do, l0, spec)
    torch.cuda.synchronize()
    assert torch.equal(g1[1], g0[1]) and torch.equal(g1[2], g0[2])
    assert torch.allclose(g1[0].float(), g0[0].float(), atol=2e-2, rtol=0)


@pytest.mark.parametrize("d", [64, 128])
def test_many_tiny_items_and_empty_items(cuda_device, d):
    # 3000 (b, h) slices of one tile each, key padding with some batches fully padded (no tiles)
    B, H, N = 30, 100, 96
    q, k, v, do = (G.make_inputs(B, H, N, N, d, "fp16"))
    vl = np.array([0 if b % 7 == 0 else N - (b % 5) for b in range(B)], dtype=np.int32)
    got = G.run_gpu(q, k, v, do, "fp16", mask="key_padding", valid_len=vl)
    ref = G.oracle_full(q, k, v, do, mask="key_padding", valid_len=vl)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key])
    empty = vl == 0
    assert np.all(got["o"][empty] == 0) and np.all(np.isneginf(got["lse"][empty]))
    assert np.all(got["dk"][empty] == 0) and np.all(got["dq"][empty] == 0)


@pytest.mark.parametrize("d", [64, 128])
def test_every_item_without_keys(cuda_device, d):
    # every batch fully padded: no (b, h, tile) item has a key tile. The issuers run through empty
    # items while the softmax / epilogue roles keep pace, which deadlocked two bugs: the d = 64
    # forward's MMA warp waited the skipped items' QFull phases late (aliased parities), and the
    # backward's Final commits could run two phases ahead of the epilogue waiting on them.
    B, H, N = 16, 40, 96
    q, k, v, do = G.make_inputs(B, H, N, N, d, "fp16")
    vl = np.zeros(B, dtype=np.int32)
    got = G.run_gpu(q, k, v, do, "fp16", mask="key_padding", valid_len=vl)
    assert np.all(got["o"] == 0) and np.all(np.isneginf(got["lse"]))
    for key in ("dq", "dk", "dv"):
        assert np.all(got[key] == 0), key


def test_graph_replay_matches_eager(cuda_device):
    q, k, v, do = _inputs(8, 12, 1024, 64)
    spec = A.AttnSpec(mask="causal")
    o = torch.empty_like(q)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = A.bwd_workspace(q, k, v, spec)
    step = lambda: (A.flash_fwd(q, k, v, spec, out=o, lse=lse),
                    A.flash_bwd(q, k, v, o, do, lse, spec, dq, dk, dv, ws))
    step()
    torch.cuda.synchronize()
    ref = [t.clone() for t in (o, lse, dk, dv, dq)]
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    for a, b in zip((o, lse, dk, dv), ref[:4]):
        assert torch.equal(a, b)
    assert torch.allclose(dq.float(), ref[4].float(), atol=2e-2, rtol=0)


_PDL_CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A
g = torch.Generator(device="cuda").manual_seed(11)
q, k, v, do = (torch.randn((4, 8, 1000, 64), generator=g, device="cuda").half() for _ in range(4))
spec = A.AttnSpec(mask="causal")
o, lse = A.flash_fwd(q, k, v, spec)
dq, dk, dv = A.flash_bwd(q, k, v, o, do, lse, spec)
torch.save({"o": o.cpu(), "lse": lse.cpu(), "dk": dk.cpu(), "dv": dv.cpu(), "dq": dq.float().cpu()}, sys.argv[1])
'''


def test_programmatic_dependent_launch_matches_plain_launches(tmp_path):
    """Every kernel is launched with programmatic stream serialization and holds itself at
    griddepcontrol.wait; TATN_PDL=0 launches plainly. The two must give the same results."""
    import os
    import subprocess
    import sys

    res = {}
    for pdl in ("1", "0"):
        out = tmp_path / f"pdl{pdl}.pt"
        env = dict(os.environ, TATN_PDL=pdl)
        subprocess.run([sys.executable, "-c", _PDL_CHILD, str(out)], env=env, check=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        res[pdl] = torch.load(out)
    for key in ("o", "lse", "dk", "dv"):
        assert torch.equal(res["1"][key], res["0"][key]), key
    assert torch.allclose(res["1"]["dq"], res["0"]["dq"], atol=2e-2, rtol=0)


@pytest.mark.parametrize("d", [64, 128])
def test_many_concurrent_streams_and_graphs_with_eager(cuda_device, d):
    """ABI v4: the forward's work-item counter is the caller's workspace, so any number of
    concurrent launches (here 80 streams, more than round 1's 64 global counter slots) plus
    graph replays interleaved with eager launches on other streams give the reference result
    (calls may run concurrently with no coordination)."""
    spec = A.AttnSpec(mask="causal")
    probs = [_inputs(1, 4, 640, d, seed=100 + i)[:3] for i in range(8)]
    refs = []
    for q, k, v in probs:
        refs.append(A.flash_fwd(q, k, v, spec))
    torch.cuda.synchronize()
    # a graph of one forward with its own workspace
    gq, gk, gv = probs[0]
    gws = A.fwd_workspace(gq.device)
    go = torch.empty_like(gq)
    glse = torch.empty(gq.shape[:3], dtype=torch.float32, device="cuda")
    A.flash_fwd(gq, gk, gv, spec, out=go, lse=glse, workspace=gws)
    torch.cuda.synchronize()
    gs = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=gs):
        A.flash_fwd(gq, gk, gv, spec, out=go, lse=glse, workspace=gws)
    streams = [torch.cuda.Stream() for _ in range(80)]
    wss = [A.fwd_workspace(gq.device) for _ in streams]
    outs = [None] * len(streams)
    torch.cuda.synchronize()
    for rep in range(3):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                q, k, v = probs[i % len(probs)]
                outs[i] = A.flash_fwd(q, k, v, spec, workspace=wss[i])
            if i % 16 == 0:
                with torch.cuda.stream(gs):
                    graph.replay()
        torch.cuda.synchronize()
        for i, (o, lse) in enumerate(outs):
            ro, rl = refs[i % len(probs)]
            assert torch.equal(o, ro) and torch.equal(lse, rl), (rep, i)
        assert torch.equal(go, refs[0][0]) and torch.equal(glse, refs[0][1])
    # every workspace is back to zero (each launch resets its counter)
    for w in wss + [gws]:
        assert int(w.sum()) == 0
