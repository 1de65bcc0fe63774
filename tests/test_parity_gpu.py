"""GPU parity: the sm_100a kernels, called through the C ABI, against the fp64
oracle on identical 16-bit-rounded inputs (tolerance: max abs <= 2e-2 and
rel-L2 <= 1e-2, BASELINE.json north star), plus the golden fixtures produced by
the reference itself and the size-independent properties used at full size.
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import gpu_helpers as G
from paper_2205_14135_b200 import attention as A
from paper_2205_14135_b200 import _lib

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def compare_all(got, ref, keys=("o", "lse", "dq", "dk", "dv")):
    for key in keys:
        if key in ref and key in got:
            G.assert_close(key, got[key], ref[key])


# ----------------------------------------------------------------------------- golden fixtures
def _golden():
    z = np.load(GOLD / "attn_golden.npz")
    return z, json.loads(bytes(z["meta"]).decode())


@pytest.mark.parametrize("idx", range(len(_golden()[1])))
def test_golden_fixture(cuda_device, idx):
    z, meta = _golden()
    m = meta[idx]
    name = m["name"]

    def dec(t):
        if m["dtype"] == "fp32":  # tf32 check mode: fp32 inputs as stored
            return z[f"{name}/{t}"].astype(np.float32).astype(np.float64)
        bits = z[f"{name}/{t}"].astype(np.uint16)
        if m["dtype"] == "fp16":
            return bits.view(np.float16).astype(np.float64)
        return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

    q, k, v, do = dec("q"), dec("k"), dec("v"), dec("do")
    grid = z[f"{name}/grid"] if m["has_grid"] else None
    vl = z[f"{name}/valid_len"] if m["has_valid_len"] else None
    got = G.run_gpu(q, k, v, do, m["dtype"], mask=m["mask"], valid_len=vl, grid=grid, visited=grid is not None,
                    p_drop=m.get("p_drop", 0.0), seed=m.get("seed", 0))
    ref = {key: z[f"{name}/{key}"].astype(np.float64) for key in ("o", "lse", "dq", "dk", "dv")}
    if m["dtype"] == "fp32":
        for key in ("o", "lse", "dq", "dk", "dv"):
            stress = name != "c1_fp32_d64"  # C1 at the absolute bar, the other fp32 fixtures at the stress bar
            G.assert_close(key, got[key], ref[key], max_abs=G.F32_MAX_ABS_STRESS if stress else G.F32_MAX_ABS,
                           rel_l2=G.F32_REL_L2, scale_max_abs=stress)
    else:
        compare_all(got, ref)
    if grid is not None:
        assert np.array_equal(got["visited_fwd"], grid)
        assert np.array_equal(got["visited_bwd"], grid)


# ----------------------------------------------------------------------------- BASELINE configs
def test_c1_shape_bf16_and_fp16(cuda_device):
    # C1: B=2 H=4 N=512 d=64 non-causal (the reference's CPU oracle shape), in 16-bit
    for dt in ("bf16", "fp16"):
        q, k, v, do = G.make_inputs(2, 4, 512, 512, 64, dt)
        compare_all(G.run_gpu(q, k, v, do, dt), G.oracle_full(q, k, v, do))


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("mask", ["none", "causal", "key_padding"])
def test_fp32_output_check_mode_is_tighter(cuda_device, d, mask):
    # the "fp32 check mode": 16-bit inputs, fp32 outputs (no output rounding);
    # tolerance 2x (max abs) and 3x (rel-L2) tighter than the 16-bit-output bar; the
    # remaining error is P and dS rounded to 16 bits inside the MMAs
    vl = np.array([700, 1], dtype=np.int32) if mask == "key_padding" else None
    q, k, v, do = G.make_inputs(2, 2, 777, 777, d, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask=mask, valid_len=vl, out_fp32=True)
    ref = G.oracle_full(q, k, v, do, mask=mask, valid_len=vl)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key], max_abs=1e-2, rel_l2=3e-3)


def test_c2_gpt2_small_causal_fp16(cuda_device):
    # C2: GPT-2 small attention, B=8 H=12 N=1024 d=64 causal fp16, every slice
    q, k, v, do = G.make_inputs(8, 12, 1024, 1024, 64, "fp16")
    compare_all(G.run_gpu(q, k, v, do, "fp16", mask="causal"), G.oracle_full(q, k, v, do, mask="causal"))


def test_c3_bert_large_padding_bf16(cuda_device):
    # C3: BERT-large, B=16 H=16 N=512 d=64 bf16, valid_len[b] ~ U{N-20..N}
    rng = np.random.default_rng(2124)
    vl = rng.integers(512 - 20, 513, size=16).astype(np.int32)
    q, k, v, do = G.make_inputs(16, 16, 512, 512, 64, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask="key_padding", valid_len=vl)
    compare_all(got, G.oracle_full(q, k, v, do, mask="key_padding", valid_len=vl))


def test_c4_long_context_n2048_d128_causal(cuda_device):
    # C4 at N=2K: B = 16384/N = 8, H = 32, d=128, bf16 causal. GPU on the full batch,
    # fp64 oracle on a sample of 8 (b, h) slices.
    B, H, N, d = 8, 32, 2048, 128
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask="causal")
    pick = [(0, 0), (1, 7), (2, 13), (3, 31), (4, 16), (5, 3), (6, 22), (7, 30)]
    bi = np.array([p[0] for p in pick]); hi = np.array([p[1] for p in pick])
    sub = lambda t: t[bi, hi][:, None]
    ref = G.oracle_full(sub(q), sub(k), sub(v), sub(do), mask="causal")
    compare_all({key: sub(val) for key, val in got.items()}, ref)


@pytest.mark.parametrize("N", [4096, 8192, 16384])
def test_c4_sampled_rows_and_identities(cuda_device, N):
    # C4 at N = 4K, 8K, 16K (B = 16384/N, H=32, d=128 causal): full-size run; sampled query rows
    # of O, LSE and dQ against the oracle for three heads, and the exact identities
    #   sum_j dK_j = 0  and  sum_j dV_j = sum_i dO_i   (rows of P sum to 1)
    B, H, d = 16384 // N, 32, 128
    heads = [(0, 0), (B - 1, 17), (B // 2, 31)]
    dev, kept = G.make_device_inputs(B, H, N, d, "bf16", keep_heads=heads)
    # fp32 outputs: D = dO.O then uses the unrounded O, as the reference does
    out = G.run_device(dev, "bf16", mask="causal", out_fp32=True)
    rows = np.unique(np.array([0, 1, 127, 128, N // 4 - 1, N // 2 - 1, N // 2, (3 * N) // 4 + 57, N - 1]))
    for (b, h) in heads:
        q, k, v, do = (kept[(b, h, n)] for n in ("q", "k", "v", "do"))
        o_r, lse_r = O.forward_rows(q, k, v, rows, mask="causal")
        G.assert_close("o", out["o"][b, h][rows].double().cpu().numpy(), o_r)
        G.assert_close("lse", out["lse"][b, h][rows].double().cpu().numpy(), lse_r)
        dq_r = O.backward_dq_rows(q, k, v, o_r, do, lse_r, rows, mask="causal")
        G.assert_close("dq", out["dq"][b, h][rows].double().cpu().numpy(), dq_r)
    G.check_identities(out, dev)


@pytest.mark.parametrize("N", [16384, 32768, 65536])
def test_c5_butterfly_visited_and_sampled_rows(cuda_device, N):
    # C5: block-sparse FlashAttention, butterfly 128x128 blocks, N = 16K, 32K, 64K (Path-X /
    # Path-256 shapes), d=64, B = 65536/N, H = 16. Visited tiles must equal the grid bit-exactly.
    B, H, d = 65536 // N, 16, 64
    tr = N // 128
    grid = O.block_mask_butterfly(tr, tr)
    heads = [(0, 0), (B - 1, 15)]
    dev, kept = G.make_device_inputs(B, H, N, d, "bf16", keep_heads=heads)
    out = G.run_device(dev, "bf16", grid=grid, visited=True, out_fp32=True)
    assert np.array_equal(out["visited_fwd"], grid)
    assert np.array_equal(out["visited_bwd"], grid)
    rows = np.array([0, 77, 128, 5000, 9999, N // 2 + 3, N - 129, N - 1])
    for (b, h) in heads:
        q, k, v, do = (kept[(b, h, n)] for n in ("q", "k", "v", "do"))
        o_r, lse_r = O.forward_rows(q, k, v, rows, grid=grid)
        G.assert_close("o", out["o"][b, h][rows].double().cpu().numpy(), o_r)
        G.assert_close("lse", out["lse"][b, h][rows].double().cpu().numpy(), lse_r)
        dq_r = O.backward_dq_rows(q, k, v, o_r, do, lse_r, rows, grid=grid)
        G.assert_close("dq", out["dq"][b, h][rows].double().cpu().numpy(), dq_r)
    G.check_identities(out, dev)


def test_c5_butterfly_n2048_full_parity(cuda_device):
    B, H, N, d = 2, 4, 2048, 64
    grid = O.block_mask_butterfly(N // 128, N // 128)
    q, k, v, do = G.make_inputs(B, H, N, N, d, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", grid=grid, visited=True)
    assert np.array_equal(got["visited_fwd"], grid) and np.array_equal(got["visited_bwd"], grid)
    compare_all(got, G.oracle_full(q, k, v, do, grid=grid))


# ----------------------------------------------------------------------------- block-sparse semantics
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_all_true_grid_is_bit_identical_to_dense(cuda_device, mask):
    # flash.hpp:62-63: with an all-true mask the outputs are bit-identical to the dense path
    N, d = 1000, 128
    q, k, v, do = G.make_inputs(2, 3, N, N, d, "bf16")
    dense = G.run_gpu(q, k, v, do, "bf16", mask=mask)
    tr = (N + 127) // 128
    sparse = G.run_gpu(q, k, v, do, "bf16", mask=mask, grid=np.ones((tr, tr), np.uint8))
    for key in ("o", "lse", "dk", "dv"):
        assert np.array_equal(dense[key], sparse[key]), key
    G.assert_close("dq", sparse["dq"], dense["dq"], max_abs=1e-3, rel_l2=1e-4)  # dQ sums in arbitrary order


def test_empty_rows_and_uncovered_key_tiles(cuda_device):
    N, d = 512, 64
    grid = O.block_mask_local_global(0, 0, 4, 4)  # diagonal
    grid[2, :] = 0       # query block 2 visits nothing: O = 0, LSE = -inf, dQ = 0
    grid[:, 3] = 0       # key block 3 covered by nothing: dK = dV = 0 exactly (flash.hpp:70)
    q, k, v, do = G.make_inputs(1, 2, N, N, d, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", grid=grid, visited=True)
    assert np.array_equal(got["visited_fwd"], grid) and np.array_equal(got["visited_bwd"], grid)
    assert np.all(got["o"][:, :, 256:384] == 0) and np.all(np.isneginf(got["lse"][:, :, 256:384]))
    assert np.all(got["dq"][:, :, 256:384] == 0)
    assert np.all(got["dk"][:, :, 384:] == 0) and np.all(got["dv"][:, :, 384:] == 0)
    assert np.all(got["dk"][:, :, 256:384] == 0) and np.all(got["dv"][:, :, 256:384] == 0)
    compare_all(got, G.oracle_full(q, k, v, do, grid=grid))


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("N", [1, 65, 129, 777])
@pytest.mark.parametrize("d", [64, 128])
def test_ragged_lengths(cuda_device, N, d):
    for mask in ("none", "causal"):
        q, k, v, do = G.make_inputs(1, 2, N, N, d, "bf16")
        compare_all(G.run_gpu(q, k, v, do, "bf16", mask=mask), G.oracle_full(q, k, v, do, mask=mask))


@pytest.mark.parametrize("mask", ["none", "causal"])
def test_key_prefix(cuda_device, mask):
    # K/V may be a key prefix (nk <= n), masks at global positions (reference.hpp:43-46)
    q, k, v, do = G.make_inputs(2, 2, 700, 333, 128, "fp16")
    compare_all(G.run_gpu(q, k, v, do, "fp16", mask=mask), G.oracle_full(q, k, v, do, mask=mask))


def test_fully_masked_rows(cuda_device):
    # valid_len = 0 -> every row fully masked: O = 0, LSE = -inf, zero gradients.
    # valid_len = 1 gives dV_0 = sum of 300 dO rows (|dV| ~ 40): fp32 outputs, since a
    # bf16 output alone rounds such values by up to 0.125.
    vl = np.array([0, 1, 200, 300], dtype=np.int32)
    q, k, v, do = G.make_inputs(4, 2, 300, 300, 64, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask="key_padding", valid_len=vl, out_fp32=True)
    assert np.all(got["o"][0] == 0) and np.all(np.isneginf(got["lse"][0]))
    assert not got["dq"][0].any() and not got["dk"][0].any() and not got["dv"][0].any()
    compare_all(got, G.oracle_full(q, k, v, do, mask="key_padding", valid_len=vl))


def test_strided_bnhd_layout(cuda_device):
    q, k, v, do = G.make_inputs(2, 3, 384, 384, 128, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask="causal", layout="bnhd")
    compare_all(got, G.oracle_full(q, k, v, do, mask="causal"))


def test_zero_cotangent_gives_zero_gradients(cuda_device):
    q, k, v, _ = G.make_inputs(1, 2, 256, 256, 64, "bf16")
    got = G.run_gpu(q, k, v, np.zeros_like(q), "bf16", mask="causal")
    assert not got["dq"].any() and not got["dk"].any() and not got["dv"].any()


def test_forward_and_dkdv_are_deterministic(cuda_device):
    q, k, v, do = G.make_inputs(2, 4, 1024, 1024, 128, "bf16")
    a = G.run_gpu(q, k, v, do, "bf16", mask="causal")
    b = G.run_gpu(q, k, v, do, "bf16", mask="causal")
    for key in ("o", "lse", "dk", "dv"):
        assert np.array_equal(a[key], b[key]), key


# ----------------------------------------------------------------------------- errors (fail loudly)
def test_error_codes_surface(cuda_device):
    q = torch.randn(1, 1, 256, 64, device="cuda", dtype=torch.bfloat16)
    bad_grid = torch.ones((3, 2), dtype=torch.uint8, device="cuda")
    with pytest.raises(_lib.TatnError) as e:
        A.flash_fwd(q, q, q, A.AttnSpec(block_grid=bad_grid))
    assert e.value.status == _lib.TATN_E_MASK
    with pytest.raises(_lib.TatnError) as e:
        A.flash_fwd(q, q, q, A.AttnSpec(tau=-1.0))
    assert e.value.status == _lib.TATN_E_ARG
    with pytest.raises(TypeError):  # fp64 is not a device input type (fp32 selects the tf32 check mode)
        A.flash_fwd(q.double(), q.double(), q.double())


# ----------------------------------------------------------------------------- dropout
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("p_drop,mask", [(0.1, "causal"), (0.5, "none"), (0.3, "key_padding")])
def test_dropout_parity(cuda_device, d, p_drop, mask):
    # same positional mask as the reference (dropout.cpp), regenerated in the backward
    vl = np.array([333, 64], dtype=np.int32) if mask == "key_padding" else None
    q, k, v, do = G.make_inputs(2, 3, 333, 333, d, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask=mask, valid_len=vl, out_fp32=True, p_drop=p_drop, seed=99)
    compare_all(got, G.oracle_full(q, k, v, do, mask=mask, valid_len=vl, p_drop=p_drop, seed=99))


@pytest.mark.parametrize("d", [64, 128])
def test_dropout_mask_bit_exact(cuda_device, d):
    # Q = K = 0 makes every P_ij = 1/N, so with V = I the forward output is O = Z / N
    # (Z = the dropout scale matrix) and with dO = I the backward gives dV^T = Z / N:
    # the zero pattern of O and of dV^T is the kept/dropped mask itself, bit for bit.
    N, p_drop, seed = d, 0.4, 2**40 + 3
    B, H = 1, 2
    zeros = np.zeros((B, H, N, d))
    eye = np.broadcast_to(np.eye(N, d), (B, H, N, d)).copy()
    got = G.run_gpu(zeros, zeros, eye, eye, "bf16", p_drop=p_drop, seed=seed, out_fp32=True)
    for h in range(H):
        ref = np.array([[O.dropout_scale(seed + h, i, j, p_drop) for j in range(N)] for i in range(N)])
        assert np.array_equal(got["o"][0, h] != 0, ref != 0), "forward mask differs"
        assert np.array_equal(got["dv"][0, h].T != 0, ref != 0), "backward mask differs"
        np.testing.assert_allclose(got["o"][0, h], ref / N, rtol=4e-3)  # P/(1-p) is rounded to bf16 for the MMA
