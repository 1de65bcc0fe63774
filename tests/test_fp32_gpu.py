"""GPU parity of the fp32-input check mode (ABI v4, TATN_DTYPE_FP32; kernels in
csrc/tatn_tf32.cuh): fp32 Q, K, V, dO multiplied on the tensor cores as tf32
(tcgen05.mma kind::tf32), P and dS rounded to tf32 on chip, fp32 outputs — against the
fp64 oracle on the SAME fp32 inputs (no 16-bit rounding anywhere).

Tolerance (north star: "tighter for an fp32-input check mode"): max abs <= 2e-3 and
rel-L2 <= 1e-3 for O, LSE, dQ, dK, dV at C1 — 10x tighter than the 16-bit bar (2e-2 / 1e-2);
the stress shapes (ragged N, key padding down to one visible key, custom masks, dropout, block
grids) hold rel-L2 <= 1e-3 and max abs <= 4e-3 * max(1, max|ref|) — tf32 keeps 11 significant
bits, a relative precision.
BASELINE configs[0] (C1: B=2 H=4 N=512 d=64 non-causal fp32) is checked at exactly its
stated precision, and against the reference's own outputs (tests/golden, c1_fp32_d64).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import gpu_helpers as G
from paper_2205_14135_b200 import attention as A

pytestmark = pytest.mark.gpu

def check(got, ref, keys=("o", "lse", "dq", "dk", "dv"), stress=True):
    """C1 (stress=False): max abs <= 2e-3, rel-L2 <= 1e-3. Stress shapes: rel-L2 <= 1e-3 and
    max abs <= 4e-3 * max(1, max|ref|) (gpu_helpers.F32_MAX_ABS_STRESS)."""
    tol = (dict(max_abs=G.F32_MAX_ABS_STRESS, scale_max_abs=True) if stress else dict(max_abs=G.F32_MAX_ABS))
    return {key: G.assert_close(key, got[key], ref[key], rel_l2=G.F32_REL_L2, **tol)
            for key in keys if key in got and key in ref}


def test_c1_fp32_input(cuda_device):
    """BASELINE configs[0]: B=2 H=4 N=512 d=64 non-causal, fp32 inputs."""
    q, k, v, do = G.make_inputs(2, 4, 512, 512, 64, "fp32")
    got = G.run_gpu(q, k, v, do, "fp32")
    assert got["o"].dtype == np.float64  # (converted) — the device tensors are fp32
    errs = check(got, G.oracle_full(q, k, v, do), stress=False)  # the absolute 2e-3 bar at C1
    print("C1 fp32 (max abs, rel-L2):", errs)


def test_fp32_is_tighter_than_16bit(cuda_device):
    """The same C1 problem: the fp32-input mode is at least 4x closer to the oracle (rel-L2)
    than bf16 inputs are to their own rounded-input oracle."""
    q, k, v, do = G.make_inputs(2, 4, 512, 512, 64, "fp32")
    ref = G.oracle_full(q, k, v, do)
    got = G.run_gpu(q, k, v, do, "fp32")
    qb, kb, vb, dob = (O.round_to(t, "bf16") for t in (q, k, v, do))
    got16 = G.run_gpu(qb, kb, vb, dob, "bf16")
    for key in ("o", "dq", "dk", "dv"):
        e32 = np.linalg.norm(got[key] - ref[key]) / np.linalg.norm(ref[key])
        e16 = np.linalg.norm(got16[key] - ref[key]) / np.linalg.norm(ref[key])  # vs the fp32-input oracle
        assert e32 * 4 <= e16, (key, e32, e16)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("mask", ["none", "causal", "key_padding", "custom"])
def test_fp32_masks_ragged(cuda_device, d, mask):
    B, H, N = 2, 2, 333
    q, k, v, do = G.make_inputs(B, H, N, N, d, "fp32")
    vl = np.array([300, 1], dtype=np.int32) if mask == "key_padding" else None
    custom = None
    if mask == "custom":
        rng = np.random.default_rng(7)
        custom = rng.random((B, N, N)) < 0.6
        custom[0, 5, :] = False  # a fully masked row: O = 0, LSE = -inf
    got = G.run_gpu(q, k, v, do, "fp32", mask=mask, valid_len=vl, custom=custom)
    check(got, G.oracle_full(q, k, v, do, mask=mask, valid_len=vl, custom=custom))


def test_fp32_key_prefix_and_strided_layout(cuda_device):
    q, k, v, do = G.make_inputs(1, 3, 400, 272, 128, "fp32")
    got = G.run_gpu(q, k, v, do, "fp32", mask="causal", layout="bnhd")
    check(got, G.oracle_full(q, k, v, do, mask="causal"))


def test_fp32_block_sparse_visited_bit_exact(cuda_device):
    N = 640
    tr = N // 128
    grid = O.block_mask_butterfly(tr, tr).astype(np.uint8)
    grid[2, :] = 0  # an empty block row: O = 0, LSE = -inf
    q, k, v, do = G.make_inputs(1, 2, N, N, 64, "fp32")
    got = G.run_gpu(q, k, v, do, "fp32", grid=grid, visited=True)
    assert np.array_equal(got["visited_fwd"], grid)
    assert np.array_equal(got["visited_bwd"], grid)
    check(got, G.oracle_full(q, k, v, do, grid=grid))


@pytest.mark.parametrize("d", [64, 128])
def test_fp32_dropout(cuda_device, d):
    q, k, v, do = G.make_inputs(1, 2, 256, 256, d, "fp32")
    got = G.run_gpu(q, k, v, do, "fp32", mask="causal", p_drop=0.2, seed=99)
    check(got, G.oracle_full(q, k, v, do, mask="causal", p_drop=0.2, seed=99))


def test_fp32_deterministic_o_lse_dk_dv(cuda_device):
    q, k, v, do = G.make_inputs(2, 2, 384, 384, 64, "fp32")
    a = G.run_gpu(q, k, v, do, "fp32", mask="causal")
    b = G.run_gpu(q, k, v, do, "fp32", mask="causal")
    for key in ("o", "lse", "dk", "dv"):
        assert np.array_equal(a[key], b[key]), key


def test_fp32_outputs_are_fp32_tensors(cuda_device):
    q, k, v, _ = (torch.randn(1, 1, 128, 64, device="cuda") for _ in range(4))
    o, lse = A.flash_fwd(q, k, v)
    assert o.dtype == torch.float32 and lse.dtype == torch.float32
    with pytest.raises(TypeError):
        A.flash_fwd(q, k, v, out=torch.empty_like(q, dtype=torch.bfloat16))
