"""Deterministic dQ (ABI v4 desc.deterministic): every key tile stores its dQ partial in its own
workspace slot and K4 sums the slots in key-tile order, so dQ is bit-reproducible run to run and an
all-true block grid reproduces the dense engine's dQ bit for bit — the contract of
flash.hpp:62-63 / SPEC.md:250 for every output, dQ included."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import gpu_helpers as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,dtype", [(64, "fp16"), (128, "bf16"), (64, "fp32")])
def test_deterministic_dq_is_bit_reproducible_and_correct(cuda_device, d, dtype):
    q, k, v, do = G.make_inputs(2, 3, 1000, 1000, d, dtype)
    a = G.run_gpu(q, k, v, do, dtype, mask="causal", deterministic=True)
    b = G.run_gpu(q, k, v, do, dtype, mask="causal", deterministic=True)
    for key in ("o", "lse", "dq", "dk", "dv"):
        assert np.array_equal(a[key], b[key]), key
    ref = G.oracle_full(q, k, v, do, mask="causal")
    tol = dict(max_abs=G.F32_MAX_ABS_STRESS, rel_l2=G.F32_REL_L2, scale_max_abs=True) if dtype == "fp32" else {}
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, a[key], ref[key], **tol)
    # the atomic (default) mode agrees to rounding
    c = G.run_gpu(q, k, v, do, dtype, mask="causal")
    G.assert_close("dq", c["dq"], a["dq"], max_abs=2e-3 if dtype != "fp32" else 1e-5, rel_l2=1e-3 if dtype != "fp32" else 1e-6)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_all_true_grid_equals_dense_bit_for_bit_including_dq(cuda_device, d, mask):
    N = 1000
    q, k, v, do = G.make_inputs(2, 3, N, N, d, "bf16")
    tr = (N + 127) // 128
    dense = G.run_gpu(q, k, v, do, "bf16", mask=mask, deterministic=True)
    sparse = G.run_gpu(q, k, v, do, "bf16", mask=mask, grid=np.ones((tr, tr), np.uint8), deterministic=True)
    for key in ("o", "lse", "dq", "dk", "dv"):
        assert np.array_equal(dense[key], sparse[key]), key


def test_deterministic_with_padding_and_sparse_grid(cuda_device):
    N = 640
    vl = np.array([600, 130], np.int32)
    grid = O.block_mask_butterfly(N // 128, N // 128)
    q, k, v, do = G.make_inputs(2, 2, N, N, 64, "bf16")
    got = G.run_gpu(q, k, v, do, "bf16", mask="key_padding", valid_len=vl, deterministic=True)
    ref = G.oracle_full(q, k, v, do, mask="key_padding", valid_len=vl)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key])
    got = G.run_gpu(q, k, v, do, "bf16", grid=grid, deterministic=True)
    ref = G.oracle_full(q, k, v, do, grid=grid)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key])
