"""Custom n x n masks (MaskKind::Custom, attn_config.hpp:16,27).

CPU: the oracle's custom-mask semantics equal the reference's own standard_forward/backward
with MaskSpec::custom_additive (including fully-masked rows -> O = 0, LSE = -inf, and key
prefixes). GPU: the sm_100a kernels with the bit-packed mask of the C ABI against the oracle
(north-star tolerance), shared and per-batch masks, and a custom mask equal to the causal
pattern reproduces mask="causal".
"""
import numpy as np
import pytest

from oracle import oracle as O

need_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (the reference compiled here) not built")


def _mask(rng, n, nk, density):
    m = rng.random((n, nk)) < density
    m[min(3, n - 1), :] = False  # a fully masked row
    m[:, min(5, nk - 1)] = False  # a key nobody attends to
    return m


@need_ref
@pytest.mark.parametrize("n,nk,d,density", [(37, 37, 8, 0.6), (50, 33, 16, 0.3), (64, 64, 4, 0.9), (1, 1, 3, 1.0)])
def test_oracle_custom_matches_reference(n, nk, d, density):
    rng = np.random.default_rng(n * 7 + nk)
    q, do = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    k, v = rng.standard_normal((nk, d)), rng.standard_normal((nk, d))
    cm = _mask(rng, n, nk, density) if n > 1 else np.ones((1, 1), bool)
    r = O.ref_standard(q, k, v, do, mask="custom", custom=cm)
    o, lse = O.forward(q[None, None], k[None, None], v[None, None], mask="custom", custom=cm)
    dq, dk, dv = O.backward(q[None, None], k[None, None], v[None, None], o, do[None, None], lse, mask="custom",
                            custom=cm)
    assert np.array_equal(np.isneginf(lse[0, 0]), np.isneginf(r["lse"]))
    fin = np.isfinite(r["lse"])
    assert np.abs(lse[0, 0][fin] - r["lse"][fin]).max(initial=0) <= 1e-12
    for got, ref in ((o, r["o"]), (dq, r["dq"]), (dk, r["dk"]), (dv, r["dv"])):
        assert np.abs(got[0, 0] - ref).max() <= 1e-12
    if n > 3:
        assert np.all(o[0, 0, 3] == 0.0) and np.isneginf(lse[0, 0, 3])


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("N,d,dtype,density", [(200, 64, "bf16", 0.5), (513, 128, "fp16", 0.2),
                                               (384, 64, "fp16", 0.95), (256, 128, "bf16", 0.7)])
def test_custom_mask_parity(cuda_device, N, d, dtype, density):
    from tests import gpu_helpers as G

    rng = np.random.default_rng(N + d)
    q, k, v, do = G.make_inputs(1, 2, N, N, d, dtype)
    cm = _mask(rng, N, N, density)
    got = G.run_gpu(q, k, v, do, dtype, mask="custom", custom=cm)
    ref = G.oracle_full(q, k, v, do, mask="custom", custom=cm)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key])
    assert np.all(got["o"][:, :, 3] == 0.0) and np.all(np.isneginf(got["lse"][:, :, 3]))
    assert np.all(got["dk"][:, :, 5] == 0.0) and np.all(got["dv"][:, :, 5] == 0.0)


@pytest.mark.gpu
def test_custom_mask_per_batch_and_key_prefix(cuda_device):
    from tests import gpu_helpers as G

    rng = np.random.default_rng(11)
    B, H, Nq, Nk, d = 3, 2, 300, 190, 64
    q, k, v, do = G.make_inputs(B, H, Nq, Nk, d, "bf16")
    cm = np.stack([_mask(rng, Nq, Nk, dens) for dens in (0.2, 0.5, 0.8)])
    got = G.run_gpu(q, k, v, do, "bf16", mask="custom", custom=cm)
    ref = G.oracle_full(q, k, v, do, mask="custom", custom=cm)
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key])


@pytest.mark.gpu
@pytest.mark.parametrize("d", [64, 128])
def test_custom_causal_pattern_equals_causal(cuda_device, d):
    from tests import gpu_helpers as G

    N = 640
    q, k, v, do = G.make_inputs(2, 2, N, N, d, "bf16")
    tri = np.tril(np.ones((N, N), bool))
    a = G.run_gpu(q, k, v, do, "bf16", mask="custom", custom=tri)
    b = G.run_gpu(q, k, v, do, "bf16", mask="causal")
    # same result up to rounding (one output ulp): causal full tiles take 1/8 of their exponentials from the
    # FMA-pipe polynomial, every custom tile goes through the masked (MUFU) path
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, a[key], b[key], max_abs=4e-2, rel_l2=2e-3)  # <= ~1 bf16 ulp of |dV| ~ 5
