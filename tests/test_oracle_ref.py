"""Pin the C restatement (oracle/tatn_oracle.c) against the reference's own
sources compiled into oracle/_ref (CPU only).

SPEC.md:486 asks flash == standard within 1e-10 over randomized configs with
ragged N, all mask kinds; the same bar is used here for oracle == reference.
Skipped where oracle/_ref was not built (a box without /root/reference at build
time); tests/test_oracle_golden.py pins the oracle in that case.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (compiled reference) not built")


@pytest.mark.parametrize("seed", [0, 1, 1000, 1003, 2**40 + 7, 2**63 + 5])
def test_gaussian_generator_bit_exact(seed):
    for rows, cols in ((1, 1), (3, 5), (17, 9)):
        assert np.array_equal(O.gaussian_matrix(rows, cols, seed), O.ref_gaussian_matrix(rows, cols, seed))


def _rand_case(rng):
    n = int(rng.integers(1, 200))
    nk = int(rng.integers(1, n + 1))
    d = int(rng.choice([1, 2, 4, 16, 64]))
    mask = str(rng.choice(["none", "causal", "key_padding"]))
    vl = int(rng.integers(0, nk + 1)) if mask == "key_padding" else None
    tau = float(rng.uniform(0.05, 2.0))
    return n, nk, d, mask, vl, tau


def _check(n, nk, d, mask, vl, tau, grid=None, br=128, bc=128, rng=None):
    rng = rng or np.random.default_rng(0)
    q = rng.standard_normal((n, d)); k = rng.standard_normal((nk, d)); v = rng.standard_normal((nk, d))
    do = rng.standard_normal((n, d))
    r = O.ref_standard(q, k, v, do, tau=tau, mask=mask, valid_len=vl, grid=grid, br=br, bc=bc)
    o, lse = O.forward(q[None, None], k[None, None], v[None, None], tau=tau, mask=mask, valid_len=vl, grid=grid,
                       br=br, bc=bc, threads=1)
    dq, dk, dv = O.backward(q[None, None], k[None, None], v[None, None], o, do[None, None], lse, tau=tau, mask=mask,
                            valid_len=vl, grid=grid, br=br, bc=bc, threads=1)
    np.testing.assert_allclose(o[0, 0], r["o"], rtol=0, atol=1e-10)
    # -inf rows must agree exactly (fully masked convention, softmax.cpp:30-33)
    assert np.array_equal(np.isneginf(lse[0, 0]), np.isneginf(r["lse"]))
    fin = np.isfinite(r["lse"])
    np.testing.assert_allclose(lse[0, 0][fin], r["lse"][fin], rtol=0, atol=1e-10)
    for a, b in ((dq, r["dq"]), (dk, r["dk"]), (dv, r["dv"])):
        np.testing.assert_allclose(a[0, 0], b, rtol=0, atol=1e-10)


@pytest.mark.parametrize("case", range(60))
def test_random_configs_match_reference(case):
    rng = np.random.default_rng(100 + case)
    n, nk, d, mask, vl, tau = _rand_case(rng)
    _check(n, nk, d, mask, vl, tau, rng=rng)


@pytest.mark.parametrize("kind", ["butterfly", "local_global", "random_rows"])
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_block_sparse_matches_reference_custom_mask(kind, mask):
    # blocksparse == standard with the expanded element mask (block_mask.hpp:42-46)
    br = bc = 16
    n = 8 * br - 5  # ragged last block
    tr = tc = (n + br - 1) // br
    if kind == "butterfly":
        g = O.block_mask_butterfly(tr, tc)
    elif kind == "local_global":
        g = O.block_mask_local_global(1, 1, tr, tc)
    else:
        g = (np.random.default_rng(5).random((tr, tc)) < 0.3).astype(np.uint8)
        g[2, :] = 0  # an empty block row -> O = 0, LSE = -inf
    _check(n, n, 8, mask, None, 0.3, grid=g, br=br, bc=bc)


def test_memeff_reference_agrees_with_oracle():
    rng = np.random.default_rng(7)
    n, d = 96, 16
    q = rng.standard_normal((n, d)); k = rng.standard_normal((n, d)); v = rng.standard_normal((n, d))
    r = O.ref_standard(q, k, v, mask="causal")
    o, lse = O.forward(q[None, None], k[None, None], v[None, None], mask="causal")
    np.testing.assert_allclose(o[0, 0], r["o"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(lse[0, 0], r["m"] + np.log(r["l"]), atol=1e-12, rtol=0)


def test_standard_counters_equal_closed_forms():
    # io_predict.hpp:25-37 closed forms == the reference's instrumented counters
    rng = np.random.default_rng(1)
    for n, d in ((1, 1), (33, 4), (64, 16)):
        x = rng.standard_normal((n, d))
        r = O.ref_standard(x, x, x, x)
        assert tuple(int(c) for c in r["fwd_counters"][:2]) == O.predict_io("standard_forward", n, d)
        assert tuple(int(c) for c in r["bwd_counters"][:2]) == O.predict_io("standard_backward", n, d)
        assert int(r["fwd_counters"][2]) == O.flop_model(0, n, d)
        assert int(r["bwd_counters"][2]) == O.flop_model(1, n, d)


def test_dropout_generator_bit_exact():
    # dropout.cpp:7-27: the oracle's restatement of the positional PRNG equals the reference's
    rng = np.random.default_rng(9)
    for _ in range(300):
        seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        i, j = int(rng.integers(0, 1 << 20)), int(rng.integers(0, 1 << 20))
        p = float(rng.choice([0.0, 0.1, 0.5, 0.9, float(rng.random())]))
        assert O.dropout_scale(seed, i, j, p) == O.ref_dropout_scale(seed, i, j, p)


@pytest.mark.parametrize("p_drop,seed,mask", [(0.1, 7, "none"), (0.5, 3, "causal"), (0.2, 2**40 + 1, "key_padding")])
def test_dropout_matches_reference(p_drop, seed, mask):
    # flash == standard with the same seed (here: the oracle == the reference)
    rng = np.random.default_rng(11)
    n, d = 90, 8
    vl = 61 if mask == "key_padding" else None
    q, k, v, do = (rng.standard_normal((n, d)) for _ in range(4))
    r = O.ref_standard(q, k, v, do, mask=mask, valid_len=vl, p_drop=p_drop, seed=seed)
    o, lse = O.forward(q[None, None], k[None, None], v[None, None], mask=mask, valid_len=vl, p_drop=p_drop, seed=seed)
    dq, dk, dv = O.backward(q[None, None], k[None, None], v[None, None], o, do[None, None], lse, mask=mask,
                            valid_len=vl, p_drop=p_drop, seed=seed)
    for a, b in ((o, r["o"]), (dq, r["dq"]), (dk, r["dk"]), (dv, r["dv"])):
        np.testing.assert_allclose(a[0, 0], b, rtol=0, atol=1e-10)
