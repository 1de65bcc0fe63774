"""Pin the oracle against committed golden vectors and SPEC known answers (CPU).

tests/golden/*.npz were produced by the reference itself (oracle/_ref, see
tests/golden/make_golden.py), so these tests hold the oracle to the reference
even on a machine where the reference cannot be compiled.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def load_cases():
    z = np.load(GOLD / "attn_golden.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def decode16(bits, dtype):
    if dtype == "fp32":  # fp32 cases store the float32 values themselves
        return np.asarray(bits, dtype=np.float32).astype(np.float64)
    bits = np.asarray(bits, dtype=np.uint16)
    if dtype == "fp16":
        return bits.view(np.float16).astype(np.float64)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def case_inputs(z, m):
    name = m["name"]
    q, k, v, do = (decode16(z[f"{name}/{t}"], m["dtype"]) for t in ("q", "k", "v", "do"))
    grid = z[f"{name}/grid"] if m["has_grid"] else None
    vl = z[f"{name}/valid_len"] if m["has_valid_len"] else None
    return q, k, v, do, grid, vl


def test_golden_inputs_come_from_the_reference_generator():
    z, meta = load_cases()
    for m in meta:
        q, k, v, do, _, _ = case_inputs(z, m)
        B, H = m["B"], m["H"]
        for b in range(B):
            for h in range(H):
                raw = O.gaussian_matrix(m["Nq"], m["d"], O.slice_seed(b, h, H, 0))
                assert np.array_equal(O.round_to(raw, m["dtype"]), q[b, h])


def test_generator_matches_golden_seeds():
    g = np.load(GOLD / "ref_misc.npz")
    for key in g.files:
        if key.startswith("seed_"):
            seed = int(key[5:])
            assert np.array_equal(O.gaussian_matrix(8, 8, seed), g[key])


N_CASES = len(load_cases()[1])


@pytest.mark.parametrize("idx", range(N_CASES))
def test_oracle_matches_golden(idx):
    z, meta = load_cases()
    m = meta[idx]
    q, k, v, do, grid, vl = case_inputs(z, m)
    name = m["name"]
    pd, sd = m.get("p_drop", 0.0), m.get("seed", 0)
    o, lse = O.forward(q, k, v, mask=m["mask"], valid_len=vl, grid=grid, p_drop=pd, seed=sd)
    dq, dk, dv = O.backward(q, k, v, o, do, lse, mask=m["mask"], valid_len=vl, grid=grid, p_drop=pd, seed=sd)
    gl = z[f"{name}/lse"].astype(np.float64)
    assert np.array_equal(np.isneginf(lse), np.isneginf(gl))
    fin = np.isfinite(gl)
    np.testing.assert_allclose(lse[fin], gl[fin], rtol=2e-7, atol=2e-6)
    for key, val in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        ref = z[f"{name}/{key}"].astype(np.float64)
        np.testing.assert_allclose(val, ref, rtol=2e-6, atol=2e-6, err_msg=f"{name}/{key}")


def test_golden_semantics_empty_row_and_uncovered_keys():
    z, meta = load_cases()
    m = next(mm for mm in meta if mm["name"].startswith("sparse_emptyrow"))
    name = m["name"]
    assert np.all(np.isneginf(z[f"{name}/lse"][0, 0, 128:256]))
    assert np.all(z[f"{name}/o"][0, 0, 128:256] == 0)
    # padding case with valid_len = 0: every row fully masked, zero gradients
    mp = next(mm for mm in meta if mm["name"].startswith("padding"))
    nm = mp["name"]
    assert np.all(np.isneginf(z[f"{nm}/lse"][2])) and np.all(z[f"{nm}/dq"][2] == 0) and np.all(z[f"{nm}/dv"][2] == 0)


# ----------------------------------------------------------------------------- SPEC known answers
def test_singleton_attention_is_one():
    # N = d = 1, Q = K = V = [[1]], tau = 1 -> O = [[1]], l = 1, m = 1
    one = np.ones((1, 1, 1, 1))
    o, lse = O.forward(one, one, one, tau=1.0)
    assert o[0, 0, 0, 0] == 1.0 and lse[0, 0, 0] == 1.0
    dq, dk, dv = O.backward(one, one, one, o, one * 3.0, lse, tau=1.0)
    assert dv[0, 0, 0, 0] == 3.0 and dq[0, 0, 0, 0] == 0.0 and dk[0, 0, 0, 0] == 0.0


def test_zero_keys_give_column_mean():
    # K = 0 -> P uniform -> O = column mean of V
    rng = np.random.default_rng(3)
    v = rng.standard_normal((1, 1, 10, 4))
    q = rng.standard_normal((1, 1, 10, 4))
    o, _ = O.forward(q, np.zeros_like(v), v)
    np.testing.assert_allclose(o[0, 0], np.broadcast_to(v[0, 0].mean(0), (10, 4)), atol=1e-14)


def test_zero_cotangent_zero_gradients():
    # SPEC.md:144,241
    rng = np.random.default_rng(4)
    q, k, v = (rng.standard_normal((1, 2, 33, 8)) for _ in range(3))
    o, lse = O.forward(q, k, v, mask="causal")
    dq, dk, dv = O.backward(q, k, v, o, np.zeros_like(q), lse, mask="causal")
    assert not dq.any() and not dk.any() and not dv.any()


def test_plan_tiles_examples():
    # SPEC.md:223-225
    rc, p = O.plan_tiles(1024, 64, 65536)
    assert rc == 0 and (p["bc"], p["br"], p["tc"], p["tr"]) == (256, 64, 4, 16)
    rc, p = O.plan_tiles(1024, 64, 1024)
    assert (p["bc"], p["br"]) == (4, 4)
    rc, p = O.plan_tiles(1024, 64, 1 << 20, br=8, bc=8)
    assert rc == 0 and (p["bc"], p["br"]) == (8, 8) and p["working_set"] == O.lib().orc_working_set_elems(8, 8, 64)
    assert O.plan_tiles(64, 64, 100)[0] == -1  # M < 4d rejected


def test_butterfly_8x8_has_32_blocks():
    # 8 diagonal + 24 off-diagonal (i xor j in {1, 2, 4})
    g = O.block_mask_butterfly(8, 8)
    assert int(g.sum()) == 32 and np.array_equal(g, g.T) and np.all(np.diag(g) == 1)


def test_io_closed_forms_match_reference_counters():
    g = np.load(GOLD / "ref_misc.npz")
    for n, d in ((1, 1), (64, 16), (128, 8)):
        assert tuple(int(x) for x in g[f"std_fwd_{n}_{d}"][:2]) == O.predict_io("standard_forward", n, d)
        assert tuple(int(x) for x in g[f"std_bwd_{n}_{d}"][:2]) == O.predict_io("standard_backward", n, d)
    # SPEC.md:331 (code/header truth): n = 1024, d = 64 standard forward
    assert O.predict_io("standard_forward", 1024, 64) == (4390912, 2162688)
    # block-sparse with every block visited reproduces the tiled closed form (io_predict.hpp:86-90)
    n, d, br, bc = 1024, 64, 64, 256
    tr, tc = n // br, n // bc
    assert O.predict_io("blocksparse_forward", n, d, br=br, visited=tr * tc) == O.predict_io("flash_forward", n, d, tc=tc)
    assert O.predict_io("blocksparse_backward", n, d, br=br, visited=tr * tc) == O.predict_io(
        "flash_backward", n, d, tc=tc)
