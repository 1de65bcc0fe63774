"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libtatn_ref.so).

Run in the container that has /root/reference (after `make -C oracle`):
    python tests/golden/make_golden.py
The fixtures are committed; nothing at test time needs /root/reference.

attn_golden.npz holds, per case, the inputs (16-bit cases: raw uint16 bit patterns of
the RNE-rounded N(0,1) inputs from tatn::gaussian_matrix with the SURVEY §8(d)
seeds; fp32 cases — the tf32 check mode, BASELINE configs[0] — the inputs rounded to
binary32, stored as float32) and the reference's fp64 standard_forward /
standard_backward outputs (reference.cpp:39-204) on those rounded inputs, stored as fp32.
Block-sparse cases run the reference's standard path with the block grid
composed into a Custom additive mask (compose_block_mask, block_mask.hpp:42-46).
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

CASES = [
    # name, B, H, Nq, Nk, d, dtype, mask, valid_len, grid
    ("dense_bf16_d64", 1, 1, 256, 256, 64, "bf16", "none", None, None),
    ("causal_fp16_d128_ragged", 1, 1, 200, 200, 128, "fp16", "causal", None, None),
    ("padding_bf16_d64", 3, 1, 160, 160, 64, "bf16", "key_padding", [141, 160, 0], None),
    ("prefix_causal_bf16_d128", 1, 1, 256, 160, 128, "bf16", "causal", None, None),
    ("butterfly_bf16_d64", 1, 1, 512, 512, 64, "bf16", "none", None, "butterfly"),
    ("sparse_emptyrow_causal_bf16_d64", 1, 1, 384, 384, 64, "bf16", "causal", None, "emptyrow"),
    # dropout p = 0.2, seed 1234 (slice (b, h) uses seed + b*H + h, the C ABI's batched convention)
    ("dropout_causal_bf16_d64", 1, 2, 192, 192, 64, "bf16", "causal", None, None),
    # fp32 inputs (ABI v4 tf32 check mode): C1 itself (B=2 H=4 N=512 d=64 non-causal fp32) and two
    # masked / ragged shapes
    ("c1_fp32_d64", 2, 4, 512, 512, 64, "fp32", "none", None, None),
    ("causal_fp32_d128_ragged", 1, 2, 200, 200, 128, "fp32", "causal", None, None),
    ("padding_fp32_d64", 2, 1, 300, 300, 64, "fp32", "key_padding", [250, 17], None),
]
DROPOUT = {"dropout_causal_bf16_d64": (0.2, 1234)}


def grid_for(kind, tr, tc):
    if kind is None:
        return None
    if kind == "butterfly":
        return O.block_mask_butterfly(tr, tc)
    if kind == "emptyrow":
        g = O.block_mask_local_global(1, 0, tr, tc)
        g[1, :] = 0  # query block 1 visits nothing -> O = 0, LSE = -inf
        return g
    raise ValueError(kind)


def bits16(x, dtype):
    if dtype == "fp32":  # stored as float32 values
        return x.astype(np.float32)
    if dtype == "fp16":
        return x.astype(np.float16).view(np.uint16)
    f = x.astype(np.float32)  # already bf16-exact
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def main():
    out = {}
    meta = []
    for (name, B, H, Nq, Nk, d, dt, mask, vl, gk) in CASES:
        q = np.empty((B, H, Nq, d)); k = np.empty((B, H, Nk, d)); v = np.empty((B, H, Nk, d)); do = np.empty((B, H, Nq, d))
        for b in range(B):
            for h in range(H):
                q[b, h] = O.ref_gaussian_matrix(Nq, d, O.slice_seed(b, h, H, 0))
                k[b, h] = O.ref_gaussian_matrix(Nk, d, O.slice_seed(b, h, H, 1))
                v[b, h] = O.ref_gaussian_matrix(Nk, d, O.slice_seed(b, h, H, 2))
                do[b, h] = O.ref_gaussian_matrix(Nq, d, O.slice_seed(b, h, H, 3))
        q, k, v, do = (O.round_to(t, dt) for t in (q, k, v, do))
        tr, tc = (Nq + 127) // 128, (Nk + 127) // 128
        grid = grid_for(gk, tr, tc)
        res = {key: [] for key in ("o", "lse", "dq", "dk", "dv")}
        for b in range(B):
            for h in range(H):
                pd, sd = DROPOUT.get(name, (0.0, 0))
                r = O.ref_standard(q[b, h], k[b, h], v[b, h], do[b, h], mask=mask,
                                   valid_len=(vl[b] if vl is not None else None), grid=grid, br=128, bc=128,
                                   p_drop=pd, seed=sd + b * H + h)
                for key in res:
                    res[key].append(r[key])
        for key in res:
            shape = {"o": q.shape, "dq": q.shape, "dk": k.shape, "dv": v.shape, "lse": (B, H, Nq)}[key]
            out[f"{name}/{key}"] = np.stack(res[key]).reshape(shape).astype(np.float32)
        for key, t in (("q", q), ("k", k), ("v", v), ("do", do)):
            out[f"{name}/{key}"] = bits16(t, dt)
        if grid is not None:
            out[f"{name}/grid"] = grid
        if vl is not None:
            out[f"{name}/valid_len"] = np.asarray(vl, dtype=np.int32)
        pd, sd = DROPOUT.get(name, (0.0, 0))
        meta.append(dict(name=name, B=B, H=H, Nq=Nq, Nk=Nk, d=d, dtype=dt, mask=mask, p_drop=pd, seed=sd,
                         has_grid=grid is not None, has_valid_len=vl is not None))
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(ROOT / "tests" / "golden" / "attn_golden.npz", **out)

    gauss = {}
    for seed in (0, 1000, 1003, (1 << 40) + 7):
        gauss[f"seed_{seed}"] = O.ref_gaussian_matrix(8, 8, seed)
    # reference counters for the standard path (charged by reference.cpp itself)
    ctr = {}
    rng = np.random.default_rng(0)
    for n, d in ((1, 1), (64, 16), (128, 8)):
        x = rng.standard_normal((n, d))
        r = O.ref_standard(x, x, x, x)
        ctr[f"std_fwd_{n}_{d}"] = r["fwd_counters"]
        ctr[f"std_bwd_{n}_{d}"] = r["bwd_counters"]
    np.savez_compressed(ROOT / "tests" / "golden" / "ref_misc.npz", **gauss, **ctr)
    print("wrote", ROOT / "tests" / "golden")


if __name__ == "__main__":
    main()
