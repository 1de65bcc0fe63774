"""TEST INFRASTRUCTURE: write TATN golden directories for `paper_2205_14135_b200.cli verify`.

Inputs come from the reference's generator (oracle.gaussian_inputs, SURVEY.md §8(d) seeds),
rounded to the 16-bit dtype; expected outputs from the fp64 oracle on those rounded inputs
(o, lse = m + ln l, dq, dk, dv). Files use the reference's binary matrix format
(matrix_io.hpp:15-16) via paper_2205_14135_b200.tatn_io, which tests pin byte-for-byte
against the reference's own writer.

    python tests/golden/make_tatn.py OUT_DIR [n d mask dtype]
The committed fixture tests/golden/tatn_causal_n256_d64 was made with
    python tests/golden/make_tatn.py tests/golden/tatn_causal_n256_d64 256 64 causal bf16
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2205_14135_b200 import tatn_io  # noqa: E402


def make(out, n=256, d=64, mask="causal", dtype="bf16", grid=None, p_drop=0.0, seed=0):
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    q, k, v, do = (O.round_to(t, dtype) for t in O.gaussian_inputs(1, 1, n, n, d))
    kind, vl = mask, None
    if mask.startswith("padding:"):
        kind, vl = "key_padding", int(mask.split(":")[1])
    o, lse = O.forward(q, k, v, mask=kind, valid_len=vl, grid=grid, p_drop=p_drop, seed=seed)
    dq, dk, dv = O.backward(q, k, v, o, do, lse, mask=kind, valid_len=vl, grid=grid, p_drop=p_drop, seed=seed)
    for name, a in (("q", q), ("k", k), ("v", v), ("do", do), ("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
        tatn_io.write_matrix_binary(a[0, 0], out / f"{name}.tatn")
    tatn_io.write_matrix_binary(lse[0, 0].reshape(-1, 1), out / "lse.tatn")
    if grid is not None:
        tatn_io.write_matrix_binary(np.asarray(grid, dtype=np.float64), out / "grid.tatn")
    (out / "meta.json").write_text(json.dumps({"n": n, "nk": n, "d": d, "tau": None, "mask": mask, "dtype": dtype,
                                               "p_drop": p_drop, "seed": seed}))
    return out


if __name__ == "__main__":
    a = sys.argv[1:]
    make(a[0], *(int(x) for x in a[1:3]), *a[3:5])
