"""Error report of the fp32-input (tf32) check mode vs the fp64 oracle (debug aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tests import gpu_helpers as G  # noqa: E402

for (B, H, N, d, mask) in [(1, 1, 128, 64, "none"), (1, 1, 128, 128, "none"), (1, 1, 256, 64, "none"),
                           (2, 4, 512, 64, "none"), (1, 1, 256, 128, "causal")]:
    q, k, v, do = G.make_inputs(B, H, N, N, d, "fp32")
    got = G.run_gpu(q, k, v, do, "fp32", mask=mask)
    ref = G.oracle_full(q, k, v, do, mask=mask)
    line = []
    for key in ("o", "lse", "dq", "dk", "dv"):
        e = np.abs(got[key] - ref[key])
        rel = np.linalg.norm(got[key] - ref[key]) / np.linalg.norm(ref[key])
        line.append(f"{key}: max {e.max():.2e} rel {rel:.2e}")
    print(B, H, N, d, mask, " | ".join(line), flush=True)
    if N == 128 and d == 64:
        print("o[0,0,0,:8] got", got["o"][0, 0, 0, :8], "\n            ref", ref["o"][0, 0, 0, :8])
        print("lse got", got["lse"][0, 0, :4], "ref", ref["lse"][0, 0, :4])
