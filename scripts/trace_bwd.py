"""Per-CTA timeline of the backward kernel K3 from a -DTATN_TRACE build (lib/variants/lib_trace.so)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ["TATN_B200_LIB"] = os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so")
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
cases = [(8, 12, 1024, 64, "causal"), (16, 16, 512, 64, "key_padding"), (1, 32, 4096, 128, "causal")]
for (B, H, N, d, mask) in cases:
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    do = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    if mask == "key_padding":
        spec.valid_len = torch.full((B,), N - 7, dtype=torch.int32, device="cuda")
    o, lse = A.flash_fwd(q, k, v, spec)
    for _ in range(3): A.flash_bwd(q, k, v, o, do, lse, spec)
    buf = torch.zeros(200000 * 16, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    A.flash_bwd(q, k, v, o, do, lse, spec); torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    t = buf.view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    start, kv, s0, lastp, final, sm, n, end, dqdone = (t[:, i] for i in range(9))
    s9, p10, m11, q12, q13 = (t[:, i] for i in range(9, 14))
    us = lambda a, b, m=None: float(((b - a) / 1000.0)[m if m is not None else slice(None)].mean())
    print(f"== B{B} H{H} N{N} d{d} {mask}: {len(t)} CTAs, kernel span {(end.max() - t0) / 1000:.1f} us")
    dur = (end - start) / 1000.0
    print(f"   CTA dur us: mean {dur.mean():.2f} min {dur.min():.2f} max {dur.max():.2f}; iters mean {n.mean():.1f} max {n.max()}")
    print(f"   start->KV landed {us(start, kv):.2f}; start->first S {us(start, s0):.2f}; first S->last P {us(s0, lastp):.2f}"
          f" (per iter {float(((lastp - s0) / np.maximum(n - 1, 1) / 1000).mean()):.3f}); last P->final {us(lastp, final):.2f};"
          f" final->end {us(final, end):.2f}; dQ done->end {us(dqdone, end):.2f}")
    m = n >= 4
    print(f"   iter 2: S->P {us(s9, p10, m):.3f}; P->MMA back {us(p10, m11, m):.3f}; back->dQ full {us(m11, q12, m):.3f};"
          f" dQ full->reduce {us(q12, q13, m):.3f}")
    for s_ in sorted(set(sm.tolist()))[:3]:
        mm = sm == s_
        order = np.argsort(start[mm])
        print(f"   SM {s_}: " + ", ".join(f"[{(a - t0) / 1000:.1f},{(b - t0) / 1000:.1f}]x{c}"
                                      for a, b, c in zip(start[mm][order], end[mm][order], n[mm][order])))
