"""CTA timeline summary of the d=128 (NQ=2) forward, -DTATN_TRACE build: per-CTA prologue /
loop / epilogue split and SM occupancy gaps between consecutive CTAs on an SM."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
for (B, H, N, d, mask) in [(8, 32, 2048, 128, "causal"), (4, 32, 4096, 128, "causal"), (1, 32, 16384, 128, "causal")]:
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    for _ in range(3): A.flash_fwd(q, k, v, spec)
    buf = torch.zeros(200000 * 16 + 1024 * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); A.flash_fwd(q, k, v, spec); e1.record()
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    t = buf[:200000 * 16].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    start, first_s, last_p, ofin, end, sm, steps = (t[:, i] for i in range(7))
    t0 = start.min()
    dur = (end - start) / 1e3
    ok = steps > 0
    print(f"N{N}: {len(t)} CTAs, events {e0.elapsed_time(e1)*1e3:.0f} us, span {(end.max()-t0)/1e3:.0f} us; CTA mean {dur.mean():.1f} us;"
          f" start->first S {((first_s-start)[ok]/1e3).mean():.2f}; first S->last P {((last_p-first_s)[ok]/1e3).mean():.2f};"
          f" last P->O final {((ofin-last_p)[ok]/1e3).mean():.2f}; O final->end {((end-ofin)[ok]/1e3).mean():.2f}")
    gaps = []
    for s_ in set(sm.tolist()):
        m = sm == s_
        o = np.argsort(start[m])
        st, en = start[m][o], end[m][o]
        gaps += list((st[1:] - en[:-1]) / 1e3)
    busy = dur.sum() / (len(set(sm.tolist())) * (end.max() - t0) / 1e3)
    print(f"      SM busy fraction {busy:.2f}; gap between CTAs on an SM: mean {np.mean(gaps):.2f} us")
