"""CTA start/end spans of a persistent kernel (globaltimer, -DTATN_TRACE build): fwd for d=64, bwd."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
for which in ("fwd", "bwd"):
    for (B, H, N, d, mask) in [(8, 12, 1024, 64, "causal"), (16, 16, 512, 64, "none")]:
        q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
        do = torch.randn_like(q)
        spec = A.AttnSpec(mask=mask)
        o, lse = A.flash_fwd(q, k, v, spec)
        run = (lambda: A.flash_fwd(q, k, v, spec)) if which == "fwd" else (lambda: A.flash_bwd(q, k, v, o, do, lse, spec))
        for _ in range(3): run()
        buf = torch.zeros(200000 * 16 + 1024 * 8, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record()
        torch.cuda.synchronize()
        lib.tatn_debug_set_trace(ctypes.c_void_p(0))
        t = buf[:200000 * 16].view(-1, 16).cpu().numpy()
        t = t[t[:, 0] > 0]
        start, end, sm = t[:, 0], t[:, 7], t[:, 5]
        t0 = start.min()
        span = (end.max() - t0) / 1e3
        busy = (end - start) / 1e3
        print(f"{which} B{B} H{H} N{N} d{d} {mask}: {len(t)} CTAs, events {e0.elapsed_time(e1)*1e3:.1f} us, CTA span {span:.1f} us;"
              f" start offsets max {(start.max()-t0)/1e3:.1f} us; busy mean {busy.mean():.1f} min {busy.min():.1f} max {busy.max():.1f} us")
        print("   end deciles (us):", " ".join(f"{x:.1f}" for x in np.percentile((end - t0) / 1e3, [0, 10, 50, 90, 100])))
