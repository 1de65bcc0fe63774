"""CTA start / end spread of the persistent forward kernels (-DTATN_TRACE build, global timer ns)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
for (B, H, N, d, mask) in [(8, 12, 1024, 64, "causal"), (16, 16, 512, 64, "none"), (2, 32, 8192, 64, "none"),
                           (1, 32, 16384, 128, "causal")]:
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    for _ in range(3): A.flash_fwd(q, k, v, spec)
    buf = torch.zeros(200000 * 16 + 1024 * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); A.flash_fwd(q, k, v, spec); e1.record(); torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    t = buf[:200000 * 16].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    if len(t) == 0:
        print(f"== B{B} H{H} N{N} d{d} {mask}: no CTA trace (kernel without TATN_TRACE_AT)")
        continue
    st, en = t[:, 0], t[:, 7]
    t0 = st.min()
    rel = lambda x: (x - t0) / 1000.0
    print(f"== B{B} H{H} N{N} d{d} {mask}: {len(t)} CTAs; event time {e0.elapsed_time(e1)*1000:.1f} us; "
          f"start spread {rel(st.max()):.2f} us; end min/median/max {rel(en.min()):.1f}/{rel(np.median(en)):.1f}/{rel(en.max()):.1f} us")
    print("   end-time deciles:", " ".join(f"{x:.1f}" for x in np.percentile(rel(en), [10, 30, 50, 70, 90, 99])))
