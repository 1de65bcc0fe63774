"""Per-CTA timeline of the forward kernel from a -DTATN_TRACE build (lib/variants/lib_trace.so)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ["TATN_B200_LIB"] = os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so")
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
for (B,H,N,d,mask) in [(8,12,1024,64,"causal"), (16,16,512,64,"key_padding"), (1,32,4096,128,"causal")]:
    q = torch.randn(B,H,N,d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    if mask == "key_padding":
        spec.valid_len = torch.full((B,), N - 7, dtype=torch.int32, device="cuda")
    for _ in range(3): A.flash_fwd(q,k,v,spec)
    buf = torch.zeros(200000*16, dtype=torch.int64, device="cuda")
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    A.flash_fwd(q,k,v,spec); torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    t = buf.view(-1, 16).cpu().numpy()
    t = t[t[:,0] > 0]
    t0 = t[:,0].min()
    start, first_s, last_p, ofinal, end, sm, steps, qld = (t[:,i] for i in range(8))
    s8, s9, s10, m11, m12, s13 = (t[:,i] for i in range(8, 14))
    ok3 = steps >= 4
    seg = lambda a, b: ((b[ok3] - a[ok3]) / 1000.0).mean()
    print(f"   step 2 (us): S got -> max done {seg(s8, s9):.3f}; max -> P signalled {seg(s9, s10):.3f}; "
          f"P signalled -> MMA sees P {seg(s10, m11):.3f}; MMA sees P -> next QK issued {seg(m11, m12):.3f}; "
          f"QK issued -> softmax has S {seg(m12, s13):.3f}; total {seg(s8, s13):.3f}")
    rel = lambda x: (x - t0) / 1000.0
    dur = (end - start) / 1000.0
    print(f"== B{B} H{H} N{N} d{d} {mask}: {len(t)} CTAs, kernel span {rel(end.max()):.1f} us")
    print(f"   CTA duration us: mean {dur.mean():.2f} min {dur.min():.2f} max {dur.max():.2f}")
    print(f"   start->Q landed us: mean {((qld-start)/1000).mean():.2f}; start->first S: {((first_s-start)/1000).mean():.2f}")
    ok = steps > 0
    per_step = (last_p[ok] - first_s[ok]) / np.maximum(steps[ok] - 1, 1) / 1000
    print(f"   steps mean {steps.mean():.1f}; per-step (first S..last P)/(n-1) us: mean {per_step[steps[ok]>1].mean():.3f}")
    print(f"   last P -> O final us: {((ofinal[ok]-last_p[ok])/1000).mean():.2f}; O final -> end us: {((end-ofinal)/1000).mean():.2f}")
    # SM occupancy timeline: CTAs concurrently resident per SM
    for s_ in sorted(set(sm.tolist()))[:2]:
        m = sm == s_
        order = np.argsort(start[m])
        print(f"   SM {s_}: " + ", ".join(f"[{rel(a):.1f},{rel(b):.1f}]x{c}" for a, b, c in zip(start[m][order], end[m][order], steps[m][order])))
