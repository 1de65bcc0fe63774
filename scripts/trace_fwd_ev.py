"""Per-tile event timeline (SM clocks) of CTA 0 of the d=64 forward kernel, -DTATN_TRACE build."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
names = ["S_seen", "S_free", "P_arrive", "MMA_sawP", "QKnext_iss", "item_seen", "OFinal", "O_staged"]
for (B, H, N, d, mask) in [(8, 12, 1024, 64, "causal"), (2, 32, 8192, 64, "none")]:
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    for _ in range(3): A.flash_fwd(q, k, v, spec)
    buf = torch.zeros(200000 * 16 + 1024 * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    A.flash_fwd(q, k, v, spec); torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    ev = buf[200000 * 16:].view(1024, 8).cpu().numpy().astype(np.int64)[:, :8]
    n = int((ev[:, 2] > 0).sum())
    ev = ev[:n]
    t0 = ev[ev > 0].min()
    print(f"== B{B} H{H} N{N} d{d} {mask}: CTA0 tiles {n}")
    print("   t  " + " ".join(f"{x:>11}" for x in names))
    for g in range(min(n, 24)):
        print(f"  {g:3d} " + " ".join(f"{(x - t0) if x > 0 else -1:11d}" for x in ev[g]))
    if n > 6:
        s = ev[2:n - 1]
        med = lambda a, b: int(np.median(s[:, b] - s[:, a]))
        print(f"   median: S_seen->S_free {med(0,1)} S_free->P {med(1,2)} P->MMA_sawP {med(2,3)} per-tile {int(np.median(np.diff(ev[1:n,0])))}")
