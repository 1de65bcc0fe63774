"""Per-step SM-clock stamps of CTA (0,0,0) of the tf32 check-mode forward (-DTATN_TRACE build)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
q, k, v = (torch.randn(2, 4, 512, 64, device="cuda") for _ in range(3))
for _ in range(3): A.flash_fwd(q, k, v)
buf = torch.zeros(200000 * 16 + 1024 * 8 + 1024, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
torch.cuda.synchronize()
A.flash_fwd(q, k, v); torch.cuda.synchronize()
lib.tatn_debug_set_trace(ctypes.c_void_p(0))
ev = buf[200000 * 16:200000 * 16 + 8192].view(1024, 8).cpu().numpy().astype(np.int64)
t0 = ev[0, 7]
print("start->griddep", ev[0, 5] - t0, "->Q landed", ev[0, 6] - t0)
for n in range(4):
    print(f"step {n}: K landed {ev[n,1]-t0}  S ready {ev[n,2]-t0}  softmax done {ev[n,3]-t0}  PV done {ev[n,4]-t0}")
