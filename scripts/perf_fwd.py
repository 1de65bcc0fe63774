"""Forward/backward timing sweep for one library build (TATN_B200_LIB selects the variant)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A
name = os.environ.get("TATN_B200_LIB", "default").split("/")[-1]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cfgs = [(8,12,1024,64,"causal"),(4,32,4096,128,"causal"),(4,32,4096,128,"none"),(1,32,16384,128,"causal"),(2,32,8192,64,"none")]
do_bwd = "--bwd" in sys.argv
for (B,H,N,d,mask) in cfgs:
    q = torch.randn(B,H,N,d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q); do = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    o, lse = A.flash_fwd(q,k,v,spec)
    fn = (lambda: A.flash_bwd(q,k,v,o,do,lse,spec)) if do_bwd else (lambda: A.flash_fwd(q,k,v,spec,out=o,lse=lse))
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(10):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); tot += a.elapsed_time(b)
    ms = tot / 10
    pairs = N*(N+1)/2 if mask=="causal" else N*N
    tf = (10 if do_bwd else 4)*d*pairs*B*H/ms/1e9
    print(f"{name} {'bwd' if do_bwd else 'fwd'} B{B} H{H} N{N} d{d} {mask}: {ms:.3f} ms {tf:.1f} TFLOP/s", flush=True)
