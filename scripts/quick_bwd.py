"""First-light GPU check of the backward kernels against torch fp32 autograd."""
import math, sys
import torch
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A

def ref(q, k, v, do, tau, mask, valid_len=None):
    qf, kf, vf = [t.float().detach().requires_grad_() for t in (q, k, v)]
    s = torch.einsum("bhqd,bhkd->bhqk", qf, kf) * tau
    Nq, Nk = q.shape[2], k.shape[2]
    if mask == "causal":
        i = torch.arange(Nq, device=q.device)[:, None]; j = torch.arange(Nk, device=q.device)[None, :]
        s = s.masked_fill(j > i, float("-inf"))
    if mask == "key_padding":
        j = torch.arange(Nk, device=q.device)
        m = j[None, :] >= valid_len[:, None].long()
        s = s.masked_fill(m[:, None, None, :], float("-inf"))
    p = torch.softmax(s, -1).nan_to_num(0.0)
    o = torch.einsum("bhqk,bhkd->bhqd", p, vf)
    o.backward(do.float())
    return qf.grad, kf.grad, vf.grad

torch.manual_seed(0)
ok = True
for (B, H, N, d, dt, mask) in [(1,1,128,64,torch.bfloat16,"none"), (1,1,64,128,torch.bfloat16,"none"),
                               (1,1,256,128,torch.bfloat16,"none"), (2,3,512,64,torch.bfloat16,"none"),
                               (2,2,384,128,torch.bfloat16,"none"), (2,2,1000,128,torch.float16,"causal"),
                               (2,2,777,64,torch.bfloat16,"causal"), (4,2,512,64,torch.bfloat16,"key_padding"),
                               (1,2,2048,128,torch.bfloat16,"causal")]:
    q = torch.randn(B,H,N,d, device="cuda", dtype=dt); k = torch.randn_like(q); v = torch.randn_like(q)
    do = torch.randn_like(q)
    vl = torch.randint(N-20, N+1, (B,), device="cuda", dtype=torch.int32) if mask == "key_padding" else None
    spec = A.AttnSpec(mask=mask, valid_len=vl)
    try:
        o, lse = A.flash_fwd(q, k, v, spec)
        dq, dk, dv = A.flash_bwd(q, k, v, o, do, lse, spec)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAIL launch", B,H,N,d,dt,mask, repr(e)); ok = False; continue
    rq, rk, rv = ref(q, k, v, do, 1/math.sqrt(d), mask, vl)
    msg = []
    good = True
    for name, a, r in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        e = (a.float()-r).abs().max().item(); rel = ((a.float()-r).norm()/r.norm().clamp_min(1e-30)).item()
        good &= (e < 2e-2 or rel < 1e-2) and rel < 1e-2
        msg.append(f"{name} max={e:.2e} rel={rel:.2e}")
    ok &= good
    print(("OK  " if good else "BAD ") + f"B{B} H{H} N{N} d{d} {dt} {mask}: " + "  ".join(msg), flush=True)

for (B,H,N,d,mask) in [(16,16,512,64,"none"),(8,12,1024,64,"causal"),(4,32,4096,128,"causal"),(4,32,4096,128,"none"),(1,32,16384,128,"causal"),(2,16,8192,64,"none")]:
    q = torch.randn(B,H,N,d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q); do = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    o, lse = A.flash_fwd(q,k,v,spec)
    ws = A.bwd_workspace(q,k,v,spec)
    dq = torch.empty_like(q); dk = torch.empty_like(q); dv = torch.empty_like(q)
    for _ in range(3): A.flash_bwd(q,k,v,o,do,lse,spec,dq,dk,dv,ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it): A.flash_bwd(q,k,v,o,do,lse,spec,dq,dk,dv,ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/it
    pairs = N*(N+1)/2 if mask=="causal" else N*N
    tf = 10*d*pairs*B*H/ms/1e9
    print(f"TIME bwd B{B} H{H} N{N} d{d} {mask}: {ms:.3f} ms  {tf:.1f} TFLOP/s", flush=True)
print("ALLOK" if ok else "SOMEFAIL")
