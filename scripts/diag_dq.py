import sys, math
import numpy as np, torch
sys.path.insert(0, ".")
from tests import gpu_helpers as G
from paper_2205_14135_b200 import attention as A
B,H,N,d = 1, 2, int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 128
dev, kept = G.make_device_inputs(B,H,N,d,"bf16",keep_heads=[(0,0)])
out = G.run_device(dev,"bf16",mask="causal")
rows = [0,1,2,3,127,128,1000,4095,8191,8192,12345,N-1]
q,k,v,do = (dev[n][0,0].double() for n in ("q","k","v","do"))
tau = 1/math.sqrt(d)
for i in rows:
    s = (q[i] @ k[:i+1].T) * tau
    p = torch.softmax(s, 0)
    dp = do[i] @ v[:i+1].T
    o = p @ v[:i+1]
    D_exact = (p*dp).sum()
    D_bf16o = (do[i] * out["o"][0,0,i].double()).sum()
    dq_ref = tau * ((p*(dp-D_exact)) @ k[:i+1])
    dq_ob = tau * ((p*(dp-D_bf16o)) @ k[:i+1])
    g = out["dq"][0,0,i].double()
    rel = lambda a,b: float((a-b).norm()/b.norm())
    print(f"row {i:6d} |dq|={float(dq_ref.norm()):.3e} gpu_rel={rel(g,dq_ref):.3e} refDfromO_rel={rel(dq_ob,dq_ref):.3e} gpu_vs_refDfromO={rel(g,dq_ob):.3e} |O err|={float((out['o'][0,0,i].double()-o).abs().max()):.2e} dD={float(D_bf16o-D_exact):.2e} lse_err={float(out['lse'][0,0,i].double()-torch.logsumexp(s,0)):.2e}")
