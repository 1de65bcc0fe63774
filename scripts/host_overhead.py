import sys, time, torch
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A
q, k, v, do = (torch.randn(8, 12, 1024, 64, device="cuda").half() for _ in range(4))
spec = A.AttnSpec(mask="causal")
o = torch.empty_like(q); lse = torch.empty(8, 12, 1024, device="cuda"); ws = A.bwd_workspace(q, k, v, spec); fws = A.fwd_workspace(q.device)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for _ in range(5):
    A.flash_fwd(q, k, v, spec, out=o, lse=lse, workspace=fws); A.flash_bwd(q, k, v, o, do, lse, spec, dq, dk, dv, ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    A.flash_fwd(q, k, v, spec, out=o, lse=lse, workspace=fws)
t1 = time.perf_counter()
for _ in range(200):
    A.flash_bwd(q, k, v, o, do, lse, spec, dq, dk, dv, ws)
t2 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per flash_fwd call {1e6*(t1-t0)/200:.1f} us, per flash_bwd call {1e6*(t2-t1)/200:.1f} us")
