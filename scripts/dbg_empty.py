import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A
mode, d, B, H, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
q, k, v, do = (torch.randn(B, H, N, d, device="cuda").half() for _ in range(4))
if mode == "none":
    spec = A.AttnSpec(mask="none")
else:
    zero = mode == "pad0"
    vl = torch.tensor([0 if (zero and b % 7 == 0) else N - (b % 5) for b in range(B)], dtype=torch.int32, device="cuda")
    spec = A.AttnSpec(mask="key_padding", valid_len=vl)
try:
    o, lse = A.flash_fwd(q, k, v, spec); torch.cuda.synchronize()
    print(sys.argv[1:], "fwd ok", flush=True)
    A.flash_bwd(q, k, v, o, do, lse, spec); torch.cuda.synchronize()
    print(sys.argv[1:], "ok", flush=True)
except Exception as e:
    print(sys.argv[1:], "FAIL", repr(e)[:80], flush=True)
