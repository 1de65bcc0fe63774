"""Per-Q-tile event timeline (SM clocks) of CTA 0 of the backward kernel, -DTATN_TRACE build."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("TATN_B200_LIB", os.path.abspath("paper_2205_14135_b200/lib/variants/lib_trace.so"))
from paper_2205_14135_b200 import attention as A, _lib
lib = _lib.load()
names = ["S_seen", "P_arrive", "MMA_sawP", "front_s_issued", "dq_issued", "dQ_seen", "reduce|dsfree", "QFull_seen"]
for (B, H, N, d, mask) in [(8, 12, 1024, 64, "causal"), (1, 32, 4096, 128, "causal")]:
    q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    do = torch.randn_like(q)
    spec = A.AttnSpec(mask=mask)
    o, lse = A.flash_fwd(q, k, v, spec)
    for _ in range(3): A.flash_bwd(q, k, v, o, do, lse, spec)
    buf = torch.zeros(200000 * 16 + 9216 + 1024 * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    A.flash_bwd(q, k, v, o, do, lse, spec); torch.cuda.synchronize()
    lib.tatn_debug_set_trace(ctypes.c_void_p(0))
    evi = buf[200000 * 16 + 8192:200000 * 16 + 8192 + 1024].view(256, 4).cpu().numpy().astype(np.int64)
    ev = buf[200000 * 16:200000 * 16 + 8192].view(1024, 8).cpu().numpy().astype(np.int64)
    ev2 = buf[200000 * 16 + 9216:200000 * 16 + 9216 + 8192].view(1024, 8).cpu().numpy().astype(np.int64)
    n = int((ev[:, 1] > 0).sum())
    ev = ev[:n]
    ev2 = ev2[:n]
    t0 = ev[ev > 0].min()
    print(f"== B{B} H{H} N{N} d{d} {mask}: CTA0 tiles {n}, span {(ev.max() - t0)} cyc, per tile {(ev[:,1].max()-ev[:,0].min())/max(n-1,1):.0f} cyc")
    ni = int((evi[:, 0] > 0).sum())
    print("   items (claimed / KV-free / MMA took item / KV landed):")
    for n_ in range(ni):
        print(f"   item {n_}: " + " ".join(f"{(x - t0) if x > 0 else -1:9d}" for x in evi[n_]))
    print("   g  " + " ".join(f"{x:>9}" for x in names))
    for g in range(min(n, 40)):
        print(f"  {g:3d} " + " ".join(f"{(x - t0) if x > 0 else -1:9d}" for x in ev[g]))
    names2 = ["mma_iter", "mma_xfree", "mma_qfull+2", "sm_half0", "sm_dqempty", "mma_back", "sm_half1", "sm_xfree"]
    print("   g  " + " ".join(f"{x:>11}" for x in names2))
    for g in range(min(n, 40)):
        print(f"  {g:3d} " + " ".join(f"{(x - t0) if x > 0 else -1:11d}" for x in ev2[g]))
    s2 = ev2[4:n - 2]; s1 = ev[4:n - 2]
    if len(s2):
        m = lambda a: int(np.median(a))
        print(f"   MMA fronts (warp 13): front(g) waits XFree(g-2) {m(s2[:,1]-s2[:,0])}  ->QFull(g) {m(s2[:,2]-s2[:,1])}"
              f"  ->front_s(g) issued {m(s1[:,3]-s2[:,2])}  per front {m(np.diff(s1[:,3]))}")
        print(f"   MMA backs (warp 14): P->sawP {m(s1[:,2]-s1[:,1])}  sawP->back issued {m(s2[:,5]-s1[:,2])}  ->dQ issued {m(s1[:,4]-s2[:,5])}"
              f"  per back {m(np.diff(s1[:,2]))}")
        print(f"   softmax: S_seen->ld done {m(s1[:,6]-s1[:,0])}  ->half0 {m(s2[:,3]-s1[:,6])}  ->xfree arrive {m(s2[:,7]-s2[:,3])}"
              f"  ->dqempty {m(s2[:,4]-s2[:,7])}  ->half1 {m(s2[:,6]-s2[:,4])}  ->P {m(s1[:,1]-s2[:,6])}")
    sel = ev[4:n - 2]
    if len(sel):
        med = lambda a, b: int(np.median(sel[:, b] - sel[:, a]))
        print(f"   median: S_seen->P {med(0,1)}  P->MMA_sawP {med(1,2)}  MMA_sawP->dq_issued {med(2,4)}  dq_issued->dQ_seen {med(4,5)}  dQ_seen->reduce {med(5,6)}")
        nxt = sel[:, 0][2:] - sel[:, 1][:-2]
        print(f"   P(g) -> S_seen(g+2) median {int(np.median(nxt))}; front_s issued(g+2) - MMA_sawP(g) median {int(np.median(sel[2:,3]-sel[:-2,2]))}")
