import torch, time
n = 50 * 2**20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(it): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / it
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
a = t(h2d); b = t(d2h); c = t(both)
print(f"H2D {n/a/1e9:.1f} GB/s  D2H {n/b/1e9:.1f} GB/s  both: {n/c/1e9:.1f} GB/s each ({c*1e3:.3f} ms per 50MB pair)")
# chunked 4 x 12.5MB
hs = [torch.empty(n//4, dtype=torch.uint8).pin_memory() for _ in range(4)]
ds = [torch.empty(n//4, dtype=torch.uint8, device="cuda") for _ in range(4)]
def h2d4():
    with torch.cuda.stream(s1):
        for h, d in zip(hs, ds): d.copy_(h, non_blocking=True)
print(f"H2D 4x12.5MB {n/t(h2d4)/1e9:.1f} GB/s")
big_h = torch.empty(n, dtype=torch.uint8).pin_memory(); big_d = torch.empty(n, dtype=torch.uint8, device="cuda")
views_h = big_h.view(4, -1); views_d = big_d.view(4, -1)
def h2d4v():
    with torch.cuda.stream(s1):
        for i in range(4): views_d[i].copy_(views_h[i], non_blocking=True)
print(f"H2D 4 views of one pinned buffer {n/t(h2d4v)/1e9:.1f} GB/s")
def h2d1c():
    with torch.cuda.stream(s1): ds[0].copy_(hs[0], non_blocking=True)
print(f"H2D 1x12.5MB {n/4/t(h2d1c)/1e9:.1f} GB/s")
hf = [torch.empty((n // 8,), dtype=torch.float16).pin_memory() for _ in range(4)]
dfl = [torch.empty((n // 8,), dtype=torch.float16, device="cuda") for _ in range(4)]
def h2d4f():
    with torch.cuda.stream(s1):
        for h, d in zip(hf, dfl): d.copy_(h, non_blocking=True)
print(f"H2D 4x12.5MB fp16 tensors {n/t(h2d4f)/1e9:.1f} GB/s")
