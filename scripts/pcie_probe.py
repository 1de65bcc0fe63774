"""PCIe copy throughput probe (pinned host <-> device): single vs chunked vs multi-stream copies,
one direction and full duplex. Informs bench.py's e2e copy layout."""
import time

import torch

n = 50 * 2**20
s = [torch.cuda.Stream() for _ in range(4)]


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / it


hin = torch.empty(n, dtype=torch.uint8).pin_memory()
hout = torch.empty(n, dtype=torch.uint8).pin_memory()
din = torch.empty(n, dtype=torch.uint8, device="cuda")
dout = torch.empty(n, dtype=torch.uint8, device="cuda")


def copies(nin, nout, streams_in, streams_out):
    def fn():
        ci, co = n // nin, n // nout
        for i in range(nin):
            with torch.cuda.stream(s[i % streams_in]):
                din[i * ci:(i + 1) * ci].copy_(hin[i * ci:(i + 1) * ci], non_blocking=True)
        for i in range(nout):
            with torch.cuda.stream(s[2 + i % streams_out]):
                hout[i * co:(i + 1) * co].copy_(dout[i * co:(i + 1) * co], non_blocking=True)
    return fn


for name, args in [("in 1", (1, 0, 1, 1)), ("out 1", (0, 1, 1, 1)), ("duplex 1+1", (1, 1, 1, 1)),
                   ("duplex 2+2 one stream each", (2, 2, 1, 1)), ("duplex 2+2 two streams each", (2, 2, 2, 2)),
                   ("duplex 4+4 two streams each", (4, 4, 2, 2))]:
    nin, nout, si, so = args
    if nin == 0:
        fn = lambda: [torch.cuda.stream(s[2]).__enter__(), hout.copy_(dout, non_blocking=True)]
        with torch.cuda.stream(s[2]):
            dt = t(lambda: hout.copy_(dout, non_blocking=True))
    elif nout == 0:
        with torch.cuda.stream(s[0]):
            dt = t(lambda: din.copy_(hin, non_blocking=True))
    else:
        dt = t(copies(nin, nout, si, so))
    print(f"{name:32s} {dt * 1e3:.3f} ms per 50 MB each way ({n / dt / 1e9:.1f} GB/s per direction)")
