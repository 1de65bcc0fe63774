"""A/B forward timing of the product library vs variants on d=128 workloads, interleaved runs."""
import os, subprocess, sys, json
libs = ["product"] + sys.argv[1:]
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
import bench
from paper_2205_14135_b200 import attention as A
res = {}
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = lambda: flush_buf.zero_()
for name in ["long-2k", "long-4k", "long-8k", "long-16k", "long-4k-noncausal"]:
    w = bench.WORKLOADS[name]
    q, k, v, do, spec = bench.make_inputs(w, torch.device("cuda"))
    st = bench.Step(q, k, v, do, spec)
    ms = sorted(bench.timed(bench.graphed(st.fwd), 20, flush))[10]
    res[name] = round(bench.flops(w)[0] / ms / 1e9, 1)
    del q, k, v, do, st
    torch.cuda.empty_cache()
print(json.dumps(res))
'''
for rep in range(2):
    for lib in libs:
        env = dict(os.environ)
        if lib != "product":
            env["TATN_B200_LIB"] = os.path.abspath(f"paper_2205_14135_b200/lib/variants/lib_{lib}.so")
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(lib, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:], flush=True)
