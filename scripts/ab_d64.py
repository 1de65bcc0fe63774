"""A/B forward+backward timing (variants: lib/variants/lib_NAME.so, or VAR=VALUE env settings) (graph replays, L2 flushed) of the product library vs variants on
the d=64 workloads, interleaved subprocess runs: python scripts/ab_d64.py VARIANT... [REPS]."""
import os, subprocess, sys
args = [a for a in sys.argv[1:] if not a.isdigit()]
reps = int(next((a for a in sys.argv[1:] if a.isdigit()), "3"))
libs = ["product"] + args
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
import bench
res = {}
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = lambda: flush_buf.zero_()
import os
for name in os.environ.get("AB_WORKLOADS", "gpt2-small,bert-large,long-8k-d64,butterfly-16k").split(","):
    w = bench.WORKLOADS[name]
    q, k, v, do, spec = bench.make_inputs(w, torch.device("cuda"))
    st = bench.Step(q, k, v, do, spec)
    f = bench.flops(w)
    fw = sorted(bench.timed(bench.graphed(st.fwd), 21, flush))[10]  # median
    bw = sorted(bench.timed(bench.graphed(st.bwd), 21, flush))[10]
    res[name] = (round(f[0] / fw / 1e9), round(f[1] / bw / 1e9))
    del q, k, v, do, st
    torch.cuda.empty_cache()
print(json.dumps(res))
'''
for rep in range(reps):
    for lib in libs:
        env = dict(os.environ)
        if "=" in lib:  # product library with an environment setting, e.g. TATN_PDL=0
            k_, v_ = lib.split("=", 1)
            env[k_] = v_
        elif lib != "product":
            env["TATN_B200_LIB"] = os.path.abspath(f"paper_2205_14135_b200/lib/variants/lib_{lib}.so")
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{lib:>10}", out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:], flush=True)
