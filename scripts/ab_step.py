"""A/B of the whole step (forward + backward captured in ONE graph, so programmatic launches
between K1 and K2 take effect; L2 flushed between replays): product library vs variants
(lib/variants/lib_NAME.so, or VAR=VALUE env settings), interleaved subprocess runs:
python scripts/ab_step.py VARIANT... [REPS]. Prints step TFLOP/s (median of 21) per workload."""
import os, subprocess, sys
args = [a for a in sys.argv[1:] if not a.isdigit()]
reps = int(next((a for a in sys.argv[1:] if a.isdigit()), "3"))
libs = ["product"] + args
code = r'''
import sys, os, torch, json
sys.path.insert(0, ".")
import bench
res = {}
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = lambda: flush_buf.zero_()
for name in os.environ.get("AB_WORKLOADS", "gpt2-small,bert-large,long-4k,butterfly-16k").split(","):
    w = bench.WORKLOADS[name]
    q, k, v, do, spec = bench.make_inputs(w, torch.device("cuda"))
    st = bench.Step(q, k, v, do, spec)
    f = bench.flops(w)
    t = sorted(bench.timed(bench.graphed(st), 21, flush))[10]
    res[name] = round((f[0] + f[1]) / t / 1e9, 1)
    del q, k, v, do, st
    torch.cuda.empty_cache()
print(json.dumps(res))
'''
for rep in range(reps):
    for lib in libs:
        env = dict(os.environ)
        if "=" in lib:
            k_, v_ = lib.split("=", 1)
            env[k_] = v_
        elif lib != "product":
            env["TATN_B200_LIB"] = os.path.abspath(f"paper_2205_14135_b200/lib/variants/lib_{lib}.so")
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{lib:>10}", out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:], flush=True)
