#!/bin/bash
# quick GPU iteration: parity suite, bench (no CPU baseline), bwd/fwd traces
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x --tb=short -o timeout=240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_ours.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], {k: (v["avg_launch_ms"], v["tflops"]) for k, v in d["kernels"].items()})
for s in d.get("sweep", []):
    print(f'{s["workload"]:>14} fwd {s["fwd_tflops"]:7.1f} bwd {s["bwd_tflops"]:7.1f}')
PY
[ -f paper_2205_14135_b200/lib/variants/lib_trace.so ] && timeout 120 python scripts/trace_${TRACE:-bwd}.py 2>&1 | grep -v Warn
