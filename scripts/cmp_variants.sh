#!/bin/bash
# bench sweep for the product library and each variant in lib/variants given as args
mkdir -p gpurun_out
for v in product "$@"; do
  if [ "$v" = product ]; then unset TATN_B200_LIB; else export TATN_B200_LIB=$PWD/paper_2205_14135_b200/lib/variants/lib_$v.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cmp_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/cmp_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(f"## {sys.argv[1]}: value {d['value']} ms {d['ms_per_step']} fwd {d['kernels']['fwd_K1']['tflops']} bwd {d['kernels']['bwd_K3']['tflops']}")
print("   " + " | ".join(f"{s['workload']} {s['fwd_tflops']:.0f}/{s['bwd_tflops']:.0f}" for s in d.get("sweep", []) if "fwd_tflops" in s))
PY
done
