#!/bin/bash
# GPU session: parity suite, drop-in acceptance, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --tb=short -o timeout=240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 paper_2205_14135_b200/dropin/build/dropin_check > gpurun_out/dropin_check.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/dropin_check.log
