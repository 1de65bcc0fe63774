#!/bin/bash
# one GPU session: bench (ours + reference arm), launch list, ncu full captures of K1 / K3
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi > gpurun_out/nvidia-smi.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_gpt2.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_bwd_kernel -s 3 -c 1 -o gpurun_out/prof_bwd_gpt2 \
    python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_fwd_kernel -s 3 -c 1 -o gpurun_out/prof_fwd_gpt2 \
    python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd_16k \
    python bench.py --workload long-16k --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_bwd16k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd_16k \
    python bench.py --workload long-16k --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_fwd16k.log 2>&1
ls -la gpurun_out
