#!/bin/bash
# one GPU session for the record: parity suite, full bench (ours + reference arm), launch list of
# one step, ncu --set full captures of K1 / K3 (headline and N=16K) exported to CSV on the box
# (raw metrics + per-SASS source counters) so only small files come back in gpurun_out/
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi > gpurun_out/nvidia-smi.txt
timeout 900 python -m pytest tests -q -m gpu --tb=short -o timeout=240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_gpt2.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
mkdir -p /tmp/ncu
for k in bwd fwd; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_${k}[12]?_kernel -s 3 -c 1 -o /tmp/ncu/prof_${k}_gpt2 \
      python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_${k}[12]?_kernel -s 1 -c 1 -o /tmp/ncu/prof_${k}_16k \
      python bench.py --workload long-16k --steps 1 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
done
for r in /tmp/ncu/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > gpurun_out/${b}_sass.csv 2>/dev/null
done
cp /tmp/ncu/prof_bwd_gpt2.ncu-rep gpurun_out/ 2>/dev/null
tail -2 gpurun_out/pytest_gpu.log
du -sh gpurun_out; ls gpurun_out
