#!/bin/bash
# One GPU session for the record (TAG = run name, e.g. r02o): parity suite, full bench (ours +
# reference arm), launch list of one headline step, ncu --set full captures of K1 / K3 (headline
# and N = 16K, d = 128) and of the tf32 check-mode kernels at C1, exported to CSV on the box (raw
# metrics + per-SASS source counters) so only small files come back in gpurun_out/.
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nproc > $O/nproc.txt
nvidia-smi > $O/nvidia-smi.txt
timeout 1500 python -m pytest tests -q -m gpu --tb=short -o timeout=900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
./paper_2205_14135_b200/dropin/build/dropin_check > $O/dropin_check.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_ours.json 2> $O/bench_ours.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_gpt2.csv \
    python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
mkdir -p /tmp/ncu
for k in bwd fwd; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_${k}[12]?_kernel -s 3 -c 1 -o /tmp/ncu/prof_${k}_gpt2 \
      python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tatn_${k}[12]?_kernel -s 1 -c 1 -o /tmp/ncu/prof_${k}_16k \
      python bench.py --workload long-16k --steps 1 --warmup 3 --no-sweep --no-cpu-baseline --no-graph > /dev/null 2>&1
done
# tf32 check mode at C1 (B=2 H=4 N=512 d=64 fp32)
cat > /tmp/c1_fp32.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2205_14135_b200 import attention as A
q, k, v, do = (torch.randn(2, 4, 512, 64, device="cuda") for _ in range(4))
for _ in range(3):
    o, lse = A.flash_fwd(q, k, v)
    A.flash_bwd(q, k, v, o, do, lse)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:tf32 -s 2 -c 2 -o /tmp/ncu/prof_tf32_c1 python /tmp/c1_fp32.py > /dev/null 2>&1
for r in /tmp/ncu/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > $O/${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $O/${b}_sass.csv 2>/dev/null
done
tail -2 $O/pytest_gpu.log
du -sh $O; ls $O
