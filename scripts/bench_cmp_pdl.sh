for r in 1 2; do
for v in product pdl0 noearly; do
  if [ $v = pdl0 ]; then export TATN_PDL=0; unset TATN_B200_LIB; elif [ $v = noearly ]; then unset TATN_PDL; export TATN_B200_LIB=$PWD/paper_2205_14135_b200/lib/variants/lib_noearly.so; else unset TATN_PDL TATN_B200_LIB; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['kernels']['fwd_K1']['tflops'], d['kernels']['bwd_K3']['tflops'])"
done; done
