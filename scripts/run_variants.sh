#!/bin/bash
# time every variant in lib/variants with scripts/perf_fwd.py (args passed through)
for f in paper_2205_14135_b200/lib/variants/*.so; do
  TATN_B200_LIB=$PWD/$f timeout 120 python scripts/perf_fwd.py "$@" 2>&1 | grep -v Warning
done
