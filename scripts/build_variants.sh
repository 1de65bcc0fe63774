#!/bin/bash
# Build tuning variants of the C-ABI library into paper_2205_14135_b200/lib/variants/ (experiments only).
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2205_14135_b200/lib/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $flags -shared \
    -o paper_2205_14135_b200/lib/variants/lib_$name.so paper_2205_14135_b200/csrc/tatn_capi.cu &
done
wait
ls paper_2205_14135_b200/lib/variants
