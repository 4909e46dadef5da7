#!/bin/bash
# Build an alternative libscmwu.so with extra nvcc defines into ab/<name>.so
# (A/B performance runs: SCMWU_LIB=ab/<name>.so python tools/gpu_perf.py ...)
#   tools/build_variant.sh timing -DSCMWU_PHASE_TIMING
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/$name ab
for f in paper_2405_09157_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" -diag-suppress 177 \
       -gencode arch=compute_100a,code=sm_100a -c $f -o build/$name/$(basename $f .cu).o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ab/$name.so build/$name/*.o -lcudart
echo ab/$name.so
