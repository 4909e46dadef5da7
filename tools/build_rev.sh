#!/bin/bash
# Build the CUDA engine of a git revision into ab/<name>.so (same-box A/B runs:
# SCMWU_LIB=ab/<name>.so python tools/gen_perf.py ...).
#   tools/build_rev.sh <rev> <name> [extra nvcc flags]
set -e
rev=$1; name=$2; shift 2
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
git archive "$rev" paper_2405_09157_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$tmp/obj" ab
for f in "$tmp"/paper_2405_09157_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" -diag-suppress 177 \
       -gencode arch=compute_100a,code=sm_100a -c "$f" -o "$tmp/obj/$(basename "$f" .cu).o" &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "ab/$name.so" "$tmp"/obj/*.o -lcudart
rm -rf "$tmp"
echo "ab/$name.so"
