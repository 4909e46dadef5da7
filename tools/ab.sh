#!/bin/bash
# Same-box A/B of per-pass throughput: tools/ab.sh <libA> <libB> (run on the GPU box)
A=$1; B=$2
for rep in 1 2; do
  for lib in $A $B; do
    echo "== $lib"
    SCMWU_LIB=$lib python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
    SCMWU_LIB=$lib python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  done
done
