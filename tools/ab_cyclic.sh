for rep in 1 2; do
 for mode in contig cyclic; do
  if [ $mode = contig ]; then export SCMWU_CONTIG=1; else unset SCMWU_CONTIG; fi
  echo "== $mode"
  python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
 done
done
unset SCMWU_CONTIG
SCMWU_TIMING=1 SCMWU_LIB=ab/timing.so python tools/gpu_perf.py ses_c2 --horizon 576 2>&1 | tail -7
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
