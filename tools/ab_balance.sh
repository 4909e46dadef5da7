# same-box A/B of the calibrated per-SM partition (SCMWU_BALANCE=0 vs default)
for rep in 1 2; do
 for mode in 0 1; do
  export SCMWU_BALANCE=$mode
  echo "== balance $mode"
  python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
 done
done
unset SCMWU_BALANCE
python tools/gen_perf.py svm 1000000 512 --horizon 256 --reps 2 2>&1 | grep -v generate
python tools/gen_perf.py ses 10000000 100 --horizon 128 --reps 2 2>&1 | grep -v generate
SCMWU_TIMING=1 SCMWU_LIB=ab/timing.so python tools/gpu_perf.py ses_c2 --horizon 576 2>&1 | tail -7
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
