# same-box A/B of the grid-reduction scheme (SCMWU_FOLD=0 two barriers, 1 redundant fold)
for rep in 1 2; do
 for mode in 0 1; do
  export SCMWU_FOLD=$mode
  echo "== fold $mode"
  python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  python tools/gen_perf.py ses 10000 10 --horizon 8192 --reps 2 --dist gaussian 2>&1 | grep -v generate
 done
done
export SCMWU_FOLD=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
