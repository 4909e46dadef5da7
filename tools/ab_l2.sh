# same-box A/B of L2 residency of part of X across passes (SCMWU_L2_KEEP_MB)
for rep in 1 2; do
 for mb in 0 25 40 55; do
  export SCMWU_L2_KEEP_MB=$mb
  echo "== keep $mb MB"
  python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
  python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v generate
 done
done
