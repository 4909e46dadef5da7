# same-box A/B of engine builds: tools/ab_runs.sh libA libB ... (ab/<name>.so)
for rep in 1 2; do
for lib in "$@"; do
  echo "== $lib rep $rep"
  SCMWU_LIB=ab/$lib.so python tools/gen_perf.py ses 10000000 100 --horizon 256 --reps 2 2>&1 | grep -v "^generate"
  SCMWU_LIB=ab/$lib.so python tools/gen_perf.py ses 1000000 100 --horizon 1024 --reps 2 2>&1 | grep -v "^generate"
  SCMWU_LIB=ab/$lib.so python tools/gen_perf.py svm 5000000 100 --horizon 256 --reps 2 2>&1 | grep -v "^generate"
  SCMWU_LIB=ab/$lib.so python tools/gen_perf.py svm 500000 100 --horizon 1024 --reps 2 2>&1 | grep -v "^generate"
done; done
