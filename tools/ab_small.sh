# same-box A/B on the sync-bound configs[0] (SES n=1e4, d=10) and C2: tools/ab_small.sh libA libB
for rep in 1 2; do for lib in "$@"; do echo "== $lib rep $rep"
  SCMWU_LIB=ab/$lib.so python tools/gpu_perf.py ses_c1 --horizon 4096 2>&1 | grep "refine h" | tail -2
  SCMWU_LIB=ab/$lib.so python bench.py --workload ses_c1 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 solve', round(d['value'],4), d['config']['iterations'], round(d['roofline']['us_per_pass'],2))"
done; done
