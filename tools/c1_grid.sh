set -u
for g in 148 74 48 37 24 16 8; do
  echo "grid $g"; python tools/gpu_perf.py ses_c1 --grid $g --horizon 4096 2>&1 | grep refine | tail -2
done
