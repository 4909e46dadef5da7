#!/bin/bash
# Round-2 profiling of the default workload (configs[3], SES n=10^7 d=100) on one GPU:
#  1. launch list of one bench step (ncu, duration only: cold-cache, serialised);
#  2. one --set full capture of a 24-pass refine launch of the persistent kernel.
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
out=gpurun_out
mkdir -p $out
if python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/plain_bench.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_r02_ses_c4.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
fi
if python tools/gpu_perf.py ses_c4 --horizon 24 > $out/plain_perf.log 2>&1; then
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:scmwu_kernel \
    -s 1 -c 1 -o $out/full_r02_ses_c4 \
    python tools/gpu_perf.py ses_c4 --horizon 24 > $out/ncu_r02_ses_c4.log 2>&1
fi
ls -la $out
