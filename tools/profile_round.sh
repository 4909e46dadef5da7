#!/bin/bash
# Round profiling on the GPU box (one GPU): bench line, launch list, one full ncu capture
# of the persistent kernel, summaries into gpurun_out/.  Usage:
#   tools/profile_round.sh <tag> <workload> [bench args...]
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
tag=$1; wl=$2; shift 2
out=gpurun_out
mkdir -p $out
if ! python bench.py --workload "$wl" "$@" > $out/bench_${tag}_${wl}.json 2> $out/bench_${tag}_${wl}.err; then
  echo "bench failed"; tail -5 $out/bench_${tag}_${wl}.err; exit 1
fi
cat $out/bench_${tag}_${wl}.json
# launch list (cold-cache, serialised: shares, not absolutes)
if python bench.py --workload "$wl" --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_${tag}_${wl}.csv \
    python bench.py --workload "$wl" --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  # one full capture of a persistent-kernel launch (a mid-solve sc_ftp call)
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:scmwu_kernel \
    -s 20 -c 1 -o $out/full_${tag}_${wl} \
    python bench.py --workload "$wl" --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_${tag}_${wl}.log 2>&1
fi
ls -la $out | grep "$tag"
