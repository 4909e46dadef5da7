#!/bin/bash
# ncu --set full of one 24-pass refine launch of the persistent kernel for the SVM north-star
# shape (n = 10^7, d = 100) and configs[1] (SES n = 10^6), final round-2 build
set -u
out=gpurun_out
mkdir -p $out
for wl in svm_c4 ses_c2; do
  if python tools/gpu_perf.py $wl --horizon 24 > $out/plain_$wl.log 2>&1; then
    timeout 1500 ncu --set full --import-source on --clock-control none -k regex:scmwu_kernel \
      -s 1 -c 1 -o $out/full_r02_$wl python tools/gpu_perf.py $wl --horizon 24 > $out/ncu_$wl.log 2>&1
  fi
done
ls -la $out
