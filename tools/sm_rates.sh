#!/bin/bash
# per-CTA streaming cycles and SM ids with the equal partition (timing build), for
# checking whether per-SM streaming rates are a stable property across boxes
tag=$1
nvidia-smi --query-gpu=uuid --format=csv,noheader > gpurun_out/uuid_$tag.txt
for wl in svm_c3 ses_c2; do
  SCMWU_LIB=ab/timing.so SCMWU_TIMING=1 SCMWU_DUMP=gpurun_out/rates_${tag}_$wl.json \
    python tools/gpu_perf.py $wl --horizon 512 > gpurun_out/rates_${tag}_$wl.log 2>&1
done
cat gpurun_out/uuid_$tag.txt
