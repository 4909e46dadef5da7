#!/bin/bash
# round-end measurement set (GPU box): C2 profile set, C3 bench, generated C4/C5 benches
set -u
bash tools/profile_round.sh ${TAG:-r01e} ses_c2 --steps 3 --warmup 3 > gpurun_out/round_c2.log 2>&1
python bench.py --workload svm_c3 --steps 1 --warmup 3 > gpurun_out/bench_${TAG:-r01e}_svm_c3.json 2> gpurun_out/bench_${TAG:-r01e}_svm_c3.err
python bench.py --workload svm_c5_gen --steps 3 --warmup 3 > gpurun_out/bench_${TAG:-r01e}_svm_c5_gen.json 2> gpurun_out/bench_${TAG:-r01e}_svm_c5_gen.err
python bench.py --workload ses_c4_gen --steps 1 --warmup 3 > gpurun_out/bench_${TAG:-r01e}_ses_c4_gen.json 2> gpurun_out/bench_${TAG:-r01e}_ses_c4_gen.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scmwu_kernel -s 1 -c 1 -o gpurun_out/full_${TAG:-r01e}_svm_c3 python tools/gen_perf.py svm 500000 100 --horizon 64 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scmwu_kernel -s 1 -c 1 -o gpurun_out/full_${TAG:-r01e}_svm_c5 python tools/gen_perf.py svm 1000000 512 --horizon 16 --reps 1 > /dev/null 2>&1
ls -la gpurun_out | grep ${TAG:-r01e}
