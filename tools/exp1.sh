set -x
python tools/gen_perf.py ses 1000000 100 --horizon 1024
python tools/gen_perf.py ses 10000000 100 --horizon 128
SCMWU_CFG=8,13,2 python tools/gen_perf.py ses 10000000 100 --horizon 128
SCMWU_CFG=8,13,2 python tools/gen_perf.py ses 1000000 100 --horizon 1024
python tools/gen_perf.py svm 500000 100 --horizon 1024
SCMWU_CFG=8,13,2 python tools/gen_perf.py svm 500000 100 --horizon 1024
python tools/gen_perf.py svm 10000000 512 --horizon 48
SCMWU_CFG=32,16,1 python tools/gen_perf.py svm 10000000 512 --horizon 48
SCMWU_CFG=16,32,2 python tools/gen_perf.py svm 10000000 512 --horizon 48
