#!/bin/bash
mkdir -p gpurun_out
tag=${1:-g4}
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_global_big.py tests/test_gpu_lossless.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -15 gpurun_out/${tag}_tests.log
for rep in 1 2; do
echo "== fp32 $(timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-50)"
echo "== fp64 $(MA_GLOBAL_RQ_FP32=0 timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-50)"
done
timeout 600 python tools/bench_global.py 6.738415616e9 2>&1 | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:g_stats -c 30 --csv --log-file gpurun_out/${tag}_launches.csv python tools/bench_global.py 1.3e9 > /dev/null 2>&1
