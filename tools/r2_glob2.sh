#!/bin/bash
mkdir -p gpurun_out
tag=${1:-gb}
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_global_big.py tests/test_gpu_lossless.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
timeout 600 python tools/bench_global.py 1.3e9 6.738415616e9 > gpurun_out/${tag}_on.log 2>&1; cat gpurun_out/${tag}_on.log
MA_GLOBAL_BRACKET=0 MA_GLOBAL_FUSED_EMIT=0 timeout 600 python tools/bench_global.py 1.3e9 > gpurun_out/${tag}_off.log 2>&1; cat gpurun_out/${tag}_off.log
GRAD_STREAM=heavy timeout 600 python tools/bench_global.py 1.3e9 > gpurun_out/${tag}_heavy.log 2>&1; cat gpurun_out/${tag}_heavy.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python tools/bench_global.py 1.3e9 > /dev/null 2>&1
