#!/bin/bash
# global-mode tests with the in-tree library, then 1.3B / 7B step time: in-tree vs ab/* variants
mkdir -p gpurun_out
tag=${1:-g3}
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_global_big.py tests/test_gpu_lossless.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
for rep in 1 2; do
echo "== in-tree"; timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-60
for d in ab/*/; do echo "== $d"; MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-60; done
done
timeout 600 python tools/bench_global.py 6.738415616e9 2>&1 | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python tools/bench_global.py 1.3e9 > /dev/null 2>&1
