#!/bin/bash
# lean-kernel parity tests, then the configs[4] sweep points at 1.3B: in-tree build vs ab/* variants
mkdir -p gpurun_out
tag=${1:-sw}
timeout 1200 python -m pytest tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_scale.py tests/test_gpu_golden.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
P="0.01:10 0.02:10 0.05:10 0.01:20 0.01:5"
for rep in 1 2; do
echo "== in-tree"; timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-80
for d in ab/*/; do echo "== $d"; MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-80; done
done
