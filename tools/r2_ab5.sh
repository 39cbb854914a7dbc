#!/bin/bash
# lean + global parity tests on the in-tree build; 7B lean step and 1.3B / 7B global step,
# in-tree vs ab/* (alternating)
mkdir -p gpurun_out
tag=${1:-ab5}
timeout 1500 python -m pytest tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_global.py tests/test_gpu_global_big.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
for rep in 1 2 3; do
echo "== in-tree $(SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"
for d in ab/*/; do echo "== $d $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"; done
done
for rep in 1 2; do
echo "== global in-tree $(timeout 300 python tools/bench_global.py 1.3e9 2>&1 | tail -1)"
echo "== global ab/base $(MA_LIB_PATH=$PWD/ab/base/libmicroadam_cuda.so timeout 300 python tools/bench_global.py 1.3e9 2>&1 | tail -1)"
done
echo "== global in-tree 7B $(timeout 300 python tools/bench_global.py 6.738415616e9 2>&1 | tail -1)"
