#!/bin/bash
# lean parity tests on the in-tree build, then the 7B step time of in-tree vs every ab/* variant
# (alternating, 3 reps; the median of steps 7..16 of each run)
mkdir -p gpurun_out
tag=${1:-ab3}
timeout 1500 python -m pytest tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
for rep in 1 2 3; do
echo "== in-tree $(SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"
for d in ab/*/; do echo "== $d $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"; done
done
