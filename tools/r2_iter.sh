#!/bin/bash
# One build -> measure iteration on the GPU box: lean-path GPU tests with the
# in-tree library, then a same-box A/B of every ab/*/ variant (7B, fresh
# gradient each step, median of the steady steps).
mkdir -p gpurun_out
tag=${1:-it}
timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_golden.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
for rep in 1 2; do
for d in ab/*/; do
  v=$(basename $d)
  echo "== $v $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so SCAN_STEPS=${SCAN_STEPS:-16} timeout 300 python tools/scan_sizes.py ${SIZES:-6.738415616e9} 2>&1 | grep 'd=' | cut -c1-200)"
done
done
