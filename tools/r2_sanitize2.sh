#!/bin/bash
# global-mode GPU tests, then the sanitizer pass over every kernel family (tools/r2_sanitize.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_global_big.py -x -q > gpurun_out/san2_tests.log 2>&1; tail -1 gpurun_out/san2_tests.log
bash tools/r2_sanitize.sh
