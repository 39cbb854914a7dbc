mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_lossless.py tests/test_gpu_global.py} -x -q > gpurun_out/quick_tests.log 2>&1; tail -25 gpurun_out/quick_tests.log
