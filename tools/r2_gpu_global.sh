mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_global_big.py -x -q > gpurun_out/gbig_tests.log 2>&1; tail -15 gpurun_out/gbig_tests.log
