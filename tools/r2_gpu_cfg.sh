mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/cfg_tests.log 2>&1; tail -30 gpurun_out/cfg_tests.log
