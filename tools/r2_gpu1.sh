mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_collective.py -q -x > gpurun_out/coll_tests.log 2>&1; tail -3 gpurun_out/coll_tests.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2b_tests.log 2>&1; tail -3 gpurun_out/r2b_tests.log
timeout 600 python tools/phase_split.py 6.738415616e9 14
MA_LIB_PATH=$PWD/ab/base/libmicroadam_cuda.so timeout 600 python tools/phase_split.py 6.738415616e9 14
