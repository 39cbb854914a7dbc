MA_LIB_PATH=$PWD/ab/p2/libmicroadam_cuda.so MA_DEBUG_COUNTERS=1 SCAN_STEPS=13 timeout 300 python tools/scan_sizes.py 1.1e8 2>&1 | tail -14
