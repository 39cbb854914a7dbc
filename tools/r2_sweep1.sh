mkdir -p gpurun_out
P="0.01:10 0.02:10 0.05:10 0.01:20 0.01:5"
timeout 600 python tools/sweep_counters.py 1.3e9 $P > gpurun_out/sw_time.log 2>&1
MA_DEBUG_COUNTERS=1 timeout 600 python tools/sweep_counters.py 1.3e9 $P > gpurun_out/sw_cnt.log 2>&1
MA_DEBUG_COUNTERS=1 MA_LIB_PATH=$PWD/ab/prof/libmicroadam_cuda.so timeout 600 python tools/sweep_counters.py 1.3e9 $P > gpurun_out/sw_prof.log 2>&1
cat gpurun_out/sw_time.log gpurun_out/sw_cnt.log gpurun_out/sw_prof.log
