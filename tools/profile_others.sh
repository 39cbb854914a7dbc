#!/bin/bash
# ncu captures of the non-default kernel families (one GPU).
mkdir -p gpurun_out
MA_FORCE_GENERIC=1 timeout 600 ncu --set full --clock-control none -k regex:microadam_step_kernel -s 10 -c 1 -o gpurun_out/oth_generic -f python tools/profile_others.py generic 1.1e8 > gpurun_out/oth_generic.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:microadam_step_lean -s 20 -c 2 -o gpurun_out/oth_sparse -f python tools/profile_others.py sparse 1.1e8 > gpurun_out/oth_sparse.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:g_ -s 150 -c 60 --csv --log-file gpurun_out/oth_global.csv python tools/profile_others.py global 1.1e8 > gpurun_out/oth_global.log 2>&1
for f in gpurun_out/oth_*.log; do tail -n 2 $f; done
