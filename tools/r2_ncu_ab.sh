#!/bin/bash
# Instruction count / issue / time of one steady-state lean launch for each ab/*/ variant (110M bf16).
mkdir -p gpurun_out
for d in ab/*/; do
  v=$(basename $d)
  MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:microadam_step_lean -s 11 -c 1 python tools/step_driver.py --dim 110000000 --steps 13 2>&1 | grep -E "duration|inst_executed|issue_active|warps_active|bytes" | sed "s/^/$v /"
done
if [ -n "$FULL" ]; then
  for d in ab/*/; do v=$(basename $d)
  MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 11 -c 1 \
    -o gpurun_out/${v}_lean110m -f python tools/step_driver.py --dim 110000000 --steps 13 > /dev/null 2>&1
  done
fi
