#!/bin/bash
# A/B harness for the GPU box: tools/ab.sh <dir-with-variant-.cu-files> [sizes...]
# Each variant replaces csrc/ma_warp.cu, is rebuilt, then timed (scan) and its
# DRAM bytes of one steady-state launch are read with ncu (never a timing).
dir=$1; shift
sizes=${@:-1.1e8 6.738415616e9}
mkdir -p gpurun_out
for f in "$dir"/*.cu; do
  v=$(basename "$f" .cu)
  cp "$f" paper_2405_15593_b200/csrc/ma_warp.cu
  make lib > gpurun_out/ab_build_$v.log 2>&1 || { echo "$v: build failed"; continue; }
  echo "== $v"
  SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py $sizes 2>&1 | grep "d="
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none -k regex:microadam_step_warp -s 12 -c 1 \
      python tools/step_driver.py --dim 110000000 --steps 14 2>&1 | grep -E "duration|bytes|inst_executed"
done
