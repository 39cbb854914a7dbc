#!/bin/bash
# ncu source-level capture of one steady-state lean launch (110M bf16, window full).
mkdir -p gpurun_out
tag=${1:-cur}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 11 -c 1 \
  -o gpurun_out/${tag}_lean110m -f python tools/step_driver.py --dim 110000000 --steps 13 > gpurun_out/${tag}_ncu.log 2>&1
tail -2 gpurun_out/${tag}_ncu.log
ncu -i gpurun_out/${tag}_lean110m.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ncu -i gpurun_out/${tag}_lean110m.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ls -la gpurun_out | tail -5
