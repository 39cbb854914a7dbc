#!/bin/bash
# full ncu capture of one steady-state lean launch at 1.3B for a (density, window) point
mkdir -p gpurun_out
tag=${1:-ns}; pt=${2:-0.02:10}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 14 -c 1 \
  -o /tmp/${tag} -f python tools/sweep_counters.py 1.3e9 $pt > gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${tag}_src.csv.gz
tail -2 gpurun_out/${tag}.log
