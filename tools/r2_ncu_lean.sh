#!/bin/bash
# full ncu capture of one steady-state lean launch at 7B (+ source/SASS page)
mkdir -p gpurun_out
tag=${1:-nl}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 12 -c 1 \
  -o /tmp/${tag} -f python bench.py --steps 1 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${tag}_src.csv.gz
tail -2 gpurun_out/${tag}.log
