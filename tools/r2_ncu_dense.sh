#!/bin/bash
# full ncu capture of one steady-state lean launch at OPT-1.3B, 5% density (16-slot variant) and m = 20
mkdir -p gpurun_out
tag=${1:-nd}
for cfg in "0.05 10" "0.01 20"; do
  set -- $cfg
  t=${tag}_$1_$2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 21 -c 1 \
    -o /tmp/${t} -f python bench.py --workload opt-1.3b --density $1 --window $2 --steps 1 --warmup 21 --no-e2e --no-cpu-baseline > gpurun_out/${t}.log 2>&1
  ncu -i /tmp/${t}.ncu-rep --page raw --csv > gpurun_out/${t}_raw.csv 2>/dev/null
  ncu -i /tmp/${t}.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${t}_src.csv.gz
  tail -1 gpurun_out/${t}.log
done
