#!/bin/bash
# Full ncu capture of one steady-state launch (110M bf16) of kernel regex $1
# with env $2 (e.g. MA_TILE=1); exports raw + source CSV into gpurun_out/ and
# drops the .ncu-rep (reports exceed gpurun's copy-back limit).
k=${1:-microadam_step_lean}; envs=${2:-}; tag=${3:-k}; dim=${DIM:-110000000}
mkdir -p gpurun_out
env $envs timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s ${SKIP:-11} -c 1 \
  -o /tmp/${tag} -f python tools/step_driver.py --dim $dim --steps ${STEPS:-13} > gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>/dev/null
gzip -f gpurun_out/${tag}_src.csv
