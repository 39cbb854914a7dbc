#!/bin/bash
mkdir -p gpurun_out
tag=${1:-gn}
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k 'regex:^(g_bracket|g_stats_sparse)$' -s 40 -c 4 -o /tmp/${tag} -f python tools/bench_global.py 1.3e9 > gpurun_out/${tag}.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${tag}_src.csv.gz
tail -3 gpurun_out/${tag}.log
