#!/bin/bash
# Round-2 profile evidence on the GPU box (never bench values: ncu runs are serialized/cold).
mkdir -p gpurun_out
tag=${1:-r02}
# 1. launch list of the bench command (per-launch times, cold/serialized)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${tag}_launches_7B.csv python bench.py --steps 3 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_launch_bench.log 2>&1
# 2. full capture of one steady-state lean launch at 7B (window full)
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 12 -c 1 \
  -o /tmp/${tag}_full7b -f python bench.py --steps 1 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full7b.log 2>&1
ncu -i /tmp/${tag}_full7b.ncu-rep --page raw --csv > gpurun_out/${tag}_full7b_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_full7b.ncu-rep --page details > gpurun_out/${tag}_full7b_details.txt 2>/dev/null
ncu -i /tmp/${tag}_full7b.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${tag}_full7b_src.csv.gz
# 3. phase split at 7B
timeout 600 python tools/phase_split.py 6.738415616e9 14 > gpurun_out/${tag}_phase_split.txt 2>&1
# 4. configs[4] sweep (Llama-2-13B-sized bf16 vector)
: > gpurun_out/${tag}_sweep.jsonl
for dm in "0.001 10" "0.005 10" "0.01 10" "0.02 10" "0.05 10" "0.01 5" "0.01 20"; do
  set -- $dm
  timeout 900 python bench.py --workload llama2-13b --density $1 --window $2 --steps 6 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/${tag}_sweep.jsonl 2> gpurun_out/${tag}_sweep_err.log
done
# 5. global Top-K mode
timeout 900 python tools/bench_global.py 1.3e9 6.738415616e9 > gpurun_out/${tag}_global.txt 2>&1
tail -3 gpurun_out/${tag}_phase_split.txt gpurun_out/${tag}_global.txt; wc -l gpurun_out/${tag}_sweep.jsonl
