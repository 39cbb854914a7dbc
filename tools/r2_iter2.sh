#!/bin/bash
# full GPU suite + the configs[4] points most affected by shared-memory staging + a 7B timing
mkdir -p gpurun_out
tag=${1:-it}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
: > gpurun_out/${tag}_sweep.jsonl
for dm in "0.02 10" "0.05 10" "0.01 20" "0.01 10"; do
  set -- $dm
  timeout 900 python bench.py --workload llama2-13b --density $1 --window $2 --steps 6 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/${tag}_sweep.jsonl 2>/dev/null
done
python3 -c "
import json
for l in open('gpurun_out/${tag}_sweep.jsonl'):
    d=json.loads(l); print(d['config']['workload'][-60:], round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"
SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-120
