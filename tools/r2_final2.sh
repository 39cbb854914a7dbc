#!/bin/bash
# Round-2 closing evidence: full GPU suite, smoke, bench (ours + reference arm), the 13B configs[4]
# sweep, global mode, launch list of the 7B bench step.
mkdir -p gpurun_out
tag=${1:-fin}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 300 gpurun_out/${tag}_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 200 gpurun_out/${tag}_bench_ref.json
for pt in "0.001 10" "0.005 10" "0.01 10" "0.02 10" "0.05 10" "0.01 5" "0.01 20"; do
  set -- $pt
  timeout 900 python bench.py --workload llama2-13b --density $1 --window $2 --steps 6 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_sweep_$1_$2.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/${tag}_sweep_$1_$2.json')); print('sweep', '$1', '$2', round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
timeout 600 python tools/bench_global.py 1.3e9 6.738415616e9 > gpurun_out/${tag}_global.log 2>&1; cat gpurun_out/${tag}_global.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${tag}_launches_7B.csv python bench.py --steps 3 --warmup 10 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep -c $tag
