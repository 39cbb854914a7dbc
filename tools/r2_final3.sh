#!/bin/bash
# closing evidence of the session: full GPU suite, smoke, bench (ours + reference arm), launch list
mkdir -p gpurun_out
tag=${1:-fin3}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; tail -1 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 300 gpurun_out/${tag}_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; tail -c 200 gpurun_out/${tag}_bench_ref.json
for cfg in "0.05 10" "0.02 10" "0.01 20"; do
  set -- $cfg
  timeout 900 python bench.py --workload llama2-13b --density $1 --window $2 --steps 6 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_sweep_$1_$2.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_sweep_$1_$2.json').read().strip().splitlines()[-1]); print('sweep', '$1', '$2', round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${tag}_launches_7B.csv python bench.py --steps 3 --warmup 10 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep -c $tag
