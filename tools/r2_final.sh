#!/bin/bash
# Final round-2 evidence: full GPU suite, smoke, bench (ours + reference arm), ncu capture + launch list.
mkdir -p gpurun_out
tag=${1:-r2f}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 400 gpurun_out/${tag}_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 900 python bench.py --mode sparse > gpurun_out/${tag}_bench_sparse.json 2> gpurun_out/${tag}_bench_sparse.err
timeout 900 python bench.py --grad-stream heavy --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_heavy.json 2> gpurun_out/${tag}_bench_heavy.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${tag}_launches_7B.csv python bench.py --steps 3 --warmup 10 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 12 -c 1 \
  -o /tmp/${tag}_full7b -f python bench.py --steps 1 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full7b.log 2>&1
ncu -i /tmp/${tag}_full7b.ncu-rep --page raw --csv > gpurun_out/${tag}_full7b_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_full7b.ncu-rep --page details > gpurun_out/${tag}_full7b_details.txt 2>/dev/null
ncu -i /tmp/${tag}_full7b.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${tag}_full7b_src.csv.gz
ls -la gpurun_out | grep $tag | wc -l
