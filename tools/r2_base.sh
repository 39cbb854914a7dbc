#!/bin/bash
# Round-2 baseline evidence on the GPU box: full GPU suite (no -x), smoke, bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_gpu.txt
lscpu > gpurun_out/r2_lscpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2_tests.log 2>&1; tail -30 gpurun_out/r2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 3000 gpurun_out/r2_bench.json
