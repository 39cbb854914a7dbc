#!/bin/bash
# lean parity tests on the in-tree build; 7B (1%) lean step and 1.3B at 5% / m = 20, in-tree vs ab/* (alternating)
mkdir -p gpurun_out
tag=${1:-ab6}
timeout 1500 python -m pytest tests/test_gpu_lean.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
b13() { python bench.py --workload opt-1.3b --density $1 --window $2 --steps 10 --warmup 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3))"; }
for rep in 1 2 3; do
echo "== in-tree $(SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"
for d in ab/*/; do echo "== $d $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so SCAN_STEPS=16 timeout 300 python tools/scan_sizes.py 6.738415616e9 2>&1 | grep 'd=' | cut -c1-60)"; done
done
for rep in 1 2; do
for cfg in "0.05 10" "0.01 20" "0.02 10"; do
echo "== in-tree 1.3B $cfg: $(b13 $cfg)"
for d in ab/*/; do echo "== $d 1.3B $cfg: $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so b13 $cfg)"; done
done
done
