#!/bin/bash
# One GPU iteration of the tile kernel: oracle check, 7B bench (tile vs lean), 1.3B ncu capture.
# usage (under gpurun): bash tools/tile_round.sh TAG [ncu]
TAG=${1:-x}
MA_DEBUG_COUNTERS=1 timeout 300 python tools/tile_check.py > gpurun_out/tile_check_$TAG.log 2>&1; echo check rc=$?
grep -c "^ok" gpurun_out/tile_check_$TAG.log; grep -m3 "MISMATCH\|Error\|error" gpurun_out/tile_check_$TAG.log
timeout 300 python bench.py --steps 10 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("7B tile: ms/step %.2f frac %.3f steps %s" % (d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel_ms_per_step"]))
PY
if [ "$2" = "ncu" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:microadam_step_tile -s 12 -c 1 -o gpurun_out/tile_$TAG python bench.py --workload opt-1.3b --steps 2 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
fi
