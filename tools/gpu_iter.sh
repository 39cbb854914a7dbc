#!/bin/bash
# One build -> measure iteration on the GPU box: lean-kernel tests, full GPU
# suite, a size scan (timing), and the debug counters of a short run.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lean.py -x -q > gpurun_out/it_lean.log 2>&1; tail -15 gpurun_out/it_lean.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_tests.log 2>&1; tail -15 gpurun_out/it_tests.log
SCAN_STEPS=16 SCAN_CYCLE=8 timeout 600 python tools/scan_sizes.py 1.1e8 6.738415616e9 2>&1 | grep "d=" | cut -c1-200
timeout 600 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 9 -c 1 -o gpurun_out/it_lean -f python tools/step_driver.py --dim 110000000 --steps 11 > gpurun_out/it_ncu.log 2>&1; tail -1 gpurun_out/it_ncu.log
