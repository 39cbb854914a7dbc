set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1b_tests.log 2>&1; tail -2 gpurun_out/r1b_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b_smoke.log 2>&1; tail -2 gpurun_out/r1b_smoke.log
timeout 900 python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err; tail -c 3000 gpurun_out/r1b_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1b_bench_ref.json 2> gpurun_out/r1b_bench_ref.err; tail -c 1500 gpurun_out/r1b_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches.csv python bench.py --steps 3 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/r1b_launch_bench.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:microadam_step_lean -s 13 -c 1 -o gpurun_out/r1b_full7b -f python bench.py --steps 2 --warmup 12 --no-e2e --no-cpu-baseline > gpurun_out/r1b_full7b.log 2>&1
MA_LIB_PATH=$PWD/ab/prof/libmicroadam_cuda.so MA_DEBUG_COUNTERS=1 SCAN_CYCLE=1000 timeout 600 python tools/prof_phases.py 1.1e9 > gpurun_out/r1b_phases.log 2>&1; tail -4 gpurun_out/r1b_phases.log
ls -la gpurun_out | tail -8
