#!/bin/bash
# global-mode 1.3B step time + bracket kernel time: in-tree vs ab/* variants
mkdir -p gpurun_out
tag=${1:-abg}
for rep in 1 2; do
echo "== in-tree"; timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-50
for d in ab/*/; do echo "== $d"; MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 python tools/bench_global.py 1.3e9 2>&1 | cut -c1-50; done
done
for d in ab/*/; do v=$(basename $d); MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:g_requant8 -c 30 --csv --log-file gpurun_out/${tag}_$v.csv python tools/bench_global.py 1.3e9 > /dev/null 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:g_requant8 -c 30 --csv --log-file gpurun_out/${tag}_intree.csv python tools/bench_global.py 1.3e9 > /dev/null 2>&1
