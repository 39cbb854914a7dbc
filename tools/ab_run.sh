#!/bin/bash
# Time each ab/<variant>/libmicroadam_cuda.so with tools/scan_sizes.py (GPU box).
sizes=${SIZES:-6.738415616e9}
for d in ab/*/; do
  v=$(basename $d)
  echo "== $v $(MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so SCAN_STEPS=${SCAN_STEPS:-16} SCAN_CYCLE=8 timeout 300 python tools/scan_sizes.py $sizes 2>&1 | grep 'd=' | cut -c1-220)"
done
