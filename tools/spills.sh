#!/bin/sh
# registers / spills of the warp kernel's hot (non-report) instantiations
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xptxas -v -Iinclude -dc -o /tmp/_w.o paper_2405_15593_b200/csrc/ma_warp.cu 2>&1 \
  | grep -A2 "Compiling entry.*microadam_step_warp.*Lb0E" | grep -E "Used|spill" | sort | uniq -c
