#!/bin/bash
# Build libmicroadam_cuda.so with one source file replaced (A/B on the GPU box):
#   tools/ab_variant.sh <name> <replacement ma_warp.cu> [EXTRA nvcc flags]
# -> ab/<name>/libmicroadam_cuda.so (tools/ab_run.sh times every ab/*/ variant).
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
tmp=/tmp/ab_tree_$name
rm -rf $tmp && mkdir -p $tmp
cp -r Makefile include paper_2405_15593_b200 $tmp/
rm -rf $tmp/paper_2405_15593_b200/lib
cp "$src" $tmp/paper_2405_15593_b200/csrc/$(basename "$src")
make -s -j8 -C $tmp lib EXTRA="$*" > /tmp/ab_build_$name.log 2>&1 || { echo "build $name failed"; tail -20 /tmp/ab_build_$name.log; exit 1; }
mkdir -p ab/$name && cp $tmp/paper_2405_15593_b200/lib/libmicroadam_cuda.so ab/$name/
echo "built ab/$name"
