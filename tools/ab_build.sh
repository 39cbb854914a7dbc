#!/bin/bash
# Build libmicroadam_cuda.so variants with extra -D flags; only the .so lands in
# ab/<name>/ (it travels to the GPU box for tools/ab_run.sh):
#   tools/ab_build.sh name "-DMA_LEAN_PERSIST=0 ..." ...
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p ab/$name /tmp/ab_build_$name
  make -s lib LIBDIR=/tmp/ab_build_$name EXTRA="$flags" >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
  cp /tmp/ab_build_$name/libmicroadam_cuda.so ab/$name/
  echo "built ab/$name ($flags)"
done
