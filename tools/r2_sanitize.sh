#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small runs).
mkdir -p gpurun_out
out=gpurun_out/r2_sanitize.txt
: > $out
for w in lean warp generic global sparse reduce; do
  envs=""; [ $w = warp ] && envs="MA_WARP_EXACT=1"
  for tool in memcheck racecheck synccheck; do
    echo "=== $w / $tool" >> $out
    env $envs timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py $w >> $out 2>&1
    echo "exit=$?" >> $out
  done
done
grep -E "^===|ERROR SUMMARY|exit=|RACECHECK SUMMARY|^ok" $out
