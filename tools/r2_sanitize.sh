#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small runs);
# one summary line per (family, tool) in gpurun_out/r2_sanitize_summary.txt
mkdir -p gpurun_out
out=gpurun_out/r2_sanitize.txt
sum=gpurun_out/r2_sanitize_summary.txt
: > $out; : > $sum
for w in lean warp generic global sparse reduce; do
  envs=""; [ $w = warp ] && envs="MA_WARP_EXACT=1"
  for tool in memcheck racecheck synccheck; do
    log=/tmp/san_${w}_${tool}.log
    env $envs timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py $w > $log 2>&1
    rc=$?
    cat $log >> $out
    res=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $log | tail -1 | sed 's/=========//')
    ok=$(grep -c "^ok " $log)
    echo "$w $tool exit=$rc run_ok=$ok $res" >> $sum
  done
done
cat $sum
