#!/bin/bash
# Per-variant ncu metrics (110M bf16, one steady-state lean launch) + phase split timing (7B).
for d in ab/*/; do
  v=$(basename $d)
  MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_not_selected,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_branch_resolving \
    --clock-control none -k regex:microadam_step_lean -s 11 -c 1 python tools/step_driver.py --dim 110000000 --steps 13 2>&1 | grep -E "duration|inst_executed|issue_active|warps_active|bytes|lts__t|stalled" | sed "s/^/$v /"
  MA_LIB_PATH=$PWD/$d/libmicroadam_cuda.so timeout 600 python tools/phase_split.py 6.738415616e9 14 | sed "s/^/$v /"
done
