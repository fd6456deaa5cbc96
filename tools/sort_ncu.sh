#!/bin/bash
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for s in 0 1; do
  if [ $s = 1 ]; then export INET_B200_SORT=1; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:inet_jit_kernel --launch-skip 1 -c 1 --csv \
    python tools/profile_run.py --workload batch --repeat 2 2>/dev/null | grep -v "^==" | grep inet_jit | awk -F'","' '{print "'sort=$s' " $(NF-2) " " $NF}'
done
