#!/bin/bash
# ncu warp-state capture of the single-net fib(18) kernel: tier M (default) and tier S (whole net in smem)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:inet_jit -c 1 -f -o gpurun_out/fib18_M python tools/profile_run.py --workload fib18 > /dev/null 2>&1
INET_B200_SINGLE_S=13824,12288,4096,8192 INET_B200_JITSTYLE=0 ncu --set full --import-source on --clock-control none -k regex:inet_jit -c 2 -f -o gpurun_out/fib18_S python tools/profile_run.py --workload fib18 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
