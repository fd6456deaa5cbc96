#!/bin/bash
for S in 13824,12288,4096,8192 13568,12288,4096,8192; do
  for st in 0 1 3; do
    echo "S$st $S fib18: $(INET_B200_DEBUG=1 INET_B200_SINGLE_S=$S INET_B200_JITSTYLE=$st timeout 300 python tools/profile_run.py --workload fib18 --repeat 2 2>&1 | grep -v '^  ' | tail -3 | tr '\n' ' ' | cut -c1-400)"
  done
done
export INET_B200_LIB=tools/libinetb200_trace.so
for st in 0 3; do
INET_B200_SINGLE_S=13824,12288,4096,8192 INET_B200_JITSTYLE=$st INET_B200_CACHE=/tmp/trs$st INET_B200_TRACE_R0=800 timeout 300 python tools/mtrace.py fib18 > gpurun_out/mtrace_S${st}_fib18.txt 2>&1
done
