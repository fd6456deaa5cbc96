#!/bin/bash
# tier S (whole net in shared memory) vs tier M for single nets: timing and round traces
mkdir -p gpurun_out
S=8192,8192,4096,8192
for w in fib18 a38; do
  echo "M   $w: $(timeout 300 python tools/profile_run.py --workload $w --g 1 --repeat 3 2>&1 | tail -1 | cut -c1-140)"
  for st in 0 1; do
    echo "S$st  $w: $(INET_B200_SINGLE_S=$S INET_B200_JITSTYLE=$st timeout 300 python tools/profile_run.py --workload $w --g 1 --repeat 3 2>&1 | tail -1 | cut -c1-140)"
  done
done
export INET_B200_LIB=tools/libinetb200_trace.so
for st in 0 1; do
  INET_B200_SINGLE_S=$S INET_B200_JITSTYLE=$st INET_B200_CACHE=/tmp/trs$st INET_B200_TRACE_R0=800 timeout 300 python tools/mtrace.py fib18 > gpurun_out/mtrace_S${st}_fib18.txt 2>&1
  INET_B200_SINGLE_S=$S INET_B200_JITSTYLE=$st INET_B200_CACHE=/tmp/trs$st INET_B200_TRACE_R0=3000 timeout 300 python tools/mtrace.py a38 > gpurun_out/mtrace_S${st}_a38.txt 2>&1
done
INET_B200_JITSTYLE=0 INET_B200_CACHE=/tmp/trm0 INET_B200_TRACE_R0=800 timeout 300 python tools/mtrace.py fib18 > gpurun_out/mtrace_M0_fib18.txt 2>&1
