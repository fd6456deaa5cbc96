#!/bin/bash
export INET_B200_LIB=tools/libinetb200_trace.so
mkdir -p gpurun_out
for spec in "fib18 800" "fib18 1200" "a38 3000" "a38 9000" "add 150"; do
  set -- $spec
  INET_B200_CACHE=/tmp/trc_$1_$2 INET_B200_TRACE_R0=$2 timeout 300 python tools/mtrace.py $1 > gpurun_out/mtrace_$1_$2.txt 2>&1
  echo "$1 $2 rc=$? lines=$(wc -l < gpurun_out/mtrace_$1_$2.txt)"
done
