#!/bin/bash
# tier S single nets with capacities that fit fib(18): styles 0/1/3 vs the default path
S=${S:-14336,12288,2048,8192}
for w in fib18 a38 a310; do
  echo "auto $w: $(timeout 300 python tools/profile_run.py --workload $w --repeat 2 2>&1 | tail -1 | cut -c1-140)"
  for st in 0 1 3; do
    echo "S$st  $w: $(INET_B200_DEBUG=0 INET_B200_SINGLE_S=$S INET_B200_JITSTYLE=$st timeout 300 python tools/profile_run.py --workload $w --repeat 2 2>&1 | tail -1 | cut -c1-140)"
  done
done
