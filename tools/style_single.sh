#!/bin/bash
# single nets by rule-code style (tier M prefix / tier C)
for st in "" 1 0; do
  for w in fib18 a38 a310; do
    echo "style '${st}' $w: $(INET_B200_JITSTYLE=$st timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-70)"
  done
done
