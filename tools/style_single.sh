#!/bin/bash
# single nets and batches by rule-code style (unset = the engine's choice)
for st in unset 3 1; do
  for w in fib18 a38 a310; do
    if [ "$st" = unset ]; then
      echo "style $st $w: $(timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-70)"
    else
      echo "style $st $w: $(INET_B200_JITSTYLE=$st timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-70)"
    fi
  done
done
echo "== batches, style 3"; INET_B200_JITSTYLE=3 timeout 600 python tools/batch_round_cost.py
