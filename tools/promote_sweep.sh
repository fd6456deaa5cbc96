#!/bin/bash
# tier M -> tier C hand-over threshold (interactions) on A(3,8) / A(3,10)
for p in 65536 131072 262144 524288 1048576 2097152; do
  for w in a38 a310; do
    echo "promote $p $w: $(INET_B200_PROMOTE=$p timeout 600 python tools/profile_run.py --workload $w --repeat 2 2>&1 | tail -1 | cut -c1-50)"
  done
done
