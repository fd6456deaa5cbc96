#!/bin/bash
# tier S round cost by rule-code style (0: one case per rule; 1: uniform selects; 2: warp-collective)
for st in 1 0 2; do
  echo "== style $st"
  INET_B200_JITSTYLE=$st timeout 900 python tools/batch_round_cost.py
done
