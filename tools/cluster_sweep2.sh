#!/bin/bash
# tier C (cluster) by code style and CTA size, NVRTC 12.8 kernels (auto path: tier M prefix then the cluster)
for w in a38 a310; do
  for st in 1 0 3; do
    for t in 256 512; do
      echo "$w style $st threads $t: $(INET_B200_JITSTYLE=$st timeout 600 python tools/profile_run.py --workload $w --threads $t --repeat 2 2>&1 | tail -1 | cut -c1-60)"
    done
  done
done
