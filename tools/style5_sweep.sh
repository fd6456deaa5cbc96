#!/bin/bash
for st in 0 1 3 5; do
  echo "style $st batch: $(INET_B200_JITSTYLE=$st timeout 600 python tools/style_batch.py 512x128 512x256 1024x128 4096x128 2>&1 | tail -1)"
  for w in fib18 a38; do echo "style $st $w: $(INET_B200_JITSTYLE=$st timeout 300 python tools/profile_run.py --workload $w --repeat 2 2>&1 | tail -1 | cut -c1-90)"; done
done
