#!/bin/bash
# tier S rounds sorted by rule (INET_B200_SORT=1) vs not; bench checks every net's text and the totals
B() { timeout 300 python bench.py --steps 10 --warmup 3 --no-single --no-cpu-baseline --api-steps 1 --e2e-steps 1 "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "ms")'; }
for i in 1 2; do
  echo "base : $(B) | $(timeout 300 python tools/style_batch.py 512x128 2048x128 2>&1 | tail -1)"
  echo "sort : $(INET_B200_SORT=1 B) | $(INET_B200_SORT=1 timeout 300 python tools/style_batch.py 512x128 2048x128 2>&1 | tail -1)"
done
