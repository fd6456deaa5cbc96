#!/bin/bash
# A/B: this library vs tools/lib_prev.so (the previous device code), same box
for lib in "" tools/lib_prev.so "" tools/lib_prev.so; do
  if [ -z "$lib" ]; then pre="X=1"; name=this; else pre="INET_B200_LIB=$lib"; name=prev; fi
  echo "$name batch: $(env $pre timeout 300 python bench.py --steps 10 --warmup 3 --no-single --no-cpu-baseline --api-steps 1 --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "ms")')"
  for w in fib18 a38; do echo "$name $w: $(env $pre timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-45)"; done
done
