#!/bin/bash
export INET_B200_CACHE=/tmp/zc_cache
for lib in tools/lib_this.so tools/lib_prev.so tools/lib_this.so tools/lib_prev.so; do
  echo "== $lib"
  INET_B200_LIB=$lib timeout 300 python tools/e2e_split.py | tail -2
  INET_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-single --no-cpu-baseline --api-steps 2 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bench ms", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["value"]/1e9,2), "api", round(d["e2e_api"]["value"]/1e9,2))'
done
