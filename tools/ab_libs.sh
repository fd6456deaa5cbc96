#!/bin/bash
# A/B of two libraries on one box, both JIT-compiling their kernels at run time: tools/ab_libs.sh LIB_A LIB_B
A=${1:-tools/lib_this.so}; B=${2:-tools/lib_prev.so}
export INET_B200_CACHE=/tmp/ab_cache_$$
for lib in $A $B $A $B; do
  echo "$lib batch: $(INET_B200_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-single --no-cpu-baseline --api-steps 1 --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "ms")')"
  for w in fib18 a38; do echo "$lib $w: $(INET_B200_LIB=$lib timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-45)"; done
  echo "$lib fib18 default: $(INET_B200_LIB=$lib timeout 600 python tools/profile_run.py --workload fib18 --default-path --repeat 3 2>&1 | tail -1 | cut -c1-45)"
done
