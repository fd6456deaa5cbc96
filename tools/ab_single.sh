#!/bin/bash
# single-net A/B of two libraries (run-time JIT): tools/ab_single.sh LIB_A LIB_B
A=${1:-tools/lib_this.so}; B=${2:-tools/lib_prev.so}
export INET_B200_CACHE=/tmp/abs_cache_$$
for lib in $A $B $A $B; do
  for w in fib18 a38 a310; do echo "$lib $w: $(INET_B200_LIB=$lib timeout 600 python tools/profile_run.py --workload $w --repeat 3 2>&1 | tail -1 | cut -c1-60)"; done
  echo "$lib fib18 default: $(INET_B200_LIB=$lib timeout 600 python tools/profile_run.py --workload fib18 --default-path --repeat 3 2>&1 | tail -1 | cut -c1-60)"
  echo "$lib a38 one CTA: $(INET_B200_LIB=$lib timeout 600 python tools/profile_run.py --workload a38 --g 1 --repeat 2 2>&1 | tail -1 | cut -c1-60)"
done
