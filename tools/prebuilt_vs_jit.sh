#!/bin/bash
# the same library with its prebuilt kernels/ vs compiling at run time (into a fresh cache)
mkdir -p gpurun_out/pvj
B() { timeout 300 python bench.py --steps 10 --warmup 3 --no-single --no-cpu-baseline --api-steps 1 --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "ms")'; }
for i in 1 2; do
  echo "prebuilt: $(B)"
  mv paper_1404_0076_b200/kernels /tmp/kernels_off
  echo "runtime : $(INET_B200_CACHE=/tmp/pvj_cache B)"
  mv /tmp/kernels_off paper_1404_0076_b200/kernels
done
cp /tmp/pvj_cache/*.cubin gpurun_out/pvj/ 2>/dev/null; ls gpurun_out/pvj | head
