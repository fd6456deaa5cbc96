#!/bin/bash
# Round-2 baseline evidence: GPU tests, bench, compute-sanitizer over every tier.
# usage: tools/r02_baseline.sh TAG
T=${1:-r02b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for tool in memcheck synccheck racecheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py $q \
    > gpurun_out/${T}_sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/${T}_sanitize_$tool.txt
done
ls -la gpurun_out | tail -20
