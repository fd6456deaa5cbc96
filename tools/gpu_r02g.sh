#!/bin/bash
# tests, bench, sanitizers (tier R included), host split of the single-net end-to-end path
T=${1:-r02g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for tool in memcheck synccheck racecheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py $q \
    > gpurun_out/${T}_sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/${T}_sanitize_$tool.txt
done
timeout 300 python tools/host_split.py > gpurun_out/${T}_host_split.txt 2>&1
ls -la gpurun_out | tail -12
