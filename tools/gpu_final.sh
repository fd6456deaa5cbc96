#!/bin/bash
# Evidence run: GPU tests, bench (both arms), sanitizers over every tier, launch list.
T=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py $q \
    > gpurun_out/${T}_sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/${T}_sanitize_$tool.txt
done
tail -3 gpurun_out/${T}_pytest.txt; for t in memcheck racecheck synccheck; do tail -n 3 gpurun_out/${T}_sanitize_$t.txt; done
