#!/bin/bash
# Round-2 closing evidence: ncu of the timed kernels, GPU tests, bench (both arms), launch list, sanitizers.
T=${1:-r02final}
mkdir -p gpurun_out/$T
bash tools/gpu_r02_ncu.sh $T > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$T/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/$T/${T}_bench.json 2> gpurun_out/$T/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$T/${T}_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$T/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  q=""; [ $tool != memcheck ] && q="--quick"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py $q \
    > gpurun_out/$T/${T}_sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/$T/${T}_sanitize_$tool.txt
done
tail -2 gpurun_out/$T/${T}_pytest.txt; for t in memcheck racecheck synccheck; do tail -n 2 gpurun_out/$T/${T}_sanitize_$t.txt; done
python -c "import json; d=json.load(open('gpurun_out/$T/${T}_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
