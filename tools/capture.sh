#!/bin/bash
# Evidence run: GPU parity tests, bench line, launch list, ncu of the batch and cluster kernels.
# usage: tools/capture.sh TAG
TAG=${1:-r01b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 --ref-seconds 3 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:inet_jit -c 1 \
  -o gpurun_out/prof_batch_$TAG python tools/profile_run.py --workload batch > gpurun_out/ncu_batch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:inet_jit -c 1 \
  -o gpurun_out/prof_a38c_$TAG python tools/profile_run.py --workload a38 --g 16 --threads 256 > gpurun_out/ncu_a38c_$TAG.log 2>&1
ls -la gpurun_out
