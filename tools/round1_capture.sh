#!/bin/bash
# Round-1 evidence: bench line, launch list of the bench command, full ncu of the batch kernel.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 --ref-seconds 3 > gpurun_out/bench_ref_r01.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
  python bench.py --steps 2 --warmup 3 --no-single --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -c 1 \
  -o gpurun_out/prof_batch_r01 python tools/profile_run.py --workload batch > gpurun_out/ncu_batch_r01.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -c 1 \
  -o gpurun_out/prof_a310_r01 python tools/profile_run.py --workload a310 > gpurun_out/ncu_a310_r01.log 2>&1
python tools/round_profile.py ackermann 3 10 > gpurun_out/rounds_a310_r01.txt 2>&1
ls -la gpurun_out
