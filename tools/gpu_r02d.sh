#!/bin/bash
# Round-2 evidence: GPU tests, bench, ncu launch list and instruction metrics of the timed kernels.
T=${1:-r02d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__cycles_active.avg
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launches_bench.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:inet_jit_kernel --launch-skip 1 -c 1 --csv \
  --log-file gpurun_out/${T}_issue_batch.csv python bench.py --steps 1 --warmup 3 --no-single --no-cpu-baseline \
  --api-steps 1 --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:inet_jit_kernel --launch-skip 2 -c 2 --csv \
  --log-file gpurun_out/${T}_issue_a310.csv python bench.py --workload a310 --steps 1 --warmup 3 --no-single \
  --no-cpu-baseline --api-steps 1 --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:reduce_ordered --launch-skip 1 -c 1 --csv \
  --log-file gpurun_out/${T}_issue_fib18_tierR.csv python tools/order_timing.py > gpurun_out/${T}_order_timing_ncu.log 2>&1
timeout 300 python tools/order_timing.py > gpurun_out/${T}_order_timing.txt 2>&1
ls -la gpurun_out | tail -20
