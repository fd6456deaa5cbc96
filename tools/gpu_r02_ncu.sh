#!/bin/bash
# ncu captures of the timed kernels (instruction metrics + one --set full of the batch kernel) for profiles/
T=${1:-r02ap}
mkdir -p gpurun_out/$T
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__cycles_active.avg
timeout 600 ncu --metrics $M --clock-control none -k regex:inet_jit_kernel --launch-skip 1 -c 1 --csv \
  --log-file gpurun_out/$T/${T}_issue_batch.csv python bench.py --steps 1 --warmup 3 --no-single --no-cpu-baseline \
  --api-steps 1 --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:inet_jit_kernel --launch-skip 2 -c 2 --csv \
  --log-file gpurun_out/$T/${T}_issue_a310.csv python bench.py --workload a310 --steps 1 --warmup 3 --no-single \
  --no-cpu-baseline --api-steps 1 --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:reduce_ordered --launch-skip 1 -c 1 --csv \
  --log-file gpurun_out/$T/${T}_issue_fib18_tierR.csv python tools/order_timing.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:inet_jit_kernel --launch-skip 1 -c 1 -f \
  -o gpurun_out/$T/${T}_batch_full python bench.py --steps 1 --warmup 3 --no-single --no-cpu-baseline \
  --api-steps 1 --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out/$T
