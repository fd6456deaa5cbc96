#!/bin/bash
# Status check: GPU parity tests + per-workload timing, interpreter vs rule-set JIT.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/status_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/status_pytest.txt 2>&1
for j in 0 1; do for w in batch a310 a38 fib18; do
  timeout 300 python tools/profile_run.py --workload $w --jit $j --repeat 3 >> gpurun_out/status_runs.txt 2>&1
done; done
