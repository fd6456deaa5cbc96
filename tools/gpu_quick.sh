#!/bin/bash
# quick check: tier R tests + order timing
T=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ordered.py tests/test_fuzz.py -q -x -m gpu > gpurun_out/${T}_ordered.txt 2>&1
timeout 300 python tools/order_timing.py > gpurun_out/${T}_order_timing.txt 2>&1
tail -3 gpurun_out/${T}_ordered.txt; cat gpurun_out/${T}_order_timing.txt
