#!/bin/bash
T=${1:-r02n}
mkdir -p gpurun_out
timeout 300 python tools/order_rate.py > gpurun_out/${T}_order_rate.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
timeout 300 python tools/api_split.py > gpurun_out/${T}_api_split.txt 2>&1
cat gpurun_out/${T}_order_rate.txt gpurun_out/${T}_api_split.txt; tail -2 gpurun_out/${T}_bench.err
