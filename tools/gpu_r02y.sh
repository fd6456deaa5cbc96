#!/bin/bash
T=${1:-r02y}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 600 python tools/batch_round_cost.py > gpurun_out/${T}_batch_round_cost.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -3 gpurun_out/${T}_pytest.txt; cat gpurun_out/${T}_batch_round_cost.txt
