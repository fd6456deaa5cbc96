#!/bin/bash
# tier R phase split + e2e_api after the whole-batch ABI calls
T=${1:-r02h}
mkdir -p gpurun_out
INET_B200_LIB=tools/libinetb200_rt.so timeout 300 python tools/rtier_timing.py > gpurun_out/${T}_rtier_timing.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_ordered.py tests/test_gpu_parity.py -q -x > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cat gpurun_out/${T}_rtier_timing.txt; tail -2 gpurun_out/${T}_pytest.txt
