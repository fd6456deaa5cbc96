#!/bin/bash
# ncu --set full with source of the batch kernel (JIT source dumped so ncu can map lines)
T=${1:-r02q}
mkdir -p gpurun_out/$T
rm -rf paper_1404_0076_b200/kernels  # (the box's copy) force NVRTC so the source is dumped next to the run
cd gpurun_out/$T
export INET_B200_JITDUMP=1 INET_B200_CACHE=$PWD/cache
timeout 900 ncu --set full --clock-control none --import-source on -k regex:inet_jit -c 1 \
  -o prof_batch python ../../tools/profile_run.py --workload batch > ncu_batch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:inet_jit -c 1 \
  -o prof_a38c python ../../tools/profile_run.py --workload a38 --g 16 --threads 256 > ncu_a38c.log 2>&1
rm -rf cache
ls -la
