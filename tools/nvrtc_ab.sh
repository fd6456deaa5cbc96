#!/bin/bash
# kernels compiled by the system NVRTC (12.9) vs the one bundled with torch (12.8), run-time compiled
N129=/usr/local/cuda-12.9/targets/x86_64-linux/lib/libnvrtc.so.12.9.86
N128=$(python -c "import nvidia.cuda_nvrtc, os; print(os.path.join(list(nvidia.cuda_nvrtc.__path__)[0], 'lib', 'libnvrtc.so.12'))")
mv paper_1404_0076_b200/kernels /tmp/kernels_off
for rep in 1 2; do
for nv in $N129 $N128; do
  export INET_B200_NVRTC=$nv INET_B200_CACHE=/tmp/nv_$(basename $nv)
  echo "== $nv"
  INET_B200_DEBUG=1 timeout 300 python tools/style_batch.py 4096x128 512x128 2>&1 | grep -v "^  \|attempt" | tail -2
  for w in fib18 a38 a310; do echo "$w: $(timeout 600 python tools/profile_run.py --workload $w --repeat 2 2>&1 | tail -1 | cut -c1-50)"; done
done
done
mv /tmp/kernels_off paper_1404_0076_b200/kernels
