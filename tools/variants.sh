#!/bin/bash
# Time single-net workloads with several development builds of the library.
for lib in paper_1404_0076_b200/libinetb200.so tools/lib_X1.so tools/lib_X2.so tools/lib_X3.so; do
  for w in a310 a38 fib18; do
    echo -n "$lib $w t1024: "; INET_B200_LIB=$lib python tools/profile_run.py --workload $w | cut -c1-60
  done
  echo -n "$lib a310 t512: "; INET_B200_LIB=$lib python tools/profile_run.py --workload a310 --threads 512 | cut -c1-60
done
