for st in 0 1; do for j in 0 1; do for g in 2 4 16; do
 echo -n "style=$st jit=$j G=$g: "; INET_B200_JITSTYLE=$st timeout 60 python tools/profile_run.py --workload a38 --jit $j --g $g --threads 512 2>&1 | tail -1
done; done; done
