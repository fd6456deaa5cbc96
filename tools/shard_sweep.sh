# per-GPU shard sizes of the 1/2/4/8-GPU batch (4096 / N nets) x threads per net
for n in 2048 1024 512; do for t in 128 256 512; do
  echo "nets=$n t=$t: $(python tools/profile_run.py --workload batch --nets $n --threads $t --repeat 3 | tail -1 | cut -c1-60)"
done; done
