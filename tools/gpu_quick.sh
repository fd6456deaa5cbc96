# GPU suite + batch / single-net timings (development loop)
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python tools/e2e_split.py 2>&1 | tail -2
for w in fib18 a38; do echo "$w: $(python tools/profile_run.py --workload $w --repeat 3 | tail -1 | cut -c1-90)"; done
