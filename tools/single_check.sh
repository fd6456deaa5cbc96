timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for w in fib18 a38 a310; do echo "$w: $(python tools/profile_run.py --workload $w --repeat 3 | tail -1 | cut -c1-90)"; done
