# GPU suite + batch / single-net timings (development loop)
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python tools/e2e_split.py 2>&1 | tail -2
for w in fib18 a38; do echo "$w: $(python tools/profile_run.py --workload $w --repeat 3 | tail -1 | cut -c1-90)"; done
python tools/text_speed.py 2>&1 | grep lsystem
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9); print({k:(round(v['device_ms'],3),v['tier']) for k,v in d['single_nets'].items()})"
