"""First loop where the stamped fast tier's rows leave the reference's (fibonacci)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("fibonacci")
ctx = _native.context(0)
for n in range(3, 19):
    cfg = p.build_input(n)
    want = O.run_config(cfg, O.rules_for("fibonacci"), collect=True)
    prep = engine.prepare([cfg], p.rules)
    for rep in range(2):
        with ctx.lock:
            outs, _ = engine._reduce(ctx, prep, EngineConfig(), engine.MODE_STAMPS, False, True)
        o = outs[0]
        rows = [tuple(int(v) for v in r[:3]) for r in o.rows]
        wr = [tuple(r) for r in want.rows]
        first = next((i for i, (a, b) in enumerate(zip(rows, wr)) if a != b), None)
        print(f"fib({n}) rep {rep}: status {o.stats.status} tier {o.stats.tier} loops {len(rows)}/{len(wr)} "
              f"comms {o.stats.communications}/{want.communications} first diff {first}", flush=True)
        if first is not None:
            lo = max(0, first - 2)
            print("  dev", rows[lo:first + 3])
            print("  ref", wr[lo:first + 3])
