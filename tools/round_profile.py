"""Per-round device time vs. active pairs (from LoopStats.elapsed ns)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

name, params = sys.argv[1], tuple(int(x) for x in sys.argv[2:])
p = program(name)
prep = engine.prepare([p.build_input(*params)], p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
k = engine.native_cfg(EngineConfig(collect_stats=True))
code, ms = ctx.reduce(k)
rows = ctx.rounds(0).astype(np.float64)
ints, ns = rows[:-1, 0], rows[1:, 3]  # row r's time is stored with row r (time of round r)
ns = rows[:, 3][:-1]
print(f"{name}{params}: {ms:.2f} ms, rounds {len(rows)}, sum(ns) {rows[:,3].sum()/1e6:.2f} ms")
for lo, hi in [(0, 1), (1, 33), (33, 129), (129, 513), (513, 1025), (1025, 2049), (2049, 4097), (4097, 10**9)]:
    m = (ints >= lo) & (ints < hi)
    if m.any():
        print(f"  ints in [{lo},{hi}): rounds {m.sum():6d}  mean ints {ints[m].mean():8.1f}  mean us {ns[m].mean()/1e3:7.2f}  "
              f"total ms {ns[m].sum()/1e6:8.2f}")
A = np.vstack([np.ones_like(ints), ints]).T
coef, *_ = np.linalg.lstsq(A, ns, rcond=None)
print(f"  fit: {coef[0]/1e3:.2f} us + {coef[1]:.2f} ns * ints")
