"""Per-phase clock64 totals from the INET_TIMING development build.

    INET_B200_LIB=tools/libinetb200_timing.so python tools/phase_timing.py a38
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

spec = {"a38": ("ackermann", (3, 8), 1), "a310": ("ackermann", (3, 10), 1), "fib18": ("fibonacci", (18,), 1),
        "batch": ("ackermann", (3, 6), 4096)}[sys.argv[1]]
p = program(spec[0])
prep = engine.prepare([p.build_input(*spec[1]) for _ in range(spec[2])], p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
k = engine.native_cfg(EngineConfig(collect_stats=False))
k.count_rules = 1
code, ms = ctx.reduce(k)
raw = np.zeros(8, dtype=np.uint64)
for i in range(min(spec[2], 64)):
    w = ctx.rule_counts(i, 128).astype(np.uint64)
    raw += w[64:80:2] | (w[65:80:2] << np.uint64(32))
st = ctx.stats(0)
names = ["round start->item", "agent load+pair", "rule hdr+alloc", "agent writes", "link+settle",
         "item end->reduce", "reduce+bookkeep", "barrier wait"]
tot = raw.sum()
print(f"{sys.argv[1]} {ms:.2f} ms rounds {st.rounds} ints {st.interactions}")
for n, v in zip(names, raw):
    print(f"  {n:20s} {v / tot * 100:6.2f}%   {v / max(st.interactions, 1):10.1f} thread-cycles/interaction")
