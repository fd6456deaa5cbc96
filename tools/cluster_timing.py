"""Critical-path split of tier C rounds (INET_CTIMING build).

    INET_B200_LIB=tools/libinetb200_ctiming.so python tools/cluster_timing.py a310 16 512
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

spec = {"a23": ("ackermann", (2, 3)), "a38": ("ackermann", (3, 8)), "a310": ("ackermann", (3, 10)),
        "fib18": ("fibonacci", (18,)), "a36": ("ackermann", (3, 6))}[sys.argv[1]]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 16
T = int(sys.argv[3]) if len(sys.argv) > 3 else 512
p = program(spec[0])
prep = engine.prepare([p.build_input(*spec[1])], p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
k = engine.native_cfg(EngineConfig(collect_stats=False, threads=T, ctas_per_net=G))
k.count_rules = 1
code, ms = ctx.reduce(k)
w = ctx.rule_counts(0, 128).astype(np.uint64)
raw = w[64:72:2] | (w[65:72:2] << np.uint64(32))
st = ctx.stats(0)
rounds = max(st.rounds, 1)
names = ["work (slowest thread)", "reduce+arrive", "barrier wait", "gather"]
tot = raw.sum()
print(f"{sys.argv[1]} G={G} T={T} code={code} {ms:.2f} ms rounds {st.rounds} ints {st.interactions} "
      f"-> {ms * 1e3 / rounds:.3f} us/round")
for n, v in zip(names, raw):
    print(f"  {n:22s} {v / tot * 100:6.2f}%   {v / G / rounds:9.1f} cycles/round")
