"""One reduction of a named workload (for ncu captures; prints nothing timed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="a38")
ap.add_argument("--nets", type=int, default=4096)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--jit", type=int, default=1)
ap.add_argument("--g", type=int, default=0, help="CTAs per net (tier C cluster)")
ap.add_argument("--exact", type=int, default=1, help="reference loop mode")
ap.add_argument("--default-path", action="store_true", help="the evaluation order evaluate() picks (stamps / tier R)")
a = ap.parse_args()
spec = {"a38": ("ackermann", (3, 8), 1), "a310": ("ackermann", (3, 10), 1), "fib18": ("fibonacci", (18,), 1),
        "batch": ("ackermann", (3, 6), a.nets)}[a.workload]
p = program(spec[0])
prep = engine.prepare([p.build_input(*spec[1]) for _ in range(spec[2])], p.rules)
ctx = _native.Context(0)
ctx.set_jit(bool(a.jit))
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
ecfg = EngineConfig(collect_stats=False, threads=a.threads, ctas_per_net=a.g, exact_loops=bool(a.exact))
if a.default_path:
    mode, _ = engine._plan(ecfg, p.rules, [p.build_input(*spec[1])])
    k = engine.native_cfg(ecfg, mode == engine.MODE_R, mode == engine.MODE_STAMPS)
else:
    k = engine.native_cfg(ecfg)
for _ in range(a.repeat):
    code, ms = ctx.reduce(k)
    st = ctx.stats(0)
    print(a.workload, "code", code, "ms", ms, ctx.totals(), "tier", st.tier, "jit", st.jit, "hw", st.agent_hw, st.var_hw, "MHz", st.sm_mhz)
