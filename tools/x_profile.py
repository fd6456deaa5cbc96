"""One tier X reduction of lsystem(n) (for an ncu capture)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("lsystem")
prep = engine.prepare([p.build_input(int(sys.argv[1]) if len(sys.argv) > 1 else 26)], p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
k = engine.native_cfg(EngineConfig(collect_stats=False, ctas_per_net=148))
code, ms = ctx.reduce(k)
print("code", code, "ms", ms, "tier", ctx.stats(0).tier)
