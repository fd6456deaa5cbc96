"""Per-rule interaction counts of one A(3,6) net on the device (count_rules accounting run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

name, args = (sys.argv[1], tuple(int(x) for x in sys.argv[2:])) if len(sys.argv) > 1 else ("ackermann", (3, 6))
p = program(name)
prep = engine.prepare([p.build_input(*args)] * 2, p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
k = engine.native_cfg(EngineConfig(collect_stats=False))
k.count_rules = 1
code, ms = ctx.reduce(k)
h = ctx.rule_counts(0, 128)
tot = ctx.stats(0).interactions
print(name, args, "interactions", tot, "communications", ctx.stats(0).communications)
for i, r in enumerate(p.rules.rules if hasattr(p.rules, "rules") else []):
    print(i, r, int(h[i]), f"{100 * h[i] / tot:.1f}%")
print("raw", [int(x) for x in h[:16]])
