"""Tier R (reference order) vs the fast tiers on the order-sensitive configs (device time)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

for name, params in (("fibonacci", (18,)), ("fibonacci", (15,)), ("addition", (300, 200))):
    p = program(name)
    prep = engine.prepare([p.build_input(*params)], p.rules)
    ctx = _native.Context(0)
    ctx.load_rules(prep.blob)
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    row = []
    for ordered, threads in ((False, 0), (True, 256), (True, 512), (True, 1024)):
        k = engine.native_cfg(EngineConfig(collect_stats=False, threads=threads), ordered=ordered)
        code, _ = ctx.reduce(k)
        st = ctx.stats(0)
        ms = min(ctx.rerun(k) for _ in range(5))
        row.append(f"{'R' if ordered else 'fast'}{threads or ''}: {ms:.3f} ms, {st.rounds} loops, {st.interactions} ints, "
                   f"{st.communications} comms, {1000 * ms / max(st.rounds, 1):.2f} us/loop, tier {st.tier}")
    print(f"{name}{params}: " + " | ".join(row), flush=True)
    ctx.close()
