"""Tier S round cost of one A(3,6) net against how many nets share the GPU (device timers per round)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
for n_nets in (2, 148, 296, 512, 1024, 2048, 4096):
    for threads in (64, 128, 256):
        prep = engine.prepare([p.build_input(3, 6)] * n_nets, p.rules)
        ctx = _native.Context(0)
        ctx.load_rules(prep.blob)
        ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
        code, ms = ctx.reduce(engine.native_cfg(EngineConfig(collect_stats=False, threads=threads)))
        ms = min(ctx.rerun(engine.native_cfg(EngineConfig(collect_stats=False, threads=threads))) for _ in range(3))
        st = ctx.stats(0)
        print(f"{n_nets:5d} nets, {threads:3d} threads: {ms:7.3f} ms, {1000 * ms / st.rounds:5.2f} us/round "
              f"(tier {st.tier})", flush=True)
        ctx.close()
