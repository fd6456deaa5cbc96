"""Per-phase split of a tier R loop (INET_RTIMING development build).

    make -C paper_1404_0076_b200/csrc OUT=$PWD/tools/libinetb200_rt.so NVFLAGS+=-DINET_RTIMING
    INET_B200_LIB=tools/libinetb200_rt.so python tools/rtier_timing.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

names = ["pass1+scan", "pass2", "sort B", "merge", "fold", "tail"]
for name, params in (("fibonacci", (18,)), ("fibonacci", (15,)), ("addition", (300, 200))):
    p = program(name)
    prep = engine.prepare([p.build_input(*params)], p.rules)
    ctx = _native.Context(0)
    ctx.load_rules(prep.blob)
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    k = engine.native_cfg(EngineConfig(collect_stats=False), ordered=True)
    k.count_rules = 1
    code, ms = ctx.reduce(k)
    w = ctx.rule_counts(0, 128).astype(np.uint64)
    raw = w[64:80:2] | (w[65:80:2] << np.uint64(32))
    st = ctx.stats(0)
    loops = max(st.rounds, 1)
    tot = float(raw[:6].sum())
    print(f"{name}{params}: {ms:.3f} ms, {loops} loops, {1000 * ms / loops:.2f} us/loop; cycles/loop: "
          + ", ".join(f"{n} {raw[i] / loops:.0f} ({100 * raw[i] / max(tot, 1):.0f}%)" for i, n in enumerate(names)),
          flush=True)
    ctx.close()
