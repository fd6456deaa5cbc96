"""Device time per round against its width, tier C (cluster) vs tier M (one CTA), A(3,10).

Rows come from the device's %globaltimer (collect_stats): the hybrid estimate
takes, round by round, the cheaper of the two measured costs for that width."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
params = tuple(int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (3, 10)))
prep = engine.prepare([p.build_input(*params)], p.rules)
res = {}
for label, g in (("C", 0), ("M", 1)):
    ctx = _native.Context(0)
    ctx.load_rules(prep.blob)
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    k = engine.native_cfg(EngineConfig(collect_stats=True, ctas_per_net=g))
    code, ms = ctx.reduce(k)
    rows = ctx.rounds(0).astype(np.int64)
    st = ctx.stats(0)
    print(f"tier {label}: {ms:.1f} ms, {len(rows)} rows, tier {st.tier}", flush=True)
    res[label] = rows
    ctx.close()
n = res["C"][:, 0]
tc, tm = res["C"][:, 3].astype(float), res["M"][:, 3].astype(float)
m = min(len(tc), len(tm))
n, tc, tm = n[:m], tc[:m], tm[:m]
edges = [0, 16, 64, 128, 256, 512, 768, 1024, 1536, 2048, 3072, 5000]
print("width      rounds   tierC_us  tierM_us")
for a, b in zip(edges, edges[1:]):
    sel = (n >= a) & (n < b)
    if sel.any():
        print(f"[{a:4d},{b:4d}) {sel.sum():7d}  {tc[sel].mean() / 1e3:8.2f}  {tm[sel].mean() / 1e3:8.2f}")
print(f"total: tier C {tc.sum() / 1e6:.1f} ms, tier M {tm.sum() / 1e6:.1f} ms, "
      f"per-round min (hybrid, no switching cost) {np.minimum(tc, tm).sum() / 1e6:.1f} ms")
for T in (256, 512, 768, 1024, 1536):
    hyb = np.where(n < T, tm, tc).sum()
    print(f"threshold {T}: {hyb / 1e6:.1f} ms")
