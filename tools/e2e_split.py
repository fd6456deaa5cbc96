"""Where the C-ABI e2e step of the headline batch goes (load / reduce+fetch / finalize / result), warm."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
prep = engine.prepare([p.build_input(3, 6)] * 4096, p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
k = engine.native_cfg(EngineConfig(collect_stats=False))
for it in range(6):
    t = [time.perf_counter()]
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    t.append(time.perf_counter())
    code, ms = ctx.reduce(k)
    t.append(time.perf_counter())
    ctx.finalize(0xFFFFFFFF, 0)
    t.append(time.perf_counter())
    ctx.result(0)
    t.append(time.perf_counter())
    d = [1e3 * (t[i + 1] - t[i]) for i in range(4)]
    print(f"device {ms:.2f} ms | load {d[0]:.2f} reduce+fetch {d[1]:.2f} finalize {d[2]:.2f} result {d[3]:.2f} "
          f"total {sum(d):.2f} | io {ctx.io_bytes()}", flush=True)
