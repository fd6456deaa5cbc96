"""Where the end-to-end time of the 4096 x A(3,6) batch goes (load / reduce / finalize)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402
p = program("ackermann")
prep = engine.prepare([p.build_input(3, 6) for _ in range(4096)], p.rules)
ctx = _native.Context(0)
ctx.load_rules(prep.blob)
k = engine.native_cfg(EngineConfig(collect_stats=False))
for it in range(4):
    t0 = time.perf_counter()
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    t1 = time.perf_counter()
    code, ms = ctx.reduce(k)
    t2 = time.perf_counter()
    ctx.finalize(0xFFFFFFFF, 0)
    t3 = time.perf_counter()
    a0, _, _ = ctx.result(0)
    t4 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  reduce {1e3*(t2-t1):.2f} ms (kernel {ms:.2f})  finalize {1e3*(t3-t2):.2f} ms  "
          f"result {1e3*(t4-t3):.3f} ms  io {ctx.io_bytes()}")
