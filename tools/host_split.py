"""Host-side split of one single-net evaluate_text (prepare / reduce / finalize / print)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

for name, params in (("lsystem", (26,)), ("ackermann", (3, 10))):
    p = program(name)
    cfg = p.build_input(*params)
    ctx = _native.context(0)
    ec = EngineConfig(collect_stats=False)
    for it in range(3):
        t0 = time.perf_counter()
        prep = engine.prepare([cfg], p.rules)
        t1 = time.perf_counter()
        code, ms = engine.run_prepared(ctx, prep, ec)
        t2 = time.perf_counter()
        ctx.finalize(0xFFFFFFFF, 0)
        t3 = time.perf_counter()
        text = ctx.text(0, engine.label_table(prep.labels))
        t4 = time.perf_counter()
        st = ctx.stats(0)
        print(f"{name}{params}: prepare {1e3*(t1-t0):.2f} reduce {1e3*(t2-t1):.2f} (device {ms:.2f}) "
              f"finalize {1e3*(t3-t2):.2f} print {1e3*(t4-t3):.2f} ms; agent_hw {st.agent_hw} residual {st.n_residual} "
              f"text {len(text)}", flush=True)
