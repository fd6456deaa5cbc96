"""Where evaluate_batch's time goes for the headline batch (4096 x A(3,6)), stage by stage."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
nets = [p.build_input(3, 6) for _ in range(4096)]
cfg = EngineConfig(collect_stats=False)
ctx = _native.context(0)
for it in range(3):
    t = [time.perf_counter()]
    prep = engine.prepare(nets, p.rules)
    t.append(time.perf_counter())
    ctx.load_rules(prep.blob, key=prep.blob.tobytes())
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    t.append(time.perf_counter())
    code, ms = ctx.reduce(engine.native_cfg(cfg))
    t.append(time.perf_counter())
    st = ctx.stats_all(len(nets))
    t.append(time.perf_counter())
    ctx.finalize(0xFFFFFFFF, 0)
    t.append(time.perf_counter())
    counts = ctx.result_counts_all(len(nets))
    t.append(time.perf_counter())
    texts = ctx.texts(len(nets), engine.label_table(prep.labels))
    t.append(time.perf_counter())
    out = engine.evaluate_batch(nets, p.rules, cfg, as_terms=False, as_text=True)
    t.append(time.perf_counter())
    names = ["prepare", "load", "reduce", "stats_all", "finalize", "counts", "texts", "evaluate_batch total"]
    d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
    print(f"iter {it}: device {ms:.2f} ms; " + ", ".join(f"{n} {x:.2f}" for n, x in zip(names, d)), flush=True)
