"""End to end of a single net with a large normal form: Python terms + Python
printer (evaluate + print_configuration) against the native printer (evaluate_text)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, evaluate, evaluate_text, print_configuration  # noqa: E402
from inet.bench import program  # noqa: E402

for name, params in (("ackermann", (3, 10)), ("lsystem", (26,)), ("ackermann", (3, 8))):
    p = program(name)
    cfg = p.build_input(*params)
    ec = EngineConfig(collect_stats=False)
    evaluate_text(cfg, p.rules, ec)  # warm (JIT, buffers)
    t0 = time.perf_counter()
    res = evaluate(cfg, p.rules, ec)
    t1 = time.perf_counter()
    py_text = print_configuration(res.final)
    t2 = time.perf_counter()
    text, ints, _ = evaluate_text(cfg, p.rules, ec)
    t3 = time.perf_counter()
    assert text == py_text and ints == res.total_interactions
    print(f"{name}{params}: evaluate {1e3 * (t1 - t0):.1f} ms + print_configuration {1e3 * (t2 - t1):.1f} ms "
          f"= {1e3 * (t2 - t0):.1f} ms; evaluate_text {1e3 * (t3 - t2):.1f} ms; text {len(text)} bytes", flush=True)
