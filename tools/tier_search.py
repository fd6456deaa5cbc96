"""Which tier attempts a single net goes through (INET_B200_DEBUG=1 prints each)."""
import os
import sys
import time

os.environ.setdefault("INET_B200_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, evaluate_text  # noqa: E402
from inet.bench import program  # noqa: E402

for name, params in (("lsystem", (26,)), ("lsystem", (24,)), ("ackermann", (3, 10))):
    p = program(name)
    cfg = p.build_input(*params)
    for _ in range(2):
        t0 = time.perf_counter()
        evaluate_text(cfg, p.rules, EngineConfig(collect_stats=False))
        print(f"{name}{params}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
