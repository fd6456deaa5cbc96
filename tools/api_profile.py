"""cProfile of evaluate_batch(as_text=True) on the headline batch (4096 x A(3,6)), warm (development)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, engine  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
nets = [p.build_input(3, 6) for _ in range(4096)]
cfg = EngineConfig(collect_stats=False)
for _ in range(3):
    t0 = time.perf_counter()
    engine.evaluate_batch(nets, p.rules, cfg, as_terms=False, as_text=True)
    print(f"evaluate_batch {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
engine.evaluate_batch(nets, p.rules, cfg, as_terms=False, as_text=True)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
