"""Per-loop LoopStats rows of the device (exact_loops=True) against the oracle
(the reference algorithm restated) for the large Ackermann configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1404_0076_b200 import EngineConfig, evaluate, print_configuration  # noqa: E402
from inet.bench import program  # noqa: E402

p = program("ackermann")
for n in [int(x) for x in (sys.argv[1:] or ["8", "10"])]:
    cfg = p.build_input(3, n)
    t0 = time.time()
    want = O.run_config(cfg, O.rules_for("ackermann"), collect=True)
    t1 = time.time()
    res = evaluate(cfg, p.rules, EngineConfig(collect_stats=True, exact_loops=True))
    t2 = time.time()
    got = [[s.interactions, s.communications, s.live_equations] for s in res.loops]
    same_rows = got == want.rows
    first_diff = next((i for i, (a, b) in enumerate(zip(got, want.rows)) if a != b), None)
    print(f"A(3,{n}): loops {len(got)} vs {len(want.rows)}, rows identical: {same_rows} (first diff {first_diff}), "
          f"interactions {res.total_interactions} vs {want.interactions}, communications {res.total_communications} "
          f"vs {want.communications}, normal form identical: {print_configuration(res.final) == want.printed()}; "
          f"oracle {t1 - t0:.1f} s, device run {t2 - t1:.2f} s", flush=True)
