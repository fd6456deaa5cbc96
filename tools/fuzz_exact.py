"""Long differential fuzz of the default evaluation policy (development).

Random rule sets x random nets through evaluate_batch / evaluate with the
default ``EngineConfig`` (stamped fast tiers for rule sets that equate
variables, tier R where stamps cannot decide, exactness reruns), against the
oracle, which follows the reference's list order: interaction and
communication totals, every LoopStats row and the printed normal form must be
byte-identical — no isomorphism fallback.

usage: python tools/fuzz_exact.py [n_seeds] [budget_s] [first_seed]
"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1404_0076_b200  # noqa: E402,F401  (the reference package `inet` on the path)
import fuzz_gen as F  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1404_0076_b200 import EngineConfig, evaluate, evaluate_batch, print_configuration  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
budget_s = float(sys.argv[2]) if len(sys.argv) > 2 else 300
base = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
t0 = time.time()
stats = {"rule_sets": 0, "nets": 0, "exact": 0, "bad": 0, "single": 0, "cyclic": 0}


def rows(res):
    return [(s.interactions, s.communications, s.live_equations) for s in res.loops]


for seed in range(base, base + seeds):
    if time.time() - t0 > budget_s:
        break
    rng = random.Random(seed)
    syms = F.random_signature(rng)
    rules = F.random_rules(rng, syms)
    orules = O.compile_golden_rules(F.to_golden(rules))
    nets = [F.random_net(rng, syms, rng.randint(1, 60), rng.randint(1, 6)) for _ in range(300)]
    out = evaluate_batch(nets, rules, EngineConfig(collect_stats=True), as_text=True)
    stats["rule_sets"] += 1
    for i, (net, res, text) in enumerate(zip(nets, out.results, out.texts)):
        want = O.run_config(net, orules, collect=True)
        stats["nets"] += 1
        ok = (res.total_interactions == want.interactions and res.total_communications == want.communications
              and rows(res) == [tuple(r) for r in want.rows] and text == want.printed())
        stats["exact" if ok else "bad"] += 1
        stats["cyclic"] += " = " in text
        if not ok:
            print("MISMATCH", seed, i, res.total_interactions, want.interactions, res.total_communications,
                  want.communications, len(res.loops), len(want.rows), flush=True)
    for ctas in (0, 1):  # bigger single nets (auto tiers, one CTA)
        net = F.random_net(rng, syms, 150, 6)
        want = O.run_config(net, orules, collect=True)
        res = evaluate(net, rules, EngineConfig(ctas_per_net=ctas))
        stats["single"] += 1
        ok = (res.total_interactions == want.interactions and res.total_communications == want.communications
              and rows(res) == [tuple(r) for r in want.rows] and print_configuration(res.final) == want.printed())
        if not ok:
            stats["bad"] += 1
            print("SINGLE MISMATCH", seed, ctas, flush=True)
    print("seed", seed, stats, f"{time.time() - t0:.0f} s", flush=True)
print("fuzz summary", stats, f"{time.time() - t0:.0f} s", flush=True)
