"""Long differential fuzz (development): many random rule sets x random nets,
engine (batch tier S and single-net tiers) against the oracle. Prints a
summary and every mismatch."""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import fuzz_gen as F  # noqa: E402
from netgraph import canonical  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1404_0076_b200 import EngineConfig, evaluate, evaluate_batch, print_configuration  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
budget_s = float(sys.argv[2]) if len(sys.argv) > 2 else 300
t0 = time.time()
stats = {"nets": 0, "exact": 0, "graph": 0, "bad": 0, "single": 0}
base = int(sys.argv[3]) if len(sys.argv) > 3 else 100
for seed in range(base, base + seeds):
    if time.time() - t0 > budget_s:
        break
    rng = random.Random(seed)
    syms = F.random_signature(rng)
    rules = F.random_rules(rng, syms)
    orules = O.compile_golden_rules(F.to_golden(rules))
    nets = [F.random_net(rng, syms, rng.randint(1, 60), rng.randint(1, 6)) for _ in range(300)]
    out = evaluate_batch(nets, rules, EngineConfig(collect_stats=False), as_text=True)
    for i, (net, res, text) in enumerate(zip(nets, out.results, out.texts)):
        want = O.run_config(net, orules, collect=False)
        stats["nets"] += 1
        wt = want.printed()
        if res.total_interactions != want.interactions:
            stats["bad"] += 1
            print("INTERACTIONS", seed, i, res.total_interactions, want.interactions, flush=True)
        elif text == wt:
            stats["exact"] += 1
        elif " = " in wt and canonical(res.final) == canonical(want.final_config()):
            stats["graph"] += 1
        else:
            stats["bad"] += 1
            print("NORMAL FORM", seed, i, flush=True)
    # a few bigger single nets through the single-net tiers
    for ctas in (0, 16, 148):
        net = F.random_net(rng, syms, 150, 6)
        want = O.run_config(net, orules, collect=False)
        res = evaluate(net, rules, EngineConfig(collect_stats=False, ctas_per_net=ctas))
        stats["single"] += 1
        text = print_configuration(res.final)
        ok = res.total_interactions == want.interactions and (
            text == want.printed() or canonical(res.final) == canonical(want.final_config()))
        if not ok:
            stats["bad"] += 1
            print("SINGLE", seed, ctas, res.total_interactions, want.interactions, flush=True)
    print("seed", seed, stats, f"{time.time() - t0:.0f} s", flush=True)
print("fuzz summary", stats, f"{time.time() - t0:.0f} s", flush=True)
