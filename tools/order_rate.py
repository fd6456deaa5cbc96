"""How often the stamped fast tiers leave a var = var comparison to tier R (INET_ERR_ORDER)."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1404_0076_b200  # noqa: E402,F401  (the reference package `inet` on the path)
import fuzz_gen as F  # noqa: E402
from golden_io import load, to_config, to_rules  # noqa: E402
from paper_1404_0076_b200 import EngineConfig, _native, engine  # noqa: E402
from inet.bench import program  # noqa: E402

ctx = _native.context(0)


def rate(label, nets, rules):
    prep = engine.prepare(nets, rules)
    with ctx.lock:
        outs, _ = engine._reduce(ctx, prep, EngineConfig(collect_stats=False), engine.MODE_STAMPS, False, False)
    n_order = sum(o.stats.status == _native.ORDER for o in outs)
    print(f"{label}: {len(nets)} nets, {n_order} left to tier R ({100.0 * n_order / len(nets):.1f} %)", flush=True)


arith = load("arith.json")
rate("reference random arith nets (golden)", [to_config(c["net"]) for c in arith], to_rules(load("programs.json")["arith"]))
for name, params in (("fibonacci", [(n,) for n in range(2, 20)]), ("addition", [(a, b) for a in range(6) for b in range(6)])):
    p = program(name)
    rate(name, [p.build_input(*q) for q in params], p.rules)
for seed in range(6):
    rng = random.Random(1000 + seed)
    syms = F.random_signature(rng)
    rules = F.random_rules(rng, syms)
    nets = [F.random_net(rng, syms, rng.randint(1, 40), rng.randint(1, 6)) for _ in range(200)]
    rate(f"random rule set {seed}", nets, rules)
