"""Tier C (cluster) sweep: parity of the printed normal form and device time per (G, threads, jit)."""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, _native, engine, evaluate, print_configuration  # noqa: E402
from inet.bench import program  # noqa: E402

WL = {"a23": ("ackermann", (2, 3), 90, "829772e6f0876f88"), "fib18": ("fibonacci", (18,), 50515, "0feb32862e23b545"),
      "a36": ("ackermann", (3, 6), 344964, "47b60c6a324411a9"), "a38": ("ackermann", (3, 8), 5574030, "b85606c71178de4b"),
      "a310": ("ackermann", (3, 10), 89404824, "981fd9bfe283f466"),
      "ls20": ("lsystem", (20,), 57290, ""), "ls24": ("lsystem", (24,), 0, ""), "ls26": ("lsystem", (26,), 0, "")}
ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="a23,fib18,a36,a38,a310")
ap.add_argument("--gs", default="1,2,4,8,16")
ap.add_argument("--threads", default="512")
ap.add_argument("--jit", default="1")
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--check", type=int, default=1)
a = ap.parse_args()
for w in a.workloads.split(","):
    name, params, ints, sha = WL[w]
    p = program(name)
    cfg0 = p.build_input(*params)
    prep = engine.prepare([cfg0], p.rules)
    for jit in [int(x) for x in a.jit.split(",")]:
        os.environ["INET_B200_JIT"] = str(jit)
        for g in [int(x) for x in a.gs.split(",")]:
            for t in [int(x) for x in a.threads.split(",")]:
                ok = "-"
                if a.check:
                    res = evaluate(cfg0, p.rules, EngineConfig(ctas_per_net=g, threads=t))
                    h = hashlib.sha256(print_configuration(res.final).encode()).hexdigest()
                    ok = "OK" if ((not ints or res.total_interactions == ints) and h.startswith(sha)) else f"BAD {res.total_interactions} {h[:16]}"
                    ok += f" loops={len(res.loops)} sum={sum(s.interactions for s in res.loops)}"
                ctx = _native.Context(0)
                ctx.set_jit(bool(jit))
                ctx.load_rules(prep.blob)
                ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
                k = engine.native_cfg(EngineConfig(collect_stats=False, threads=t, ctas_per_net=g))
                best = 1e30
                for _ in range(a.repeat):
                    code, ms = ctx.reduce(k)
                    best = min(best, ms)
                st = ctx.stats(0)
                tot = ctx.totals()
                print(f"{w:6s} jit={jit} G={g:2d} t={t:4d} code={code} tier={st.tier} ms={best:9.3f} "
                      f"Mips={tot[0] / best / 1e3:8.1f} rounds={tot[2]} us/round={best * 1e3 / max(tot[2], 1):6.3f} "
                      f"hw={st.agent_hw},{st.var_hw} MHz={st.sm_mhz} {ok}", flush=True)
