"""Generate the parity fixtures under tests/golden/ by running the REFERENCE.

This script is the only place that imports the reference package
(``/root/reference/pkg/src/inet``). It runs in the build container only; the
JSON it writes travels with the repo so the GPU-box tests never need the
reference.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Fixture encoding (flat, so deep successor towers never hit JSON recursion):

* a *net* is ``{"symbols": [[name, arity], ...], "agents": [[label, ref...], ...],
  "interface": [ref, ...], "equations": [[ref, ref], ...]}`` where ``ref >= 0`` is
  an agent index and ``ref < 0`` is variable ``-(ref + 1)``;
* a *rule set* is ``{"symbols": [...], "rules": [{"a": name, "a_vars": [...],
  "b": name, "b_vars": [...], "rhs": flat-net-without-interface}]}``;
* an *outcome* is the reference's ``EvalResult`` reduced to ``print`` (the
  canonical text of ``print_configuration(final)``, or its sha256/length when
  long), ``interactions``, ``communications`` and ``loops`` (per-loop
  ``[interactions, communications, live_equations]``).

References: engine ``evaluate`` src/inet/engine.py:186-228, printer
src/inet/lang.py:371-396, programs src/inet/bench.py:270-342, random nets
tests/netgen.py:62-96.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
for p in (REF_SRC, REF_TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

from inet import errors as ref_errors  # noqa: E402
from inet.bench import program  # noqa: E402
from inet.core import Agent, Var  # noqa: E402
from inet.engine import EngineConfig, evaluate  # noqa: E402
from inet.lang import parse_program, print_configuration  # noqa: E402

import netgen  # noqa: E402  (reference test helper: random arith nets)

TEXT_LIMIT = 4096


class _Flat:
    def __init__(self, symbols):
        self.labels = {name: i for i, name in enumerate(symbols)}
        self.agents: list[list[int]] = []

    def ref(self, term) -> int:
        # iterative post-order so deep towers are fine
        out = {}
        stack = [(term, False)]
        while stack:
            t, done = stack.pop()
            if type(t) is Var:
                out[id(t)] = -(t.id + 1)
                continue
            if done:
                rec = [self.labels[t.sym.name]] + [out[id(c)] for c in t.children]
                self.agents.append(rec)
                out[id(t)] = len(self.agents) - 1
            else:
                stack.append((t, True))
                for c in t.children:
                    stack.append((c, False))
        return out[id(term)]


def symbols_of(rules, config=None):
    names = list(rules.symbols.keys())
    syms = {n: s.arity for n, s in rules.symbols.items()}
    if config is not None:
        for t in list(config.interface) + [s for e in config.equations for s in (e.lhs, e.rhs)]:
            stack = [t]
            while stack:
                x = stack.pop()
                if type(x) is Agent:
                    if x.sym.name not in syms:
                        syms[x.sym.name] = x.sym.arity
                        names.append(x.sym.name)
                    stack.extend(x.children)
    return [[n, syms[n]] for n in names]


def flat_net(config, symbols):
    f = _Flat([s[0] for s in symbols])
    iface = [f.ref(t) for t in config.interface]
    eqs = [[f.ref(e.lhs), f.ref(e.rhs)] for e in config.equations]
    return {"symbols": symbols, "agents": f.agents, "interface": iface, "equations": eqs}


def flat_rules(rules):
    symbols = symbols_of(rules)
    out = []
    for rule in rules.rules.values():
        f = _Flat([s[0] for s in symbols])
        rhs = [[f.ref(e.lhs), f.ref(e.rhs)] for e in rule.rhs]
        out.append(
            {
                "a": rule.lhs_a.name,
                "a_vars": list(rule.a_vars),
                "b": rule.lhs_b.name,
                "b_vars": list(rule.b_vars),
                "agents": f.agents,
                "rhs": rhs,
                "bound_vars": list(rule.bound_vars),
            }
        )
    return {"symbols": symbols, "rules": out, "max_rhs_size": rules.max_rhs_size,
            "max_fresh": rules.max_fresh}


def outcome(result, keep_final=True):
    text = print_configuration(result.final)
    rec = {
        "interactions": result.total_interactions,
        "communications": result.total_communications,
        "loops": [[s.interactions, s.communications, s.live_equations] for s in result.loops],
        "print_len": len(text),
        "print_sha256": hashlib.sha256(text.encode()).hexdigest(),
    }
    if len(text) <= TEXT_LIMIT:
        rec["print"] = text
    if keep_final and len(text) <= TEXT_LIMIT:
        rec["final"] = flat_net(result.final, symbols_of_config(result.final))
    return rec


def symbols_of_config(config):
    names, seen = [], {}
    for t in list(config.interface) + [s for e in config.equations for s in (e.lhs, e.rhs)]:
        stack = [t]
        while stack:
            x = stack.pop()
            if type(x) is Agent:
                if x.sym.name not in seen:
                    seen[x.sym.name] = x.sym.arity
                    names.append(x.sym.name)
                stack.extend(x.children)
    return [[n, seen[n]] for n in names]


def run_case(name, config, rules, cfg=None, keep_final=True):
    symbols = symbols_of(rules, config)
    case = {"name": name, "net": flat_net(config, symbols)}
    t0 = time.perf_counter()
    try:
        res = evaluate(config, rules, cfg)
    except ref_errors.InetError as exc:
        case["error"] = type(exc).__name__
        case["error_pair"] = list(getattr(exc, "pair", ()) or ())
        return case
    case["wall_s"] = round(time.perf_counter() - t0, 4)
    case.update(outcome(res, keep_final))
    return case


ADD_RULES = """
Add(r,y) >< S(x) => Add(w,y)=x, r=S(w);
Add(r,y) >< Z => r=y;
"""


def chain_program(i):
    vs = [f"v{k}" for k in range(1, i + 1)]
    eqs = [f"A = {vs[0]}"] + [f"{vs[k]} = {vs[k + 1]}" for k in range(i - 1)] + [f"{vs[-1]} = B"]
    return "A >< B => ;\nnet : " + ", ".join(eqs) + ";"


def main():
    programs = {}
    for name in ("addition", "ackermann", "fibonacci", "lsystem", "arith"):
        from inet.bench import load_rules
        programs[name] = flat_rules(load_rules(name))
    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(programs, fh, indent=0, separators=(",", ":"))

    cases = []
    # benchmark programs (inputs built by the reference builders)
    bench_params = {
        "addition": [(1, 0), (0, 0), (3, 4), (7, 5), (2, 2)],
        "ackermann": [(2, 2), (2, 3), (3, 1), (3, 2), (3, 3), (3, 4), (3, 5), (3, 6)],
        "fibonacci": [(7,), (10,), (12,), (15,), (18,)],
        "lsystem": [(4,), (5,), (10,), (12,), (20,)],
    }
    for pname, plist in bench_params.items():
        prog = program(pname)
        for params in plist:
            cfg = prog.build_input(*params)
            case = run_case(f"{pname}{params}", cfg, prog.rules)
            case["program"] = pname
            case["params"] = list(params)
            cases.append(case)
            print(case["name"], case.get("interactions"), case.get("wall_s"), flush=True)

    # literal programs from the reference tests
    literal = [
        ("add_1_0", ADD_RULES + "net r : Add(r, Z) = S(Z);", None),
        ("add_1_0_1", ADD_RULES + "net r : Add(r, w) = S(Z), Add(w, S(Z)) = Z;", None),
        ("add_2_3", ADD_RULES + "net r : Add(r, S(S(Z))) = S(S(S(Z)));", None),
        ("no_rule", ADD_RULES + "net r : S(Z) = S(Z);", None),
        ("loop_cap", "Loop >< Z => Loop = Z;\nnet : Loop = Z;", {"max_loops": 5}),
        ("free_iface", "A >< B => ;\nnet x, y : A = B;", None),
        ("var_var_only", "A >< B => ;\nnet x : x = y, y = z, z = A;", None),
        ("cycle", "A >< B => ;\nnet : x = C(y), y = C(x);", None),
        ("self_loop", "A >< B => ;\nnet : x = x;", None),
        ("deadlock_aux", "A >< B => ;\nnet r : r = C(x), x = A;", None),
    ]
    for i in range(1, 11):
        literal.append((f"chain_{i}", chain_program(i), None))
    for name, src, kw in literal:
        try:
            sp = parse_program(src)
        except ref_errors.InetError as exc:
            print("skip", name, exc)
            continue
        cfg = EngineConfig(**kw) if kw else None
        case = run_case(name, sp.net, sp.rules, cfg)
        case["source"] = src
        case["rules"] = flat_rules(sp.rules)
        if kw:
            case["engine_config"] = kw
        cases.append(case)
        print(name, case.get("interactions"), case.get("error"), flush=True)

    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))

    # 500 random arith nets (reference differential fixture, tests/test_acceptance.py:114-122)
    rules = netgen.arith_rules()
    arith = []
    for seed in range(500):
        cfg = netgen.random_config(random.Random(seed), rules)
        case = run_case(f"arith_seed{seed}", cfg, rules)
        case["seed"] = seed
        arith.append(case)
    cfg = netgen.random_config(random.Random(99), rules, max_agents=60)
    case = run_case("arith_seed99_max60", cfg, rules)
    arith.append(case)
    for seed in range(50):
        cfg = netgen.random_two_active(random.Random(seed), rules)
        case = run_case(f"two_active_seed{seed}", cfg, rules)
        arith.append(case)
    with open(os.path.join(HERE, "arith.json"), "w") as fh:
        json.dump(arith, fh, separators=(",", ":"))
    print("arith cases", len(arith))


if __name__ == "__main__":
    main()
