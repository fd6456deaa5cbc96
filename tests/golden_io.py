"""Loading helpers for the reference-generated fixtures in tests/golden/."""

import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def to_config(net, symbols_cls=None):
    """Golden flat net -> this repo's Configuration (original variable ids)."""
    from inet.core import Agent, Configuration, Equation, Symbol, Var

    syms = [Symbol(n, a) for n, a in net["symbols"]]
    recs = net["agents"]
    built = [None] * len(recs)
    # golden agents are in post-order: children precede parents
    for i, rec in enumerate(recs):
        kids = tuple(Var(-(x + 1)) if x < 0 else built[x] for x in rec[1:])
        built[i] = Agent(syms[rec[0]], kids)
    term = lambda r: Var(-(r + 1)) if r < 0 else built[r]
    return Configuration(tuple(term(r) for r in net["interface"]),
                         tuple(Equation(term(l), term(r)) for l, r in net["equations"]))


def to_rules(rs):
    """Golden flat rule set -> this repo's RuleSet."""
    from inet.core import Agent, Equation, Rule, RuleSet, Symbol, Var

    syms = {n: Symbol(n, a) for n, a in rs["symbols"]}
    names = [n for n, _ in rs["symbols"]]
    out = RuleSet()
    for n in names:
        out.declare(syms[n])
    for r in rs["rules"]:
        built = []
        for rec in r["agents"]:
            built.append(Agent(syms[names[rec[0]]], tuple(Var(-(x + 1)) if x < 0 else built[x] for x in rec[1:])))
        term = lambda x: Var(-(x + 1)) if x < 0 else built[x]
        rhs = tuple(Equation(term(l), term(rr)) for l, rr in r["rhs"])
        out.add(Rule(syms[r["a"]], tuple(r["a_vars"]), syms[r["b"]], tuple(r["b_vars"]), rhs))
    return out
