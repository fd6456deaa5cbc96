"""Differential fuzz over random rule sets.

CPU part: the generated rule sets are well-formed for the reference's rule
checks (core.Rule), compile into rule blobs, and the rule-set compiler
(NVRTC, sm_100a) accepts their specialised kernels. GPU part: the engine and
the oracle agree on interaction counts and printed normal forms for batches
of random nets over each random rule set, and for the single-net tiers.
"""

import random
import pytest

import fuzz_gen as F
from netgraph import canonical
from oracle import oracle as O
from paper_1404_0076_b200 import EngineConfig, _native, engine, evaluate, evaluate_batch, print_configuration

SEEDS = list(range(8))


def _same_normal_form(text, final, want):
    """Byte-identical text, or — when the normal form keeps cyclic equations —
    the same net (port-graph isomorphism, tests/netgraph.py).

    A normal form with surviving equations holds cycles of parked equations
    (vicious circles); finalize cuts each cycle where its elimination queue
    meets it, and the queue follows variable ids, which are the device's here
    and the reference's fresh-id blocks there.
    """
    want_text = want.printed()
    if text == want_text:
        return True
    if " = " not in want_text:
        return False
    return canonical(final) == canonical(want.final_config())


def _case(seed, n_nets=200):
    rng = random.Random(1000 + seed)
    syms = F.random_signature(rng)
    rules = F.random_rules(rng, syms)
    nets = [F.random_net(rng, syms, rng.randint(1, 40), rng.randint(1, 6)) for _ in range(n_nets)]
    return rules, nets


@pytest.mark.parametrize("seed", SEEDS[:3])
def test_random_rule_sets_compile(seed):
    rules, nets = _case(seed, 4)
    prep = engine.prepare(nets, rules)
    for tier, threads in ((0, 128), (3, 256)):
        code, log = _native.jit_compile(prep.blob, tier, threads)
        assert code == _native.OK, log[:2000]
    orules = O.compile_golden_rules(F.to_golden(rules))
    for net in nets:
        assert O.run_config(net, orules, collect=False).status == "ok"


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_random_rule_sets_batch_against_oracle(seed):
    rules, nets = _case(seed)
    orules = O.compile_golden_rules(F.to_golden(rules))
    # the fast tiers (these rule sets equate variables, so the default would pick tier R)
    out = evaluate_batch(nets, rules, EngineConfig(collect_stats=False, reference_order=False), as_text=True)
    exact = 0
    for i, (net, res, text) in enumerate(zip(nets, out.results, out.texts)):
        want = O.run_config(net, orules, collect=False)
        assert want.status == "ok"
        assert res.total_interactions == want.interactions, (seed, i)
        assert text == print_configuration(res.final)
        assert _same_normal_form(text, res.final, want), (seed, i)
        exact += text == want.printed()
    assert exact > 0


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:3])
@pytest.mark.parametrize("ctas", [1, 16, 148])
def test_random_rule_sets_single_net_tiers(seed, ctas):
    rules, nets = _case(seed, 12)
    orules = O.compile_golden_rules(F.to_golden(rules))
    for net in nets:
        want = O.run_config(net, orules, collect=False)
        res = evaluate(net, rules, EngineConfig(collect_stats=False, ctas_per_net=ctas, reference_order=False))
        text = print_configuration(res.final)
        assert res.total_interactions == want.interactions
        assert _same_normal_form(text, res.final, want)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_random_rule_sets_reference_order_byte_identical(seed):
    """The default policy for these rule sets, which equate variables (stamped
    fast tiers, tier R for what they cannot decide and for cyclic normal
    forms): every count, every loop row and every printed normal form —
    cyclic ones included — byte-identical to the oracle, which follows the
    reference's list order (no isomorphism fallback)."""
    rules, nets = _case(seed)
    orules = O.compile_golden_rules(F.to_golden(rules))
    out = evaluate_batch(nets, rules, EngineConfig(collect_stats=True), as_text=True)
    cyclic = 0
    for i, (net, res, text) in enumerate(zip(nets, out.results, out.texts)):
        want = O.run_config(net, orules, collect=True)
        assert res.total_interactions == want.interactions, (seed, i)
        assert res.total_communications == want.communications, (seed, i)
        assert [(s.interactions, s.communications, s.live_equations) for s in res.loops] == \
            [tuple(r) for r in want.rows], (seed, i)
        assert text == want.printed(), (seed, i)
        cyclic += " = " in text
    del cyclic


def test_netgraph_canonical_form():
    """The comparison itself: invariant under equation order and orientation,
    sensitive to a changed agent or a rewired port."""
    from inet.core import Agent, Configuration, Equation, Symbol, Var

    rng = random.Random(4)
    rules, nets = _case(0, 60)
    syms = list(rules.symbols.values())
    for net in nets:
        eqs = [Equation(e.rhs, e.lhs) if rng.random() < 0.5 else e for e in net.equations]
        rng.shuffle(eqs)
        assert canonical(net) == canonical(Configuration(net.interface, tuple(eqs)))
    s, z = Symbol("S", 1), Symbol("Z", 0)
    a = Configuration((Var(0),), (Equation(Var(0), Agent(s, (Agent(z),))),))
    b = Configuration((Var(0),), (Equation(Var(0), Agent(s, (Agent(s, (Agent(z),)),))),))
    assert canonical(a) != canonical(b)
    # a two-agent ring cut in two places is one net
    t = Symbol("T", 1)
    r1 = Configuration((), (Equation(Var(0), Agent(t, (Agent(s, (Var(0),)),))),))
    r2 = Configuration((), (Equation(Var(0), Agent(s, (Agent(t, (Var(0),)),))),))
    assert canonical(r1) == canonical(r2)
    assert print_configuration(r1) != print_configuration(r2)
    del syms
