"""Tier R — the reference's equation list, in its order — against the reference.

The fast tiers reproduce every schedule-free output (interaction counts,
normal forms) and, for nets that never equate two variables, the loop rows
too. Tier R (paper_1404_0076_b200/csrc/ordered.cuh) reproduces the rest of
what engine.py:106-166 decides by its list order: which variable keys a
var = var equation (engine.py:150-153) and therefore total_communications and
every LoopStats row, the orientation of a merged pair (engine.py:161-165), the
first failing pair (engine.py:88-92), and the residual order that decides
where finalize cuts a cycle (engine.py:313-355). Here every fixture the
reference produced (tests/golden/) must match in all of them.
"""

import hashlib

import pytest

from golden_io import load, to_config, to_rules
from oracle import oracle as O
from paper_1404_0076_b200 import (
    Agent,
    Configuration,
    EngineConfig,
    Equation,
    Symbol,
    Var,
    _native,
    evaluate,
    evaluate_batch,
    parse_program,
    print_configuration,
)
from paper_1404_0076_b200 import errors
from paper_1404_0076_b200._ref import bench as programs

pytestmark = pytest.mark.gpu

PROGRAMS = load("programs.json")
CASES = load("cases.json")
ARITH = load("arith.json")


def _sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def _rows(res):
    return [[s.interactions, s.communications, s.live_equations] for s in res.loops]


def _inputs(case):
    if "program" in case:
        prog = programs.program(case["program"])
        return prog.build_input(*case["params"]), prog.rules
    if "source" in case:
        sp = parse_program(case["source"])
        return sp.net, sp.rules
    return to_config(case["net"]), to_rules(PROGRAMS["arith"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_fixture_everything_equal(case):
    config, rules = _inputs(case)
    cfg = EngineConfig(reference_order=True, **case.get("engine_config", {}))
    if "error" in case:
        with pytest.raises(getattr(errors, case["error"])) as ei:
            evaluate(config, rules, cfg)
        if case.get("error_pair"):
            assert list(ei.value.pair) == case["error_pair"]
        return
    res = evaluate(config, rules, cfg)
    assert res.total_interactions == case["interactions"]
    assert res.total_communications == case["communications"]
    assert _rows(res) == case["loops"]
    assert _sha(print_configuration(res.final)) == case["print_sha256"]
    assert _native.context(0).stats(0).tier == _native.TIER_R


def test_arith_551_nets_everything_equal():
    rules = to_rules(PROGRAMS["arith"])
    configs = [to_config(c["net"]) for c in ARITH]
    out = evaluate_batch(configs, rules, EngineConfig(collect_stats=True, reference_order=True), as_text=True)
    for case, res, text in zip(ARITH, out.results, out.texts):
        assert res.total_interactions == case["interactions"], case["name"]
        assert res.total_communications == case["communications"], case["name"]
        assert _rows(res) == case["loops"], case["name"]
        assert _sha(text) == case["print_sha256"], case["name"]


def test_fib18_default_is_reference_exact_and_repeatable():
    """Fibonacci equates variables (Add >< Z => r = y): evaluate() keys var = var
    equations by the reference's variable ids (stamps on tier M) and gives
    1,667 loops and 47,912 communications on every run."""
    prog = programs.program("fibonacci")
    runs = [evaluate(prog.build_input(18), prog.rules) for _ in range(3)]
    st = _native.context(0).stats(0)
    assert st.tier == _native.TIER_M, "the stamped fast tier, not a tier R rerun"
    for res in runs:
        assert res.total_interactions == 50_515
        assert res.total_communications == 47_912
        assert len(res.loops) == 1_667
        assert programs.nat_value(res.final.interface[0]) == 2584
    assert _rows(runs[0]) == _rows(runs[1]) == _rows(runs[2])
    want = O.run_config(prog.build_input(18), O.rules_for("fibonacci"), collect=True)
    assert _rows(runs[0]) == [list(r) for r in want.rows]


def test_stamped_fast_tiers_against_every_fixture():
    """Single-CTA tiers with reference-ordered var = var keys: every fixture and
    the 551 random nets equal in everything, or stopped with INET_ERR_ORDER
    (then tier R decides, as the default policy does)."""
    from paper_1404_0076_b200 import engine

    ctx = _native.context(0)
    undecided = 0
    cases = [c for c in CASES if "error" not in c]
    for case in cases:
        config, rules = _inputs(case)
        prep = engine.prepare([config], rules)
        with ctx.lock:
            outs, _ = engine._reduce(ctx, prep, EngineConfig(**case.get("engine_config", {})), engine.MODE_STAMPS,
                                     True, True)
        o = outs[0]
        if o.stats.status == _native.ORDER:
            undecided += 1
            continue
        assert o.stats.status == _native.OK, case["name"]
        assert o.stats.interactions == case["interactions"], case["name"]
        assert o.stats.communications == case["communications"], case["name"]
        assert [list(r[:3]) for r in o.rows] == case["loops"], case["name"]
        assert _sha(o.text) == case["print_sha256"], case["name"]
    rules = to_rules(PROGRAMS["arith"])
    prep = engine.prepare([to_config(c["net"]) for c in ARITH], rules)
    with ctx.lock:
        outs, _ = engine._reduce(ctx, prep, EngineConfig(), engine.MODE_STAMPS, False, True)
    for case, o in zip(ARITH, outs):
        if o.stats.status == _native.ORDER:
            undecided += 1
            continue
        assert o.stats.communications == case["communications"], case["name"]
        assert [list(r[:3]) for r in o.rows] == case["loops"], case["name"]
        assert _sha(o.text) == case["print_sha256"], case["name"]
    assert undecided < (len(cases) + len(ARITH)) // 4


def test_fast_tiers_remain_available():
    prog = programs.program("fibonacci")
    res = evaluate(prog.build_input(18), prog.rules, EngineConfig(reference_order=False))
    assert res.total_interactions == 50_515
    assert _native.context(0).stats(0).tier != _native.TIER_R


def test_merge_formed_no_rule_pair_keeps_the_list_orientation():
    """x = A and C = x merge into A = C (list order), C = x and x = A into C = A;
    the pair has no rule: NoRuleForPair carries the merged orientation."""
    a, b, c = Symbol("A", 0), Symbol("B", 0), Symbol("C", 0)
    rules = parse_program("A >< B => ;\nnet : A = B;").rules
    rules.declare(c)
    x = Var(0)
    one = Configuration((), (Equation(x, Agent(a)), Equation(Agent(c), x)))
    two = Configuration((), (Equation(Agent(c), x), Equation(x, Agent(a))))
    for net, pair in ((one, ("A", "C")), (two, ("C", "A"))):
        for order in (None, True):  # default: the fast run fails, tier R reruns it
            with pytest.raises(errors.NoRuleForPair) as ei:
                evaluate(net, rules, EngineConfig(reference_order=order))
            assert ei.value.pair == pair
    del b


def test_first_failing_pair_in_list_order():
    rules = parse_program("A >< B => ;\nnet : A = B;").rules
    for s in ("C", "D", "E"):
        rules.declare(Symbol(s, 0))
    sy = rules.symbols
    net = Configuration((), (Equation(Agent(sy["A"]), Agent(sy["B"])), Equation(Agent(sy["D"]), Agent(sy["E"])),
                             Equation(Agent(sy["C"]), Agent(sy["A"]))))
    with pytest.raises(errors.NoRuleForPair) as ei:
        evaluate(net, rules)
    assert ei.value.pair == ("D", "E")


def test_validate_phases_checks_every_phase_on_the_device():
    z = Agent(Symbol("Z", 0))
    rules = programs.load_rules("addition")
    bad = Configuration((), (Equation(Var(7), z), Equation(Var(7), z), Equation(Var(7), z)))
    with pytest.raises(errors.NameDisciplineError) as ei:
        evaluate(bad, rules, EngineConfig(validate_phases=True))
    assert "variable 7 occurs more than twice" in str(ei.value)
    # without the flag the reference does not check (engine.py:210-214)
    prog = programs.program("ackermann")
    plain = evaluate(prog.build_input(2, 3), prog.rules)
    checked = evaluate(prog.build_input(2, 3), prog.rules, EngineConfig(validate_phases=True))
    assert print_configuration(plain.final) == print_configuration(checked.final)
    assert _rows(plain) == _rows(checked)


def test_asymmetric_same_symbol_rule_follows_the_merge_orientation():
    """P(a, b) >< P(c, d) => a = Q(c), b = d: not symmetric. A P = P pair formed
    by a merge is applied in the list's orientation, like the reference."""
    src = ("P(a, b) >< P(c, d) => a = Q(c), b = d;\n"
           "net r, s, t, u : x = P(r, s), P(t, u) = x;")
    sp = parse_program(src)
    want = O.run_config(sp.net, O.compile_golden_rules(_golden_rules(sp.rules)), collect=True)
    res = evaluate(sp.net, sp.rules)
    assert print_configuration(res.final) == want.printed()
    assert res.total_interactions == want.interactions
    with pytest.raises(errors.UnsupportedNet):
        evaluate(sp.net, sp.rules, EngineConfig(reference_order=False))


def _golden_rules(rules):
    import fuzz_gen as F

    return F.to_golden(rules)


def test_tier_r_batch_reproducible_ids():
    """Deterministic allocation: two runs give identical flat normal forms."""
    prog = programs.program("fibonacci")
    nets = [prog.build_input(n) for n in (5, 9, 12)]
    one = evaluate_batch(nets, prog.rules, EngineConfig(reference_order=True), as_text=True)
    two = evaluate_batch(nets, prog.rules, EngineConfig(reference_order=True), as_text=True)
    assert one.texts == two.texts
    assert [r.total_communications for r in one.results] == [r.total_communications for r in two.results]
