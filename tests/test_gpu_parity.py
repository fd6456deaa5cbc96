"""GPU parity: the CUDA engine against the reference fixtures and the oracle.

Bar: the canonical printed normal form is byte-identical and
the total interaction count is identical. The per-round series is the
device's own (fixpoint linking per round), so only its invariants are checked.
"""

import hashlib
import random

import pytest

from golden_io import load, to_config, to_rules
from oracle import oracle as O
from paper_1404_0076_b200 import (
    Agent,
    Configuration,
    EngineConfig,
    Equation,
    Var,
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


def _case_inputs(case):
    if "program" in case:
        prog = programs.program(case["program"])
        return prog.build_input(*case["params"]), prog.rules
    if "source" in case:
        sp = parse_program(case["source"])
        return sp.net, sp.rules
    return to_config(case["net"]), to_rules(PROGRAMS["arith"])


def _check_loops(res):
    assert res.loops, "collect_stats=True must produce rows"
    assert sum(s.interactions for s in res.loops) == res.total_interactions
    assert sum(s.communications for s in res.loops) == res.total_communications
    assert (res.loops[-1].interactions, res.loops[-1].communications) == (0, 0)
    assert [s.loop_index for s in res.loops] == list(range(1, len(res.loops) + 1))
    if len(res.loops) >= 2:
        assert res.loops[-1].live_equations == res.loops[-2].live_equations


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reference_fixture(case):
    config, rules = _case_inputs(case)
    cfg = EngineConfig(**case.get("engine_config", {}))
    if "error" in case:
        with pytest.raises(getattr(errors, case["error"])) as ei:
            evaluate(config, rules, cfg)
        if case.get("error_pair"):
            assert list(ei.value.pair) == case["error_pair"]
        return
    res = evaluate(config, rules, cfg)
    text = print_configuration(res.final)
    assert res.total_interactions == case["interactions"]
    assert _sha(text) == case["print_sha256"]
    _check_loops(res)


def test_ackermann_communications_equal_reference():
    # no var=var equations arise in Ackermann, so the merge count is schedule-free
    for case in CASES:
        if case.get("program") == "ackermann":
            config, rules = _case_inputs(case)
            assert evaluate(config, rules).total_communications == case["communications"], case["name"]


@pytest.mark.parametrize("order", [None, False])
def test_arith_551_nets_one_launch(order):
    rules = to_rules(PROGRAMS["arith"])
    configs = [to_config(c["net"]) for c in ARITH]
    out = evaluate_batch(configs, rules, EngineConfig(collect_stats=False, reference_order=order))
    for case, res in zip(ARITH, out.results):
        assert res.total_interactions == case["interactions"], case["name"]
        assert _sha(print_configuration(res.final)) == case["print_sha256"], case["name"]


def test_arith_nets_single_launch_each():
    rules = to_rules(PROGRAMS["arith"])
    for case in ARITH[:60]:
        res = evaluate(to_config(case["net"]), rules)
        assert res.total_interactions == case["interactions"], case["name"]
        assert _sha(print_configuration(res.final)) == case["print_sha256"], case["name"]
        _check_loops(res)


def _random_arith_net(rng, syms, budget):
    """Own generator (not the reference's netgen): nested Add/Dup/Eps over literals."""
    eqs, nxt = [], [0]

    def fresh():
        nxt[0] += 1
        return Var(nxt[0] - 1)

    def lit():
        return programs.build_nat(rng.randint(0, 4))

    def expr(b):
        roll = rng.random()
        if b <= 2 or roll < 0.3:
            return lit()
        if roll < 0.6:
            r = fresh()
            eqs.append(Equation(Agent(syms["Add"], (r, expr(b // 2))), expr(b // 2)))
            return r
        if roll < 0.85:
            a, c, r = fresh(), fresh(), fresh()
            eqs.append(Equation(Agent(syms["Dup"], (a, c)), expr(b - 2)))
            eqs.append(Equation(Agent(syms["Add"], (r, a)), c))
            return r
        eqs.append(Equation(Agent(syms["Eps"]), expr(b // 3)))
        return expr(b // 2)

    top = expr(budget)
    return Configuration((top,), tuple(eqs))


def test_random_arith_nets_against_oracle():
    rules = programs.load_rules("arith")
    orules = O.rules_for("arith")
    rng = random.Random(1234)
    nets = [_random_arith_net(rng, rules.symbols, rng.choice([8, 40, 200, 1000])) for _ in range(300)]
    out = evaluate_batch(nets, rules, EngineConfig(collect_stats=False))
    for net, res in zip(nets, out.results):
        want = O.run_config(net, orules, collect=False)
        assert res.total_interactions == want.interactions
        assert print_configuration(res.final) == want.printed()


@pytest.mark.parametrize("params,interactions,sha", [
    ((3, 8), 5_574_030, "b85606c71178de4b"),
    ((3, 10), 89_404_824, "981fd9bfe283f466"),
])
def test_large_ackermann(params, interactions, sha):
    prog = programs.program("ackermann")
    res = evaluate(prog.build_input(*params), prog.rules)
    assert res.total_interactions == interactions
    text = print_configuration(res.final)
    assert _sha(text).startswith(sha)
    assert programs.nat_value(res.final.interface[0]) == programs.ackermann_value(*params)
    _check_loops(res)


def test_batch_of_ackermann_3_6():
    prog = programs.program("ackermann")
    nets = [prog.build_input(3, 6) for _ in range(512)]
    out = evaluate_batch(nets, prog.rules, EngineConfig(collect_stats=False), as_terms=True)
    assert out.total_interactions == 512 * 344_964
    for r in out.results:
        assert r.total_interactions == 344_964
        assert programs.nat_value(r.final.interface[0]) == 509


def test_headline_batch_4096_ackermann_3_6():
    """BASELINE.json configs[4], the kernel variant bench.py times: 4096 x A(3,6) through
    evaluate_batch with automatic threads (tier S, 128 threads per net, no per-rule
    counters, normal forms finalized on the device and printed natively). Every
    net's printed normal form equals the reference's (cases.json, generated by the
    reference), and the total is SURVEY.md §8(c)'s 1,412,972,544."""
    from paper_1404_0076_b200 import _native

    case = next(c for c in CASES if c.get("program") == "ackermann" and c["params"] == [3, 6])
    prog = programs.program("ackermann")
    nets = [prog.build_input(3, 6) for _ in range(4096)]
    out = evaluate_batch(nets, prog.rules, EngineConfig(collect_stats=False), as_terms=False, as_text=True)
    assert out.total_interactions == 1_412_972_544
    assert out.max_rounds == 3_499  # the reference's loop count
    assert len(out.texts) == 4096
    bad = [i for i, t in enumerate(out.texts) if _sha(t) != case["print_sha256"]]
    assert not bad, f"{len(bad)} nets differ, first {bad[:5]}"
    assert all(r.total_interactions == 344_964 for r in out.results)
    assert all(r.total_communications == case["communications"] for r in out.results)
    ctx = _native.context(0)
    st = ctx.stats(4095)
    assert (st.tier, st.threads, st.jit, st.device_final) == (_native.TIER_S, 128, 1, 1)


def test_mixed_batch_against_oracle():
    prog = programs.program("ackermann")
    orules = O.rules_for("ackermann")
    rng = random.Random(7)
    params = [(rng.randint(0, 3), rng.randint(0, 6)) for _ in range(200)]
    nets = [prog.build_input(m, n) for m, n in params]
    out = evaluate_batch(nets, prog.rules, EngineConfig(collect_stats=False))
    for (m, n), net, res in zip(params, nets, out.results):
        want = O.run_config(net, orules, collect=False)
        assert res.total_interactions == want.interactions, (m, n)
        assert print_configuration(res.final) == want.printed(), (m, n)


def test_errors_map_to_reference_classes():
    rules = programs.load_rules("addition")
    sp = parse_program("Add(r,y) >< S(x) => Add(w,y)=x, r=S(w);\nAdd(r,y) >< Z => r=y;\nnet r : Add(r, Z) = S(Z);")
    with pytest.raises(errors.SlotOverflow):
        evaluate(sp.net, sp.rules, EngineConfig(slot_count=1))
    loop = parse_program("Loop >< Z => Loop = Z;\nnet : Loop = Z;")
    with pytest.raises(errors.LoopCapExceeded) as ei:
        evaluate(loop.net, loop.rules, EngineConfig(max_loops=5))
    assert ei.value.max_loops == 5
    bad = parse_program("A >< B => ;\nnet : A = C;")
    with pytest.raises(errors.NoRuleForPair) as ei:
        evaluate(bad.net, bad.rules)
    assert ei.value.pair == ("A", "C")
    del rules


def test_collect_stats_off_and_arena_growth():
    prog = programs.program("fibonacci")
    res = evaluate(prog.build_input(15), prog.rules, EngineConfig(collect_stats=False))
    assert res.loops == [] and res.total_interactions == 11_092
    # a tiny initial arena must grow transparently
    from paper_1404_0076_b200 import _native, engine

    prep = engine.prepare([prog.build_input(18)], prog.rules)
    ctx = _native.context(0)
    with ctx.lock:
        ctx.load_rules(prep.blob)
        ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
        k = engine.native_cfg(EngineConfig(collect_stats=False))
        k.cap_agents, k.cap_vars = 128, 128
        code, _ = ctx.reduce(k)
        st = ctx.stats(0)
        ctx._blob_key = None
    assert code == _native.OK
    assert st.interactions == 50_515 and st.cap_agents > 128


# ---- tier C: one net on a thread-block cluster (distributed shared memory) ----

@pytest.mark.parametrize("g", [2, 4, 16])
def test_cluster_tier_fixtures(g):
    """Every reference fixture through the cluster engine: same normal form and interaction count."""
    for case in CASES:
        config, rules = _case_inputs(case)
        kw = dict(case.get("engine_config", {}))
        kw["ctas_per_net"] = g
        kw["reference_order"] = False  # this tier, not tier R
        cfg = EngineConfig(**kw)
        if "error" in case:
            with pytest.raises(getattr(errors, case["error"])) as ei:
                evaluate(config, rules, cfg)
            if case.get("error_pair"):
                assert list(ei.value.pair) == case["error_pair"], case["name"]
            continue
        res = evaluate(config, rules, cfg)
        assert res.total_interactions == case["interactions"], case["name"]
        assert _sha(print_configuration(res.final)) == case["print_sha256"], case["name"]
        _check_loops(res)


@pytest.mark.parametrize("params,interactions,communications,loops,sha", [
    ((3, 8), 5_574_030, 4_177_966, 14_235, "b85606c71178de4b"),
    ((3, 10), 89_404_824, 67_043_382, 57_227, "981fd9bfe283f466"),
])
def test_cluster_tier_large_ackermann(params, interactions, communications, loops, sha):
    prog = programs.program("ackermann")
    res = evaluate(prog.build_input(*params), prog.rules, EngineConfig(ctas_per_net=16))
    assert res.total_interactions == interactions
    assert res.total_communications == communications
    assert len(res.loops) == loops
    assert _sha(print_configuration(res.final)).startswith(sha)
    _check_loops(res)


def test_cluster_tier_random_arith_against_oracle():
    rules = programs.load_rules("arith")
    orules = O.rules_for("arith")
    rng = random.Random(99)
    for _ in range(40):
        net = _random_arith_net(rng, rules.symbols, rng.choice([8, 40, 200, 1000]))
        res = evaluate(net, rules, EngineConfig(ctas_per_net=8, collect_stats=False, reference_order=False))
        want = O.run_config(net, orules, collect=False)
        assert res.total_interactions == want.interactions
        assert print_configuration(res.final) == want.printed()


# ---- reference loop mode: LoopStats rows are the reference's loops ----------

# Rule sets whose right-hand sides never equate two variables. With var=var
# equations the reference's loop timing depends on its own variable numbering
# (the smaller id keys the equation, engine.py:150-153), which a parallel
# allocator does not reproduce; interactions and normal forms never depend on it.
NO_VAR_VAR = ("ackermann", "lsystem")


@pytest.mark.parametrize("g", [1, 16])
def test_loop_rows_equal_reference(g):
    """exact_loops=True: loop count, per-loop interactions and live equations equal the
    reference fixtures row for row (engine.py:215-221)."""
    checked = 0
    for case in CASES:
        if case.get("program") not in NO_VAR_VAR or not case.get("loops"):
            continue
        config, rules = _case_inputs(case)
        res = evaluate(config, rules, EngineConfig(ctas_per_net=g, exact_loops=True))
        want = case["loops"]
        got = [(s.interactions, s.live_equations) for s in res.loops]
        assert len(got) == len(want), case["name"]
        assert [w[0] for w in want] == [x[0] for x in got], case["name"]  # interactions per loop
        assert [w[2] for w in want] == [x[1] for x in got], case["name"]  # live equations per loop
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("exact", [False, True])
def test_both_loop_modes_reach_the_same_normal_form(exact):
    prog = programs.program("fibonacci")
    res = evaluate(prog.build_input(18), prog.rules, EngineConfig(exact_loops=exact))
    assert res.total_interactions == 50_515
    assert programs.nat_value(res.final.interface[0]) == 2584
    _check_loops(res)


# ---- tier X: one net on the whole GPU (cooperative grid, global memory) -------

def test_whole_gpu_tier_fixtures():
    """Every reference fixture forced through the whole-GPU tier (ctas_per_net > 16)."""
    for case in CASES:
        config, rules = _case_inputs(case)
        kw = dict(case.get("engine_config", {}))
        kw["ctas_per_net"] = 148
        kw["reference_order"] = False  # this tier, not tier R
        cfg = EngineConfig(**kw)
        if "error" in case:
            with pytest.raises(getattr(errors, case["error"])):
                evaluate(config, rules, cfg)
            continue
        res = evaluate(config, rules, cfg)
        assert res.total_interactions == case["interactions"], case["name"]
        assert _sha(print_configuration(res.final)) == case["print_sha256"], case["name"]
        _check_loops(res)


@pytest.mark.parametrize("n", [22, 24])
def test_wide_lsystem_against_oracle(n):
    """L-system nets too wide for a cluster run on the whole GPU; same result as the oracle."""
    prog = programs.program("lsystem")
    net = prog.build_input(n)
    res = evaluate(net, prog.rules)
    want = O.run_config(net, O.rules_for("lsystem"), collect=True)
    assert res.total_interactions == want.interactions
    assert print_configuration(res.final) == want.printed()
    assert len(res.loops) == want.loops
    assert [s.interactions for s in res.loops] == [row[0] for row in want.rows]


@pytest.mark.parametrize("ctas", [1, 16, 148])
def test_errors_in_every_single_net_tier(ctas):
    """LoopCapExceeded / NoRuleForPair from tiers M, C and X as the reference's classes."""
    loop = parse_program("Loop >< Z => Loop = Z;\nnet : Loop = Z;")
    with pytest.raises(errors.LoopCapExceeded) as ei:
        evaluate(loop.net, loop.rules, EngineConfig(max_loops=7, ctas_per_net=ctas, reference_order=False))
    assert ei.value.max_loops == 7
    bad = parse_program("A >< B => ;\nnet : A = C;")
    with pytest.raises(errors.NoRuleForPair) as ei:
        evaluate(bad.net, bad.rules, EngineConfig(ctas_per_net=ctas, reference_order=False))
    assert ei.value.pair == ("A", "C")
    # a cap that A(3,5)'s loop count exceeds, on a net large enough to use the tier
    prog = programs.program("ackermann")
    want = O.run_config(prog.build_input(3, 5), O.rules_for("ackermann"), collect=True)
    for cap in (len(want.rows) // 2, len(want.rows) - 1):  # the trailing no-op loop counts too
        with pytest.raises(errors.LoopCapExceeded):
            evaluate(prog.build_input(3, 5), prog.rules, EngineConfig(max_loops=cap, ctas_per_net=ctas))
    res = evaluate(prog.build_input(3, 5), prog.rules, EngineConfig(max_loops=len(want.rows), ctas_per_net=ctas))
    assert res.total_interactions == want.interactions


def test_sharded_batch_gathers_in_input_order():
    """evaluate_sharded: contiguous shards, one host thread each (here two shards
    on the one device), results gathered in input order like evaluate_batch."""
    from paper_1404_0076_b200 import evaluate_sharded

    prog = programs.program("ackermann")
    rng = random.Random(21)
    params = [(rng.randint(0, 3), rng.randint(0, 5)) for _ in range(101)]
    nets = [prog.build_input(m, n) for m, n in params]
    one = evaluate_batch(nets, prog.rules, EngineConfig(collect_stats=False))
    two = evaluate_sharded(nets, prog.rules, devices=[0, 0], cfg=EngineConfig(collect_stats=False))
    assert len(two.results) == len(nets)
    assert two.total_interactions == one.total_interactions
    for a, b in zip(one.results, two.results):
        assert a.total_interactions == b.total_interactions
        assert print_configuration(a.final) == print_configuration(b.final)


def test_symbol_only_on_a_right_hand_side():
    """A rule set built in code whose right-hand side creates an undeclared
    symbol: reduced like the reference reduces it."""
    from inet.core import Rule, RuleSet, Symbol

    a, b, c = Symbol("A", 1), Symbol("B", 0), Symbol("C", 0)
    rs = RuleSet()
    rs.add(Rule(a, (0,), b, (), (Equation(Var(0), Agent(c)),)))
    net = Configuration((Var(5),), (Equation(Agent(a, (Var(5),)), Agent(b)),))
    res = evaluate(net, rs)
    assert print_configuration(res.final) == "net C : ;"
    assert res.total_interactions == 1


def test_rule_with_the_most_equations_single_and_batch():
    """A rule with the most right-hand-side equations the rule compiler takes
    (8: a variable chain and four agent pairs; tier M sizes its queue so a
    round's pushes fit the 16-bit push counter, engine.cu tier_m_queue):
    single net and batch equal the oracle, text, counts and rows."""
    import sys

    sys.path.insert(0, __import__("os").path.dirname(__file__))
    import fuzz_gen as F

    src = "A(a) >< B(b) => a = x1, x1 = x2, x2 = x3, x3 = b, Z = Z, Z = Z, Z = Z, Z = Z;\nZ >< Z => ;\n"
    names = ", ".join(f"r{i}, s{i}" for i in range(300))
    eqs = ", ".join(f"A(r{i}) = B(s{i})" for i in range(300))
    sp = parse_program(src + f"net {names} : {eqs};")
    orules = O.compile_golden_rules(F.to_golden(sp.rules))
    want = O.run_config(sp.net, orules, collect=True)
    res = evaluate(sp.net, sp.rules, EngineConfig())
    assert res.total_interactions == want.interactions
    assert res.total_communications == want.communications
    assert [(s.interactions, s.communications, s.live_equations) for s in res.loops] == [tuple(r) for r in want.rows]
    assert print_configuration(res.final) == want.printed()
    out = evaluate_batch([sp.net] * 64, sp.rules, EngineConfig(collect_stats=False), as_text=True)
    assert all(t == want.printed() for t in out.texts)
