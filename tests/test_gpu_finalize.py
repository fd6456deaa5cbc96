"""Device-side finalize (tier S): the compacted normal form written by the
kernel equals the host finalize of the same reduction, array for array, and
the nets it cannot handle fall back to the host."""

import os
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_1404_0076_b200 import EngineConfig, _native, engine, print_configuration
from paper_1404_0076_b200._ref import bench as programs
from paper_1404_0076_b200.flat import unflatten

from test_gpu_parity import _random_arith_net

pytestmark = pytest.mark.gpu


def _ctx(dev_final):
    old = os.environ.get("INET_B200_DEVFINAL")
    os.environ["INET_B200_DEVFINAL"] = "1" if dev_final else "0"
    try:
        return _native.Context(0)
    finally:
        if old is None:
            del os.environ["INET_B200_DEVFINAL"]
        else:
            os.environ["INET_B200_DEVFINAL"] = old


def _reduce(ctx, nets, rules, cfg=None):
    prep = engine.prepare(nets, rules)
    code, _ = engine.run_prepared(ctx, prep, cfg or EngineConfig(collect_stats=False))
    assert code == _native.OK
    assert ctx.finalize(0xFFFFFFFF, 0) == _native.OK
    out = []
    for i in range(len(nets)):
        st = ctx.stats(i)
        agents, iface, eqs = ctx.result(i)
        out.append((st, np.array(agents, copy=True), np.array(iface, copy=True), np.array(eqs, copy=True)))
    return prep, out


def _compare(nets, rules, orules=None, want_device=None):
    dev = _ctx(True)
    host = _ctx(False)
    try:
        prep, got = _reduce(dev, nets, rules)
        # the reference side: host finalize by the general elimination pass
        # (not the host's own preorder-walk fast path)
        os.environ["INET_B200_HOSTWALK"] = "0"
        try:
            _, ref = _reduce(host, nets, rules)
        finally:
            del os.environ["INET_B200_HOSTWALK"]
        _, walk = _reduce(host, nets, rules)  # host fast path
    finally:
        dev.close()
        host.close()
    for (_, aw, iw, ew), (_, ah, ih, eh) in zip(walk, ref):
        assert np.array_equal(aw, ah) and np.array_equal(iw, ih) and np.array_equal(ew, eh)
    n_dev = 0
    for i, ((sd, ad, idf, ed), (sh, ah, ih, eh)) in enumerate(zip(got, ref)):
        assert sd.tier == 0, "these batches must run in tier S"
        assert sh.device_final == 0
        n_dev += sd.device_final
        assert sd.interactions == sh.interactions
        assert np.array_equal(ad, ah), i
        assert np.array_equal(idf, ih), i
        assert np.array_equal(ed, eh), i
        if orules is not None and i < 64:
            final = unflatten(ad, idf, ed, prep.labels, prep.flats[i], engine.term_classes(nets[i]))
            assert print_configuration(final) == O.run_config(nets[i], orules, collect=False).printed()
    if want_device is not None:
        assert n_dev == want_device
    return n_dev


def test_ackermann_batch_finalized_on_device():
    prog = programs.program("ackermann")
    rng = random.Random(3)
    params = [(rng.randint(0, 3), rng.randint(0, 5)) for _ in range(300)]
    nets = [prog.build_input(m, n) for m, n in params]
    # every Ackermann result is one parked equation x = S(...S(Z)) with x the interface
    _compare(nets, prog.rules, O.rules_for("ackermann"), want_device=len(nets))


def test_random_arith_batch_device_and_host_paths():
    rules = programs.load_rules("arith")
    rng = random.Random(99)
    nets = [_random_arith_net(rng, rules.symbols, rng.choice([8, 40, 200])) for _ in range(200)]
    n_dev = _compare(nets, rules, O.rules_for("arith"))
    assert n_dev > 0


def test_interface_variables_fall_back_to_host():
    # x and y wired straight through (x = y): a var-valued parked equation,
    # finalized by the host; a closed result next to it stays on the device
    from paper_1404_0076_b200 import Agent, Configuration, Equation, Var

    prog = programs.program("ackermann")
    syms = prog.rules.symbols
    wire = Configuration((Var(0), Var(1)), (Equation(Var(0), Var(1)),))
    closed = prog.build_input(2, 2)
    pair = Configuration((Var(0),), (Equation(Var(0), Agent(syms["Z"])),))
    nets = [wire, closed, pair, wire, closed]
    _compare(nets, prog.rules)


def test_native_text_equals_python_printer():
    from paper_1404_0076_b200 import evaluate, evaluate_batch, evaluate_text

    prog = programs.program("ackermann")
    rng = random.Random(11)
    nets = [prog.build_input(rng.randint(0, 3), rng.randint(0, 5)) for _ in range(100)]
    out = evaluate_batch(nets, prog.rules, EngineConfig(collect_stats=False), as_text=True)
    for res, text in zip(out.results, out.texts):
        assert text == print_configuration(res.final)
    rules = programs.load_rules("arith")
    arith = [_random_arith_net(rng, rules.symbols, rng.choice([8, 40, 200])) for _ in range(100)]
    out = evaluate_batch(arith, rules, EngineConfig(collect_stats=False), as_text=True)
    for res, text in zip(out.results, out.texts):
        assert text == print_configuration(res.final)
    # single nets (tiers M / C / X, host finalize): the big normal forms
    for name, params in (("ackermann", (3, 8)), ("lsystem", (22,)), ("fibonacci", (12,))):
        p = programs.program(name)
        cfg = p.build_input(*params)
        text, ints, _ = evaluate_text(cfg, p.rules)
        res = evaluate(cfg, p.rules, EngineConfig(collect_stats=False))
        assert ints == res.total_interactions
        assert text == print_configuration(res.final), name


@pytest.mark.parametrize("name,params", [("lsystem", (20,)), ("lsystem", (24,)), ("ackermann", (3, 7)),
                                         ("fibonacci", (14,))])
def test_host_walk_equals_general_finalize_on_single_nets(name, params):
    prog = programs.program(name)
    nets = [prog.build_input(*params)]
    ctx = _ctx(True)
    try:
        os.environ["INET_B200_HOSTWALK"] = "0"
        try:
            _, ref = _reduce(ctx, nets, prog.rules)
        finally:
            del os.environ["INET_B200_HOSTWALK"]
        _, walk = _reduce(ctx, nets, prog.rules)
    finally:
        ctx.close()
    (_, aw, iw, ew), (_, ah, ih, eh) = walk[0], ref[0]
    assert np.array_equal(aw, ah) and np.array_equal(iw, ih) and np.array_equal(ew, eh)


@pytest.mark.parametrize("n", [12, 18, 22, 26])
def test_whole_gpu_tier_finalized_on_device(n):
    """Tier X nets are finalized on the device (finalize.cuh: parallel resolution,
    Euler tour, pointer-jumping list ranking): the preorder records and the
    interface equal the host finalize's, array for array."""
    prog = programs.program("lsystem")
    nets = [prog.build_input(n)]
    cfg = EngineConfig(collect_stats=False, ctas_per_net=148)
    dev, host = _ctx(True), _ctx(False)
    try:
        prep, got = _reduce(dev, nets, prog.rules, cfg)
        _, ref = _reduce(host, nets, prog.rules, cfg)
    finally:
        dev.close()
        host.close()
    (sd, ad, idf, ed), (sh, ah, ih, eh) = got[0], ref[0]
    assert sd.tier == _native.TIER_X and sd.device_final == 1 and sh.device_final == 0
    assert np.array_equal(ad, ah) and np.array_equal(idf, ih) and np.array_equal(ed, eh)
    final = unflatten(ad, idf, ed, prep.labels, prep.flats[0], engine.term_classes(nets[0]))
    assert programs.census(final.interface[0]) == programs.lsystem_census(n)


def test_whole_gpu_tier_device_finalize_falls_back_on_cycles():
    """Random rule sets leave cyclic normal forms: the device finalize declines
    them and the host's result is the oracle's net."""
    import fuzz_gen as F
    from netgraph import canonical

    rng = random.Random(1003)
    syms = F.random_signature(rng)
    rules = F.random_rules(rng, syms)
    orules = O.compile_golden_rules(F.to_golden(rules))
    cfg = EngineConfig(collect_stats=False, ctas_per_net=148, reference_order=False)
    ctx = _ctx(True)
    try:
        for _ in range(12):
            net = F.random_net(rng, syms, rng.randint(1, 40), rng.randint(1, 6))
            prep, got = _reduce(ctx, [net], rules, cfg)
            st, a, i, e = got[0]
            final = unflatten(a, i, e, prep.labels, prep.flats[0], engine.term_classes(net))
            want = O.run_config(net, orules, collect=False)
            assert st.interactions == want.interactions
            assert canonical(final) == canonical(want.final_config())
    finally:
        ctx.close()
