"""Host side of the drop-in (CPU-only): rule-table compiler, flattener, native
host finalize, install() and the C-ABI export list. The reference's own types,
parser, printer and benchmark builders are imported, not re-implemented."""

import os
import re

import numpy as np
import pytest

from golden_io import load, to_config, to_rules
from paper_1404_0076_b200 import (
    Agent,
    Configuration,
    Equation,
    Symbol,
    Var,
    finalize,
    parse_program,
)
from inet.lang import parse_rules  # noqa: E402
from paper_1404_0076_b200 import (  # noqa: E402
    print_configuration,
    reduce_by_key,
)
from paper_1404_0076_b200 import errors, flat
from paper_1404_0076_b200._ref import bench as programs

PROGRAMS = load("programs.json")
CASES = load("cases.json")
ARITH = load("arith.json")
S, Z = Symbol("S", 1), Symbol("Z", 0)


def test_reduce_by_key_reference_example():
    assert reduce_by_key([2, 0, 3, 3, 3, 7, 5, 5], key=lambda x: x, merge=lambda a, b: a + b) == [2, 0, 9, 7, 10]
    assert reduce_by_key([], key=lambda x: x, merge=lambda a, b: a + b) == []
    assert reduce_by_key([1, 2, 1], key=lambda x: x, merge=lambda a, b: a + b) == [1, 2, 1]


# -- rule compiler: the product's blob decodes to the reference's rules -----


def _decode(blob, names):
    L, R = int(blob[1]), int(blob[2])
    pw = (L * L + 1) // 2
    pair = blob[4 : 4 + pw].view(np.uint16)[: L * L]
    recs = blob[4 + pw :].reshape(R, 16)
    out = {}
    for la in range(L):
        for lb in range(L):
            t = int(pair[la * L + lb])
            if t == 0xFFFF:
                continue
            rec = recs[t >> 1]
            nn, ne, nf = rec[0] & 0xFF, (rec[0] >> 8) & 0xFF, (rec[0] >> 16) & 0xFF
            ags = [(names[w & 0xFF], (w >> 8) & 0xFF, (w >> 16) & 0xFF, w >> 24) for w in map(int, rec[1 : 1 + nn])]
            eqs = [((int(rec[9 + e // 2]) >> (16 * (e & 1))) & 0xFF, (int(rec[9 + e // 2]) >> (16 * (e & 1) + 8)) & 0xFF)
                   for e in range(ne)]

            # canonical text of the rhs: sources resolved recursively
            def txt(s):
                if s < 6:
                    return f"p{s}"
                if s < 14:
                    return f"f{s - 6}"
                n, *ports = ags[s - 14]
                inner = ",".join(txt(p) for p in ports if p != 22)
                return f"{n}({inner})"

            out[(names[la], names[lb])] = (bool(t & 1), int(nf), tuple((txt(a), txt(b)) for a, b in eqs))
    return out


@pytest.mark.parametrize("name", ["addition", "ackermann", "fibonacci", "lsystem", "arith"])
def test_compiled_rules_match_independent_oracle_compiler(name):
    from oracle import oracle as O

    rules = programs.load_rules(name)
    labels = flat.Labels.of(rules)
    ours = _decode(flat.compile_rules(rules, labels), [s.name for s in labels.symbols])
    g = O.compile_golden_rules(PROGRAMS[name])
    theirs = _decode(g.blob, g.names)
    assert ours == theirs


def test_unsupported_arity_is_rejected():
    big = Symbol("Big", 4)
    rules = parse_rules("A >< B => ;")
    cfg = Configuration((), (Equation(Agent(big, (Var(0), Var(1), Var(2), Var(3))), Agent(Symbol("A", 0))),))
    with pytest.raises(errors.UnsupportedNet):
        flat.flatten(cfg, flat.Labels.of(rules, [cfg]))


def test_flatten_unflatten_roundtrip():
    for case in ARITH[:100]:
        cfg = to_config(case["net"])
        rules = programs.load_rules("arith")
        labels = flat.Labels.of(rules)
        f = flat.flatten(cfg, labels)
        # identity "normal form": agents already in preorder from flatten
        back = flat.unflatten(f.agents, f.iface, f.eqs, labels, f, flat.term_classes(cfg))
        assert print_configuration(back) == print_configuration(cfg)


# -- native host finalize (libinetb200.so host code; no GPU needed) ---------


def test_finalize_substitute_then_collect():
    r, x = Var(0), Var(1)
    final = finalize([Equation(r, Agent(S, (x,))), Equation(x, Agent(Z))], [r])
    assert final.equations == ()
    assert final.interface == (Agent(S, (Agent(Z),)),)


def test_finalize_nothing_to_do_and_free_variables():
    assert finalize([], [Var(0)]) == Configuration((Var(0),), ())
    assert finalize([], [Agent(S, (Var(0),))]).interface == (Agent(S, (Var(0),)),)


def test_finalize_leftover_chain():
    a = Agent(Symbol("A", 0))
    final = finalize([Equation(a, Var(0)), Equation(Var(0), Var(1))], [Var(1)])
    assert final.equations == ()
    assert final.interface == (a,)


@pytest.mark.parametrize("reverse", [False, True])
def test_finalize_deep_chain_is_linear(reverse):
    n = 20000
    eqs = [Equation(Var(i), Agent(S, (Var(i + 1),))) for i in range(n)]
    eqs.append(Equation(Var(n), Agent(Z)))
    if reverse:
        eqs.reverse()
    final = finalize(eqs, [Var(0)])
    assert final.equations == ()
    assert programs.nat_value(final.interface[0]) == n


def test_finalize_keeps_cycles_like_reference():
    c = Symbol("C", 1)
    x, y = Var(0), Var(1)
    final = finalize([Equation(x, Agent(c, (y,))), Equation(y, Agent(c, (x,)))], [])
    assert print_configuration(final) == "net : x0 = C(C(x0));"
    assert print_configuration(finalize([Equation(x, x)], [])) == "net : x0 = x0;"


# -- C ABI -------------------------------------------------------------------


def test_library_exports_every_declared_symbol():
    import os

    from paper_1404_0076_b200 import _native

    header = open(os.path.join(os.path.dirname(__file__), "..", "include", "inet_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*)\s+(inet_\w+)\s*\(", header, re.M))
    assert declared == set(_native.EXPORTS)
    lib = _native.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.strerror(_native.NO_RULE) == "no rule for active pair"


def test_context_without_device_fails_loudly():
    from paper_1404_0076_b200 import _native
    from conftest import has_gpu

    if has_gpu():
        pytest.skip("a GPU is present")
    with pytest.raises(errors.DeviceError):
        _native.Context(0)


def test_abi_struct_sizes_match_the_library():
    """The ctypes mirrors of inet_cfg / inet_net_stats have the library's layout (no GPU needed)."""
    import ctypes as C
    from paper_1404_0076_b200 import _native
    lib = _native.load_library()
    cfg_b, st_b = C.c_size_t(), C.c_size_t()
    lib.inet_abi_sizes(C.byref(cfg_b), C.byref(st_b))
    assert cfg_b.value == C.sizeof(_native.Cfg)
    assert st_b.value == C.sizeof(_native.NetStats)


def test_public_entry_points_without_device_fail_loudly():
    """No CPU fallback: evaluate / evaluate_batch / evaluate_text raise DeviceError without a GPU."""
    from conftest import has_gpu
    from paper_1404_0076_b200 import evaluate, evaluate_batch, evaluate_text
    from paper_1404_0076_b200._ref import bench as P

    if has_gpu():
        pytest.skip("a GPU is present")
    prog = P.program("ackermann")
    net = prog.build_input(2, 2)
    for call in (lambda: evaluate(net, prog.rules), lambda: evaluate_batch([net, net], prog.rules),
                 lambda: evaluate_text(net, prog.rules)):
        with pytest.raises(errors.DeviceError):
            call()


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present (build container only)")
def test_install_rebinds_reference_and_accepts_its_objects():
    """Drop-in boundary on CPU: install() rebinds the reference's evaluate, and the
    reference's own Configuration / RuleSet objects flatten to exactly the arrays
    this package's objects give (the device input is the same)."""
    import importlib
    import sys as _sys

    if REF_SRC not in _sys.path:
        _sys.path.insert(0, REF_SRC)
    inet = importlib.import_module("inet")
    ref_bench = importlib.import_module("inet.bench")
    import paper_1404_0076_b200 as b200
    from paper_1404_0076_b200 import engine
    from paper_1404_0076_b200._ref import bench as P

    saved = inet.engine.evaluate
    try:
        b200.install(inet)
        assert inet.engine.evaluate is b200.evaluate and inet.evaluate is b200.evaluate
    finally:
        inet.engine.evaluate = saved
        inet.evaluate = saved
    for name, params in (("ackermann", (2, 3)), ("fibonacci", (7,))):
        ref_prog = ref_bench.program(name)
        ours = P.program(name)
        a = engine.prepare([ref_prog.build_input(*params)], ref_prog.rules)
        b = engine.prepare([ours.build_input(*params)], ours.rules)
        for field in ("blob", "agents", "eqs", "iface", "n_vars"):
            assert np.array_equal(getattr(a, field), getattr(b, field)), (name, field)


# -- native term walks (csrc/hostpy.cpp) against the Python ones -------------


def test_native_flatten_and_unflatten_match_python():
    import random

    import fuzz_gen as F
    from paper_1404_0076_b200 import engine

    assert flat._hostpy is not None, "the native host extension was not built"
    rng = random.Random(5)
    syms = F.random_signature(rng, 6)
    rules = F.random_rules(rng, syms)
    nets = [F.random_net(rng, syms, rng.randint(1, 40), rng.randint(1, 6)) for _ in range(60)]
    nets += [to_config(c["net"]) for c in ARITH[:40]]
    rules_a = to_rules(PROGRAMS["arith"])
    for batch, rs in ((nets[:60], rules), (nets[60:], rules_a)):
        native = engine.prepare(batch, rs)
        saved, flat._hostpy = flat._hostpy, None
        try:
            python = engine.prepare(batch, rs)
        finally:
            flat._hostpy = saved
        for a in ("agents", "agent_off", "eqs", "eq_off", "iface", "iface_off", "n_vars", "blob"):
            assert np.array_equal(getattr(native, a), getattr(python, a)), a
        assert [(f.var_ids, f.fresh_base) for f in native.flats] == [(f.var_ids, f.fresh_base) for f in python.flats]
        # rebuild every input from its own flat form, both ways
        for i, cfg in enumerate(batch):
            a0, a1 = int(native.agent_off[i]), int(native.agent_off[i + 1])
            e0, e1 = int(native.eq_off[i]), int(native.eq_off[i + 1])
            f0, f1 = int(native.iface_off[i]), int(native.iface_off[i + 1])
            ag = native.agents[a0:a1]
            # preorder-like layout: the flattener numbers parents before children
            args = (ag, native.iface[f0:f1], native.eqs[e0:e1], native.labels, native.flats[i], flat.term_classes(cfg))
            got = flat.unflatten(*args)
            saved, flat._hostpy = flat._hostpy, None
            try:
                want = flat.unflatten(*args)
            finally:
                flat._hostpy = saved
            assert got == want
            assert print_configuration(got) == print_configuration(cfg)


def test_native_flatten_falls_back_for_symbols_outside_the_rules():
    from paper_1404_0076_b200 import engine

    rules = parse_program("A >< B => ;\nnet : A = B;").rules
    cfg = Configuration((Var(0),), (Equation(Var(0), Agent(Symbol("Q", 0))),))
    prep = engine.prepare([cfg], rules)
    assert "Q" in prep.labels.index


# -- right-hand-side-only symbols, private JIT cache ----------


def test_symbol_only_on_a_right_hand_side_gets_a_label():
    """A RuleSet built in code declares only its pattern symbols
    (core.py:232-239); a symbol that appears only in a rule's right-hand side
    must still be numbered (it used to raise KeyError in compile_rules)."""
    from inet.core import Rule, RuleSet

    a, b, c = Symbol("A", 1), Symbol("B", 0), Symbol("C", 0)
    rs = RuleSet()
    rs.add(Rule(a, (0,), b, (), (Equation(Var(0), Agent(c)),)))
    labels = flat.Labels.of(rs)
    assert "C" in labels.index
    blob = flat.compile_rules(rs, labels)
    assert blob[1] == len(labels.symbols)


def test_jit_cache_is_private(tmp_path, monkeypatch):
    """Compiled kernels are cached in a per-user directory created 0700 (not a
    shared /tmp path another user could plant cubins in)."""
    from paper_1404_0076_b200 import _native, engine

    monkeypatch.delenv("INET_B200_CACHE", raising=False)
    monkeypatch.setenv("XDG_CACHE_HOME", str(tmp_path))
    rules = parse_program("A >< B => ;\nnet : A = B;").rules
    rules.declare(Symbol("Q", 2))  # a rule set no prebuilt kernel covers
    prep = engine.prepare([], rules)
    code, log = _native.jit_compile(prep.blob, 1, 256)
    assert code == _native.OK, log[:500]
    d = tmp_path / "inet_b200"
    assert d.is_dir() and (d.stat().st_mode & 0o777) == 0o700
    assert any(p.suffix == ".cubin" for p in d.iterdir())
