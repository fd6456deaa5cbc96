"""Host-side mirror of the reference API (CPU-only): parser, canonical printer,
benchmark programs, rule-table compiler, flattener, native host finalize and
the C-ABI export list."""

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
    parse_rules,
    print_configuration,
    print_program,
    reduce_by_key,
)
from paper_1404_0076_b200 import errors, flat, programs
from paper_1404_0076_b200.lang import print_rule

PROGRAMS = load("programs.json")
CASES = load("cases.json")
ARITH = load("arith.json")
S, Z = Symbol("S", 1), Symbol("Z", 0)


# -- printer: byte parity with the reference's print_configuration -----------


@pytest.mark.parametrize("case", [c for c in CASES if "final" in c], ids=lambda c: c["name"])
def test_printer_reproduces_reference_text(case):
    assert print_configuration(to_config(case["final"])) == case["print"]


def test_printer_on_all_arith_finals():
    for case in ARITH:
        if "final" in case:
            assert print_configuration(to_config(case["final"])) == case["print"], case["name"]


def test_printer_canonical_examples():
    x, y = Var(7), Var(3)
    cfg = Configuration((x,), (Equation(Agent(S, (y,)), x), Equation(y, Agent(Z))))
    assert print_configuration(cfg) == "net x0 : x0 = S(x1), x1 = Z;"
    assert print_configuration(Configuration((), ())) == "net : ;"


# -- parser ------------------------------------------------------------------


def _rule_shape(rule):
    return (rule.lhs_a.name, tuple(rule.a_vars), rule.lhs_b.name, tuple(rule.b_vars), len(rule.rhs),
            tuple(rule.bound_vars), print_rule(rule))


@pytest.mark.parametrize("name", ["addition", "ackermann", "fibonacci", "lsystem", "arith"])
def test_program_rules_equal_reference_rules(name):
    ours = programs.load_rules(name)
    ref = to_rules(PROGRAMS[name])
    assert {k: _rule_shape(r) for k, r in ours.rules.items()} == {k: _rule_shape(r) for k, r in ref.rules.items()}
    assert ours.max_rhs_size == PROGRAMS[name]["max_rhs_size"]
    assert ours.max_fresh == PROGRAMS[name]["max_fresh"]
    assert {n: s.arity for n, s in ours.symbols.items()} == {n: a for n, a in PROGRAMS[name]["symbols"]}


@pytest.mark.parametrize("case", [c for c in CASES if "program" in c], ids=lambda c: c["name"])
def test_builders_equal_reference_inputs(case):
    prog = programs.program(case["program"])
    assert print_configuration(prog.build_input(*case["params"])) == print_configuration(to_config(case["net"]))


@pytest.mark.parametrize("case", [c for c in CASES if "source" in c], ids=lambda c: c["name"])
def test_parse_literal_programs(case):
    sp = parse_program(case["source"])
    assert print_configuration(sp.net) == print_configuration(to_config(case["net"]))


def test_parse_errors_carry_locations():
    with pytest.raises(errors.InetSyntaxError) as ei:
        parse_program("net r : Add(r, Z) = S(Z)")
    assert ei.value.line == 1
    with pytest.raises(errors.ArityError):
        parse_program("net r : S(r) = S(Z, Z);")
    with pytest.raises(errors.NameOccurrenceError):
        parse_program("net : x = A, x = B, x = C;")
    with pytest.raises(errors.DuplicateRuleError):
        parse_rules("A >< B => ;\nB >< A => ;")
    with pytest.raises(errors.NameOccurrenceError):
        parse_rules("A(x) >< B => ;")


def test_deep_terms_parse_and_print_iteratively():
    depth = 5000
    src = "net r : r = " + "S(" * depth + "Z" + ")" * depth + ";"
    sp = parse_program(src)
    assert programs.nat_value(sp.net.equations[0].rhs) == depth
    assert print_configuration(sp.net).count("S(") == depth


def test_print_program_roundtrip():
    text = print_program(parse_program(programs.program_text("fibonacci")))
    again = print_program(parse_program(text))
    assert text == again


def test_reduce_by_key_reference_example():
    assert reduce_by_key([2, 0, 3, 3, 3, 7, 5, 5], key=lambda x: x, merge=lambda a, b: a + b) == [2, 0, 9, 7, 10]
    assert reduce_by_key([], key=lambda x: x, merge=lambda a, b: a + b) == []
    assert reduce_by_key([1, 2, 1], key=lambda x: x, merge=lambda a, b: a + b) == [1, 2, 1]


def test_value_oracles():
    assert programs.ackermann_value(3, 5) == 253
    assert programs.ackermann_value(3, 10) == 8189
    assert programs.fibonacci_value(18) == 2584
    assert programs.lsystem_census(5) == {"Ca": 5, "Cb": 3, "Nil": 1}


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
    from paper_1404_0076_b200 import evaluate, evaluate_batch, evaluate_text, programs as P

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
    from paper_1404_0076_b200 import engine, programs as P

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
