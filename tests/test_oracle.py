"""Pin the CPU oracle to the reference (CPU-only).

Every fixture in tests/golden/ was produced by running the reference package
(tests/golden/make_golden.py). The oracle must reproduce each one exactly:
status, total interactions and communications, the full per-loop series, and
the canonical printed normal form.
"""

import hashlib

import pytest

from golden_io import load
from oracle import oracle as O

PROGRAMS = load("programs.json")
CASES = load("cases.json")
ARITH = load("arith.json")


def _rules_for_case(case):
    if "program" in case:
        return O.compile_golden_rules(PROGRAMS[case["program"]])
    if "rules" in case:
        return O.compile_golden_rules(case["rules"], extra_symbols=case["net"]["symbols"])
    return O.compile_golden_rules(PROGRAMS["arith"])


def _check(case, res):
    if "error" in case:
        assert res.status == case["error"]
        if case.get("error_pair"):
            assert list(res.error_pair) == case["error_pair"]
        return
    assert res.status == "ok"
    assert res.interactions == case["interactions"]
    assert res.communications == case["communications"]
    assert res.rows == case["loops"]
    text = res.printed()
    assert len(text) == case["print_len"]
    assert hashlib.sha256(text.encode()).hexdigest() == case["print_sha256"]
    if "print" in case:
        assert text == case["print"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_fixture(case):
    rules = _rules_for_case(case)
    ag, eqs, iface = O.flat_from_golden(case["net"], rules.names)
    kw = {}
    if "engine_config" in case:
        kw["max_loops"] = case["engine_config"]["max_loops"]
    _check(case, O.run_arrays(rules, ag, eqs, iface, **kw))


def test_oracle_matches_reference_on_551_arith_nets():
    rules = O.compile_golden_rules(PROGRAMS["arith"])
    for case in ARITH:
        ag, eqs, iface = O.flat_from_golden(case["net"], rules.names)
        _check(case, O.run_arrays(rules, ag, eqs, iface))


def test_survey_goldens_ackermann_3_7_and_3_8():
    """Totals measured on the reference in SURVEY.md §8(c) / Appendix A."""
    from inet.bench import program

    prog = program("ackermann")
    rules = O.rules_for("ackermann")
    r7 = O.run_config(prog.build_input(3, 7), rules, collect=False)
    assert (r7.interactions, r7.communications, r7.loops) == (1_388_937, 1_040_426, 7_075)
    r8 = O.run_config(prog.build_input(3, 8), rules, collect=False)
    assert (r8.interactions, r8.communications, r8.loops) == (5_574_030, 4_177_966, 14_235)
    text = r8.printed()
    assert len(text) == 6144
    assert hashlib.sha256(text.encode()).hexdigest().startswith("b85606c71178de4b")


def test_closed_form_interactions_for_ackermann_3_n():
    """I(n) = (256*4^n + 50)/3 - 72*2^n + 5n, L(n) = 56*2^n - 8n - 37."""
    from inet.bench import program

    prog = program("ackermann")
    rules = O.rules_for("ackermann")
    for n in range(1, 7):
        r = O.run_config(prog.build_input(3, n), rules, collect=False)
        assert r.interactions == (256 * 4**n + 50) // 3 - 72 * 2**n + 5 * n
        assert r.loops == 56 * 2**n - 8 * n - 37
