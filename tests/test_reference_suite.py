"""The reference's own test suite through ``install()`` on the GPU.

SURVEY.md §4 "Reuse in the new build": ``install()`` rebinds
``inet.engine.evaluate`` so the reference's tests of the evaluation path —
``tests/test_engine.py::TestEvaluate`` (reference pkg/tests/test_engine.py:169),
the acceptance criteria C1-C10 (pkg/tests/test_acceptance.py:67-212), the
benchmark and profile tests that call ``evaluate`` (test_bench.py:118-161,
test_profile.py:25-73) and the CLI (test_cli.py) — run unchanged on the device
engine. The suite is the copy ``__graft_entry__.build()`` places in
``baseline/_ref/inet_tests`` next to the installed reference package; the test
skips with the reason when that copy is absent.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "inet_tests")

SELECT = [
    "test_engine.py::TestEvaluate",
    "test_acceptance.py",
    "test_bench.py",
    "test_profile.py",
    "test_cli.py",
]


@pytest.mark.gpu
def test_reference_suite_through_install(tmp_path):
    if not os.path.isdir(SUITE):
        pytest.skip(f"reference test suite not installed at {SUITE} (run __graft_entry__.build())")
    calls = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), REF, SUITE])
    env["INET_B200_CALLS_OUT"] = str(calls)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-rA", "-p", "ref_install_plugin", "-p", "no:cacheprovider",
         "-o", "addopts=", *SELECT],
        cwd=SUITE, env=env, capture_output=True, text=True, timeout=1200,
    )
    log = proc.stdout + proc.stderr
    out = os.environ.get("INET_B200_REFSUITE_LOG")
    if out:
        with open(out, "w") as fh:
            fh.write(log)
    assert proc.returncode == 0, log[-6000:]
    n = json.loads(calls.read_text())["evaluate"]
    assert n >= 500, f"only {n} evaluate() calls reached the device engine"
