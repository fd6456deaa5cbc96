"""pytest plugin: run the reference's own test suite against this engine.

Loaded with ``-p ref_install_plugin`` by tests/test_reference_suite.py. At
configure time (before the reference's test modules import ``evaluate``) it
calls ``paper_1404_0076_b200.install()``, which rebinds ``inet.engine.evaluate``
to the GPU engine, and it counts the device calls so the outer test can prove
the engine — not the reference's Python loop — produced the results.
"""

import json
import os

import paper_1404_0076_b200 as b200
from paper_1404_0076_b200 import engine as _engine

CALLS = {"evaluate": 0}
_inner = b200.evaluate


def _counted(*args, **kwargs):
    CALLS["evaluate"] += 1
    return _inner(*args, **kwargs)


def pytest_configure(config):
    b200.evaluate = _counted
    b200.install()
    assert _engine  # the device engine module is loaded


def pytest_unconfigure(config):
    out = os.environ.get("INET_B200_CALLS_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(CALLS, fh)
