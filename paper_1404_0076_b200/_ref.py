"""Locate the reference package ``inet`` this engine plugs into.

The engine is a drop-in for one path of the reference (``inet.engine.evaluate``,
src/inet/engine.py:186-228). Everything around that path — the calculus types
(src/inet/core.py), the ``.inet`` parser and canonical printer
(src/inet/lang.py), ``LoopStats`` (src/inet/profile.py), the exception classes
(src/inet/errors.py) and the benchmark builders (src/inet/bench.py) — is the
reference's own code, consumed as-is, not re-implemented.

Lookup order: an importable ``inet`` (the user's installation), else the copy
installed next to this repository by ``__graft_entry__.build()``
(``baseline/_ref``, ``pip install --target`` of the reference package).
"""

from __future__ import annotations

import importlib
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOCAL_INSTALL = os.path.join(_REPO, "baseline", "_ref")


def _import():
    try:
        return importlib.import_module("inet")
    except ImportError:
        pass
    if os.path.isdir(os.path.join(LOCAL_INSTALL, "inet")):
        sys.path.append(LOCAL_INSTALL)
        return importlib.import_module("inet")
    raise ImportError(
        "the reference package `inet` (arxiv/paper_1404_0076, pkg/) is required: install it, "
        f"or run __graft_entry__.build() to place it under {LOCAL_INSTALL}"
    )


inet = _import()
core = importlib.import_module("inet.core")
lang = importlib.import_module("inet.lang")
profile = importlib.import_module("inet.profile")
errors = importlib.import_module("inet.errors")
bench = importlib.import_module("inet.bench")
engine = importlib.import_module("inet.engine")
