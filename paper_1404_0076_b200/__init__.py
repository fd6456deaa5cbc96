"""B200-native interaction-net evaluator: drop-in for ``inet.engine.evaluate``.

The public surface mirrors the reference package ``inet`` (src/inet/__init__.py)
for the reduction path: the calculus types, the ``.inet`` parser and canonical
printer, ``EngineConfig``/``EvalResult``/``LoopStats`` and ``evaluate`` — plus
``evaluate_batch`` / ``evaluate_sharded`` for many independent nets. The
reduction itself runs in hand-written CUDA for sm_100a behind the C ABI in
include/inet_b200.h (``libinetb200.so``, built in-tree).
"""

from .core import (
    Agent,
    Configuration,
    EqClass,
    Equation,
    FreshIdAllocator,
    Rule,
    RuleSet,
    Symbol,
    Var,
    classify,
    find_rule,
)
from .engine import (
    BatchResult,
    EngineConfig,
    EvalResult,
    check_name_discipline,
    evaluate,
    evaluate_batch,
    evaluate_sharded,
    evaluate_text,
    finalize,
    reduce_by_key,
)
from .lang import parse_program, parse_rules, print_configuration, print_program, print_rule
from .profile import LoopStats, RunProfile, record

__all__ = [
    "Agent",
    "BatchResult",
    "Configuration",
    "EngineConfig",
    "EqClass",
    "Equation",
    "EvalResult",
    "FreshIdAllocator",
    "LoopStats",
    "Rule",
    "RuleSet",
    "RunProfile",
    "Symbol",
    "Var",
    "check_name_discipline",
    "classify",
    "evaluate",
    "evaluate_batch",
    "evaluate_sharded",
    "evaluate_text",
    "finalize",
    "find_rule",
    "parse_program",
    "parse_rules",
    "print_configuration",
    "print_program",
    "print_rule",
    "record",
    "reduce_by_key",
]

__version__ = "0.1.0"


def install(module=None) -> None:
    """Rebind the reference's ``evaluate`` to this engine.

    ``install()`` patches ``inet.engine.evaluate`` and ``inet.evaluate`` (and
    ``inet.cli``'s imported name) so existing callers of the reference —
    its CLI, bench and tests — run on the GPU without edits. Objects of the
    reference's own classes go in and come out.
    """
    import importlib

    ref = module or importlib.import_module("inet")
    ref_engine = importlib.import_module(ref.__name__ + ".engine")
    ref_engine.evaluate = evaluate
    ref.evaluate = evaluate
    for sub in ("cli", "bench"):
        try:
            m = importlib.import_module(f"{ref.__name__}.{sub}")
        except ImportError:
            continue
        if hasattr(m, "evaluate"):
            m.evaluate = evaluate
