"""B200-native interaction-net evaluator: drop-in for ``inet.engine.evaluate``.

The reduction loop (src/inet/engine.py:186-228) runs in hand-written CUDA for
sm_100a behind the C ABI in include/inet_b200.h (``libinetb200.so``, built
in-tree). Everything around it is the reference package's own code, imported
(``_ref``): the calculus types, parser and printer, ``LoopStats`` and the
exception classes. This package adds ``evaluate`` (same signature and result
type as the reference's), ``evaluate_batch`` / ``evaluate_sharded`` /
``evaluate_text`` for many nets and large normal forms, and ``install()``.
"""

from ._ref import core as _core
from ._ref import lang as _lang
from ._ref import profile as _profile
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

Agent, Configuration, Equation, Rule, RuleSet, Symbol, Var = (
    _core.Agent, _core.Configuration, _core.Equation, _core.Rule, _core.RuleSet, _core.Symbol, _core.Var)
parse_program, print_configuration = _lang.parse_program, _lang.print_configuration
LoopStats = _profile.LoopStats

__all__ = [
    "Agent",
    "BatchResult",
    "Configuration",
    "EngineConfig",
    "Equation",
    "EvalResult",
    "LoopStats",
    "Rule",
    "RuleSet",
    "Symbol",
    "Var",
    "check_name_discipline",
    "evaluate",
    "evaluate_batch",
    "evaluate_sharded",
    "evaluate_text",
    "finalize",
    "install",
    "parse_program",
    "print_configuration",
    "reduce_by_key",
]

__version__ = "0.2.0"


def install(module=None) -> None:
    """Rebind the reference's ``evaluate`` to this engine.

    ``install()`` patches ``inet.engine.evaluate`` and ``inet.evaluate`` (and
    the names ``inet.cli`` / ``inet.bench`` imported) so existing callers of
    the reference — its CLI, bench and tests — run on the GPU without edits.
    """
    import importlib

    from . import _ref

    ref = module or _ref.inet
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
