"""Build step: precompile the rule-set kernels of the shipped programs.

The first ``evaluate()`` of a rule set otherwise runs NVRTC (0.7-1.1 s per
kernel variant). ``precompile_shipped()`` compiles, for the benchmark
programs (the reference's programs/*.inet), every variant the engine picks
for them — tier S batches at 128/256/512 threads, tier M single nets, the
16-CTA cluster (tier C), the whole-GPU tier X; with and without the
reference-loop code; the per-rule counters where bench.py asks for them —
into ``kernels/`` next to libinetb200.so, where every later process finds
them (jit.cpp ``package_dir``). Runs on the build host; no GPU needed.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

from . import _native
from .engine import prepare
from ._ref import bench as _bench

load_rules, program = _bench.load_rules, _bench.program

# (tier, threads, style) the engine's selection uses (engine.cu auto_threads /
# tier_style / cluster_threads): batches of > 768 nets (style 0, 128 threads),
# 401..768 (style 1, 128), fewer (style 1, 256); single nets; -1 = the tier's
# default style.
VARIANTS = [
    (_native.TIER_S, 128, 0), (_native.TIER_S, 128, 1), (_native.TIER_S, 256, 1), (_native.TIER_S, 256, 0),
    (_native.TIER_M, 256, -1), (_native.TIER_C, 256, -1), (_native.TIER_X, 256, -1),
]


def shipped_blobs() -> dict:
    """Rule blob of every shipped program, numbered as evaluate() numbers it."""
    out = {}
    for name in ("addition", "ackermann", "fibonacci", "lsystem"):
        p = program(name)
        out[name] = prepare([p.build_input(*p.default_params)], p.rules).blob
    out["arith"] = prepare([], load_rules("arith")).blob
    return out


# single-CTA variants with reference-ordered var = var keys (engine._plan: rule
# sets that equate variables — fibonacci, addition, arith)
STAMP_VARIANTS = [(_native.TIER_S, 128, 0), (_native.TIER_S, 128, 1), (_native.TIER_S, 256, 1),
                  (_native.TIER_M, 256, -1)]


def precompile_shipped(workers: int = 8) -> list:
    jobs = []
    for name, blob in shipped_blobs().items():
        for tier, threads, style in VARIANTS:
            for exact in (False, True):
                for rows in (False, True):
                    jobs.append((name, blob, tier, threads, exact, False, False, style, rows))
        if name in ("fibonacci", "addition", "arith"):
            for tier, threads, style in STAMP_VARIANTS:
                for exact in (False, True):
                    for rows in (False, True):
                        jobs.append((name, blob, tier, threads, exact, False, True, style, rows))
        # accounting runs of bench.py (per-rule histogram)
        if name in ("ackermann", "lsystem", "fibonacci"):
            for tier, threads, style in ((_native.TIER_S, 128, 0), (_native.TIER_M, 256, -1),
                                         (_native.TIER_C, 256, -1), (_native.TIER_X, 256, -1)):
                jobs.append((name, blob, tier, threads, False, True, False, style, False))
    failed = []

    def one(job):
        name, blob, tier, threads, exact, count, stamps, style, rows = job
        code, log = _native.jit_precompile(blob, tier, threads, exact, count, stamps, style, rows)
        if code != 0:
            failed.append((name, tier, threads, exact, count, log[-400:]))

    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(one, jobs))
    if failed:
        raise RuntimeError(f"precompile failed: {failed}")
    return jobs
