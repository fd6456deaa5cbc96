"""Drop-in ``evaluate`` running the reduction loop on a B200.

``evaluate(config, rules, cfg)`` has the reference's signature and result
type (src/inet/engine.py:186-228): it validates ``slot_count`` on the host,
flattens the net, compiles the rule table, and calls the C ABI
(include/inet_b200.h) which runs the whole interaction/communication loop in
one persistent CUDA kernel, then performs the sequential cleanup (finalize,
engine.py:287-362) natively on the host and rebuilds terms of the caller's
own classes.

``evaluate_batch`` reduces many independent nets in one launch (one CTA per
net). ``evaluate_sharded`` splits a batch over several GPUs, one host thread
and one context per device, with no inter-GPU traffic.

There is no CPU fallback: without the shared library or a CUDA device the
calls raise ``DeviceError``.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable, Optional, Sequence, TypeVar

import numpy as np

from . import _native
from ._ref import core as _core
from ._ref import engine as _ref_engine
from ._ref import profile as _profile
from .errors import (
    UnsupportedNet,
    ArenaExhausted,
    DeviceError,
    LoopCapExceeded,
    NameDisciplineError,
    NoRuleForPair,
    SlotOverflow,
)
from .flat import FlatNet, Labels, compile_rules, flatten, flatten_many, is_var, term_classes, unflatten

Configuration, Equation, RuleSet, Term = _core.Configuration, _core.Equation, _core.RuleSet, _core.Term
iter_vars = _core.iter_vars
LoopStats = _profile.LoopStats
EvalResult = _ref_engine.EvalResult

T = TypeVar("T")


@dataclass(slots=True)
class EngineConfig(_ref_engine.EngineConfig):
    """The reference's ``EngineConfig`` (engine.py:35-48) plus device knobs.

    The reference's own ``EngineConfig`` is accepted everywhere (the extra
    fields then take their defaults). ``worker_hint`` is accepted for
    compatibility; the device decides its own parallelism. ``device`` selects
    the GPU; ``threads`` the CTA size per net (0 = auto); ``ctas_per_net`` the
    cluster size of a single net (0 = auto); ``exact_loops`` keeps the
    reference's loop structure (a merged equation that is still var-headed
    communicates in the next loop, so ``loops`` rows are the reference's),
    False links to a fixpoint within a round. ``reference_order``: True runs
    tier R, the reference's equation list in its own order (every count, row,
    error and residual equation exactly as engine.py:106-166 produces them);
    False the fast tiers only; None (default) gives the reference's results
    the fast way where it can (``_plan``): nets that can equate two variables
    run on the single-CTA tiers with reference-ordered var = var keys
    (per-variable stamps), rule sets with an orientation-dependent same-symbol
    rule run on tier R, and a net whose fast run failed with NoRuleForPair,
    met a var = var comparison the stamps cannot decide, or left equations in
    its normal form is rerun on tier R. ``validate_phases`` also runs on tier
    R (the name discipline is checked on the device after both phases of
    every loop).
    """

    device: int = 0
    threads: int = 0
    ctas_per_net: int = 0
    exact_loops: bool = True
    reference_order: Optional[bool] = None


def as_engine_config(cfg) -> EngineConfig:
    """A copy of ``cfg`` (this package's or the reference's ``EngineConfig``) as an ``EngineConfig``."""
    out = EngineConfig()
    for cls in type(cfg).__mro__:
        for f in getattr(cls, "__slots__", ()):
            if hasattr(cfg, f):
                setattr(out, f, getattr(cfg, f))
    return out


def reduce_by_key(items: Sequence[T], key: Callable[[T], object], merge: Callable[[T, T], T]) -> list[T]:
    """Fold adjacent equal-key items (engine.py:59-74); ``[2,0,3,3,3,7,5,5]`` -> ``[2,0,9,7,10]``.

    Kept as a host utility of the API surface; the device engine replaces the
    sort + reduce_by_key pass by variable-slot exchange.
    """
    out: list[T] = []
    sentinel = last = object()
    for x in items:
        k = key(x)
        if out and last is not sentinel and k == last:
            out[-1] = merge(out[-1], x)
        else:
            out.append(x)
            last = k
    return out


def check_name_discipline(interface: Sequence[Term], eqs: Sequence[Equation]) -> None:
    """NameDisciplineError if some variable occurs more than twice (engine.py:169-183)."""
    seen: dict[int, int] = {}
    terms = list(interface) + [s for e in eqs for s in (e.lhs, e.rhs)]
    for t in terms:
        for v in iter_vars(t):
            n = seen.get(v, 0) + 1
            if n > 2:
                raise NameDisciplineError(f"variable {v} occurs more than twice")
            seen[v] = n


# ---------------------------------------------------------------------------
# error mapping


def _raise_status(code: int, st, labels: Labels, cfg: EngineConfig) -> None:
    if code == _native.NO_RULE:
        a = labels.symbols[st.err_label_a].name
        b = labels.symbols[st.err_label_b].name
        raise NoRuleForPair(a, b)
    if code == _native.LOOP_CAP:
        raise LoopCapExceeded(cfg.max_loops)
    if code == _native.ARENA:
        raise ArenaExhausted(
            f"device arena exhausted at {st.cap_agents} agents / {st.cap_vars} variables per net"
        )
    raise DeviceError(code, _native.strerror(code))


# ---------------------------------------------------------------------------
# batch plumbing


@dataclass
class Prepared:
    labels: Labels
    blob: np.ndarray
    flats: list
    agents: np.ndarray
    agent_off: np.ndarray
    eqs: np.ndarray
    eq_off: np.ndarray
    iface: np.ndarray
    iface_off: np.ndarray
    n_vars: np.ndarray


_blob_cache: dict = {}


def prepare(configs: Sequence[Configuration], rules: RuleSet) -> Prepared:
    """Flatten nets and compile the rule table (host work, no device)."""
    labels = Labels.of(rules)
    agents, agent_off, eqs, eq_off, iface, iface_off, n_vars, infos = flatten_many(configs, labels)
    blob = compile_rules(rules, labels)  # after flattening: config-only symbols get labels too
    return Prepared(labels=labels, blob=blob, flats=infos, agents=agents, agent_off=agent_off, eqs=eqs,
                    eq_off=eq_off, iface=iface, iface_off=iface_off, n_vars=n_vars)


def native_cfg(cfg: EngineConfig, ordered: bool = False, var_order: bool = False) -> _native.Cfg:
    k = _native.Cfg()
    k.max_loops = max(0, min(int(cfg.max_loops), 0xFFFFFFFE))
    k.collect_stats = 1 if cfg.collect_stats else 0
    k.threads = getattr(cfg, "threads", 0)
    k.ctas_per_net = getattr(cfg, "ctas_per_net", 0)
    k.exact_loops = 1 if getattr(cfg, "exact_loops", True) else 0
    k.reference_order = 1 if ordered else 0
    k.validate_phases = 1 if cfg.validate_phases else 0
    k.var_order = 1 if var_order else 0
    return k


def run_prepared(ctx: _native.Context, prep: Prepared, cfg: EngineConfig, ordered: bool = False,
                 var_order: bool = False) -> tuple[int, float]:
    ctx.load_rules(prep.blob, key=prep.blob.tobytes())
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    return ctx.reduce(native_cfg(cfg, ordered, var_order))


# ---------------------------------------------------------------------------
# evaluation order: the fast tiers or tier R (the reference's list order)


def _rule_equates_variables(rule) -> bool:
    return any(is_var(e.lhs) and is_var(e.rhs) for e in rule.rhs)


def _asymmetric_same_symbol(rules: RuleSet) -> bool:
    from .flat import same_symbol_rule_is_symmetric

    return any(r.lhs_a.name == r.lhs_b.name and not same_symbol_rule_is_symmetric(r) for r in rules.rules.values())


def equates_variables(rules: RuleSet, configs: Sequence[Configuration] = ()) -> bool:
    """Can a var = var equation arise (a rule right-hand side or an input equation
    between two variables)? The reference keys it on the smaller variable id
    (engine.py:150-153), which decides the loop of the merge,
    total_communications and the LoopStats rows."""
    if any(_rule_equates_variables(r) for r in rules.rules.values()):
        return True
    return any(is_var(e.lhs) and is_var(e.rhs) for c in configs for e in c.equations)


def order_sensitive(rules: RuleSet, configs: Sequence[Configuration] = ()) -> bool:
    """Can the reference's own list order show in this run's results?

    Yes when a var = var equation can arise (``equates_variables``) or when a
    same-symbol rule is not symmetric in its two agents (it is applied in the
    orientation of the equation, core.py:287-298, which for a merged pair is
    the list order, engine.py:161-165).
    """
    return _asymmetric_same_symbol(rules) or equates_variables(rules, configs)


# Evaluation modes: the reference's list on the device (tier R); the fast tiers;
# the fast single-CTA tiers with reference-ordered var = var keys (stamps).
MODE_R, MODE_FAST, MODE_STAMPS = "R", "fast", "stamps"


def _plan(cfg, rules: RuleSet, configs: Sequence[Configuration]) -> tuple[str, bool]:
    """(mode, reruns): how to reduce, and whether nets whose outcome the fast
    tiers cannot pin to the reference's order get a second run on tier R."""
    if cfg.validate_phases:
        return MODE_R, False
    forced = getattr(cfg, "reference_order", None)
    if forced is not None:
        return (MODE_R if forced else MODE_FAST), False
    if _asymmetric_same_symbol(rules):
        return MODE_R, False
    if getattr(cfg, "exact_loops", True) and equates_variables(rules, configs):
        return MODE_STAMPS, True
    return MODE_FAST, True


@dataclass
class _NetOut:
    stats: object
    arrays: Optional[tuple] = None  # (agents, iface, eqs), host copies
    text: Optional[str] = None
    rows: Optional[np.ndarray] = None
    n_eqs: int = 0


def _reduce(ctx: _native.Context, prep: Prepared, cfg, mode: str, want_arrays: bool, want_text: bool,
            finalize_threads: int = 0) -> tuple[list, float]:
    """One launch over the prepared nets; per-net outcomes (results of the nets that succeeded)."""
    _code, ms = run_prepared(ctx, prep, cfg, mode == MODE_R, mode == MODE_STAMPS)
    n = len(prep.flats)
    outs = [_NetOut(st) for st in ctx.stats_all(n)]
    ok = [o.stats.status == _native.OK for o in outs]
    if want_arrays or want_text:
        if all(ok):
            ctx.finalize(0xFFFFFFFF, finalize_threads)
        else:
            for i in range(n):
                if ok[i]:
                    ctx.finalize(i, 1)
        counts = ctx.result_counts_all(n)
        texts = ctx.texts(n, label_table(prep.labels), finalize_threads) if want_text else None
        for i in range(n):
            if not ok[i]:
                continue
            outs[i].n_eqs = int(counts[i, 2])
            if want_arrays:
                outs[i].arrays = ctx.result(i)
            if want_text:
                outs[i].text = texts[i]
    if cfg.collect_stats:
        for i in range(n):
            if ok[i]:
                outs[i].rows = ctx.rounds(i)
    return outs, ms


def _evaluate_nets(configs: Sequence[Configuration], rules: RuleSet, cfg, want_arrays: bool, want_text: bool,
                   finalize_threads: int = 0):
    """Reduce nets with the evaluation order ``cfg`` asks for; returns (prep, outs, device ms).

    The mode ``_plan`` picks first, then (default policy) tier R for exactly
    the nets where the reference's list order could still show: a
    NoRuleForPair (which pair of the loop fails first, and its orientation,
    engine.py:88-92), a var = var comparison between two variables made in one
    loop by different interactions (INET_ERR_ORDER), and a normal form that
    keeps equations (where finalize cuts a cycle depends on the list order,
    engine.py:313-355).
    """
    mode, reruns = _plan(cfg, rules, configs)
    if mode == MODE_FAST and not reruns and _asymmetric_same_symbol(rules):
        bad = next(r for r in rules.rules.values() if r.lhs_a.name == r.lhs_b.name)
        raise UnsupportedNet(
            f"rule {bad.lhs_a.name}><{bad.lhs_b.name} is not symmetric in its two agents: with "
            "reference_order=False its result would depend on the orientation of a merged pair")
    ctx = _native.context(getattr(cfg, "device", 0))
    prep = prepare(configs, rules)
    with ctx.lock:
        outs, ms = _reduce(ctx, prep, cfg, mode, want_arrays, want_text, finalize_threads)
        if reruns:
            redo = [i for i, o in enumerate(outs)
                    if o.stats.status in (_native.NO_RULE, _native.ORDER) or o.n_eqs > 0]
            if redo:
                sub = prepare([configs[i] for i in redo], rules)
                souts, sms = _reduce(ctx, sub, cfg, MODE_R, want_arrays, want_text, finalize_threads)
                for j, i in enumerate(redo):
                    outs[i] = souts[j]
                    outs[i].sub = (sub, j)
                ms += sms
    return prep, outs, ms


def _final_of(prep: Prepared, out: _NetOut, i: int, config):
    sub = getattr(out, "sub", None)
    p, j = sub if sub is not None else (prep, i)
    return unflatten(*out.arrays, p.labels, p.flats[j], term_classes(config))


def _labels_of(prep: Prepared, out: _NetOut) -> Labels:
    sub = getattr(out, "sub", None)
    return sub[0].labels if sub is not None else prep.labels


def _check_outcome(prep: Prepared, out: _NetOut, i: int, cfg, configs) -> None:
    st = out.stats
    if st.status == _native.OK:
        return
    if st.status == _native.NAME:
        sub = getattr(out, "sub", None)
        p, j = sub if sub is not None else (prep, i)
        flat = p.flats[j]
        refid = int(st.err_label_a) | (int(st.err_label_b) << 32)
        n_in = len(flat.var_ids)
        # tier R's reference ids: input variables keep their rank, fresh ones are
        # numbered exactly as the reference's allocator numbers them (engine.py:196)
        v = flat.var_ids[refid] if refid < n_in else flat.fresh_base + (refid - n_in)
        raise NameDisciplineError(f"variable {v} occurs more than twice")
    _raise_status(st.status, st, _labels_of(prep, out), cfg)


def _loops(out: _NetOut) -> list:
    if out.rows is None:
        return []
    return [LoopStats(j + 1, int(r[0]), int(r[1]), int(r[2]), int(r[3]) // 1000) for j, r in enumerate(out.rows)]


def evaluate(config: Configuration, rules: RuleSet, cfg: Optional[EngineConfig] = None) -> EvalResult:
    """Reduce ``config`` to normal form on the GPU (engine.py:186-228)."""
    cfg = cfg if cfg is not None else EngineConfig()
    if cfg.slot_count is not None and cfg.slot_count < rules.max_rhs_size:
        raise SlotOverflow(
            f"slot_count {cfg.slot_count} is smaller than the largest rule rhs ({rules.max_rhs_size})"
        )
    prep, outs, _ms = _evaluate_nets([config], rules, cfg, True, False, 1)
    out = outs[0]
    _check_outcome(prep, out, 0, cfg, [config])
    final = _final_of(prep, out, 0, config)
    return EvalResult(final, _loops(out), int(out.stats.interactions), int(out.stats.communications))


@dataclass
class BatchResult:
    """Outcome of ``evaluate_batch``: per-net results plus device timing."""

    results: list  # EvalResult per net (final is None when as_terms=False)
    device_ms: float
    total_interactions: int
    total_communications: int
    max_rounds: int
    texts: Optional[list] = None  # canonical text per net (as_text=True), printed natively


def label_table(labels: Labels) -> _native.LabelTable:
    """Names and arities of a label numbering, in the native printer's layout."""
    tab = getattr(labels, "_table", None)
    if tab is None or tab.n != len(labels.symbols):
        tab = _native.LabelTable([s.name for s in labels.symbols], [s.arity for s in labels.symbols])
        labels._table = tab
    return tab


def evaluate_text(config: Configuration, rules: RuleSet, cfg: Optional[EngineConfig] = None) -> tuple:
    """Reduce ``config`` and return ``(text, total_interactions, total_communications)``.

    ``text`` equals ``print_configuration(evaluate(config, rules, cfg).final)``
    (lang.py:371-396) but is printed by the library from the flat normal form,
    so large results (an 8,190-deep A(3,10) tower, L-system trees) never become
    Python terms.
    """
    cfg = cfg if cfg is not None else EngineConfig(collect_stats=False)
    out = evaluate_batch([config], rules, cfg, as_terms=False, as_text=True)
    r = out.results[0]
    return out.texts[0], r.total_interactions, r.total_communications


def evaluate_batch(
    configs: Sequence[Configuration],
    rules: RuleSet,
    cfg: Optional[EngineConfig] = None,
    as_terms: bool = True,
    finalize_threads: int = 0,
    as_text: bool = False,
) -> BatchResult:
    """Reduce independent nets in one launch (one CTA per net).

    ``as_text`` adds each normal form's canonical text (``print_configuration``
    of the final configuration), printed natively from the flat normal form.
    """
    cfg = cfg if cfg is not None else EngineConfig(collect_stats=False)
    if not configs:
        return BatchResult([], 0.0, 0, 0, 0)
    if cfg.slot_count is not None and cfg.slot_count < rules.max_rhs_size:
        raise SlotOverflow(
            f"slot_count {cfg.slot_count} is smaller than the largest rule rhs ({rules.max_rhs_size})"
        )
    prep, outs, ms = _evaluate_nets(configs, rules, cfg, as_terms, as_text, finalize_threads)
    for i, o in enumerate(outs):
        _check_outcome(prep, o, i, cfg, configs)
    results = []
    for i, (c, o) in enumerate(zip(configs, outs)):
        final = _final_of(prep, o, i, c) if as_terms else None
        results.append(EvalResult(final, _loops(o), int(o.stats.interactions), int(o.stats.communications)))
    return BatchResult(
        results, ms,
        sum(r.total_interactions for r in results),
        sum(r.total_communications for r in results),
        max(int(o.stats.rounds) for o in outs),
        [o.text for o in outs] if as_text else None,
    )


def evaluate_sharded(
    configs: Sequence[Configuration],
    rules: RuleSet,
    devices: Sequence[int],
    cfg: Optional[EngineConfig] = None,
    as_terms: bool = True,
) -> BatchResult:
    """Split a batch into contiguous shards, one per device, reduced concurrently.

    ctypes releases the GIL for every C call, so one host thread per device
    keeps all GPUs busy. Results are gathered in input order.
    """
    devices = list(devices)
    n = len(configs)
    if not devices:
        raise ValueError("no devices")
    bounds = [n * k // len(devices) for k in range(len(devices) + 1)]
    parts: list = [None] * len(devices)
    errors: list = []

    def work(k: int) -> None:
        try:
            c = as_engine_config(cfg if cfg is not None else EngineConfig(collect_stats=False))
            c.device = devices[k]
            parts[k] = evaluate_batch(configs[bounds[k] : bounds[k + 1]], rules, c, as_terms)
        except BaseException as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(devices)) if bounds[k] < bounds[k + 1]]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    done = [p for p in parts if p is not None]
    return BatchResult(
        results=[r for p in done for r in p.results],
        device_ms=max(p.device_ms for p in done),
        total_interactions=sum(p.total_interactions for p in done),
        total_communications=sum(p.total_communications for p in done),
        max_rounds=max(p.max_rounds for p in done),
    )


def finalize(eqs: Sequence[Equation], interface: Sequence[Term]) -> Configuration:
    """Sequential cleanup (engine.py:287-362) via the native host routine."""
    cfg = Configuration(tuple(interface), tuple(eqs))
    classes = term_classes(cfg)
    labels = Labels()
    flat = flatten(cfg, labels)
    agents, iface, feqs, alive = _native.finalize_flat(
        flat.agents.copy(), flat.iface.copy(), flat.eqs.copy(), len(flat.var_ids)
    )
    Var, Agent, Equation_, Configuration_ = classes
    syms = labels.symbols
    vmap = flat.var_ids

    def build(r: int):
        # iterative post-order over the mutated arena
        if r & 0x80000000:
            return Var(vmap[r & 0x7FFFFFFF])
        out: dict[int, object] = {}
        work = [(r, False)]
        while work:
            a, done = work.pop()
            if a in out:
                continue
            lab = int(agents[a, 0])
            ports = [int(p) for p in agents[a, 1 : 1 + syms[lab].arity]]
            if done:
                kids = tuple(Var(vmap[p & 0x7FFFFFFF]) if p & 0x80000000 else out[p] for p in ports)
                out[a] = Agent(syms[lab], kids)
            else:
                work.append((a, True))
                for p in ports:
                    if not p & 0x80000000:
                        work.append((p, False))
        return out[r]

    return Configuration_(
        tuple(build(int(r)) for r in iface),
        tuple(Equation_(build(int(l)), build(int(rr))) for (l, rr), ok in zip(feqs.reshape(-1, 2), alive) if ok),
    )
