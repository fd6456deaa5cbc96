"""Host <-> device formats: rule-table compiler and net flattener.

``compile_rules`` turns a ``RuleSet`` (the reference's Rule/RuleSet,
core.py:158-251) into the rule blob documented in
include/inet_b200.h: a dense ``[label][label] -> (rule, swap)`` table plus one
16-word record per rule listing its new agents and right-hand-side equations
as *sources* (port k of either pattern agent, fresh variable j, new agent m).
This is ``find_rule`` + ``instantiate`` (core.py:281-312) compiled once.

``flatten`` turns a ``Configuration`` into agent records / equation refs /
interface refs with variables renumbered densely; ``unflatten`` rebuilds
terms of the caller's own classes from a device normal form, mapping input
variables back to their ids and numbering fresh ones from
``config.max_var_id() + 1`` like the reference's allocator (engine.py:196).
"""

from __future__ import annotations

import sys
from dataclasses import dataclass, field

import numpy as np

from ._ref import core as _core
from .errors import UnsupportedNet

NONE = 0xFFFFFFFF
VAR = 0x80000000
MAGIC = 0x31524E49
MAX_ARITY, MAX_LABELS, MAX_RULES = 3, 64, 256
MAX_NEW, MAX_EQ, MAX_FRESH = 8, 8, 8
SRC_FRESH, SRC_NEW, SRC_NONE = 6, 14, 22


def is_var(t) -> bool:
    """Variable test on the reference's terms (core.py:33-62): agents carry ``sym``."""
    return not hasattr(t, "sym")


@dataclass
class Labels:
    """Label numbering shared by a rule blob and the nets reduced with it."""

    symbols: list = field(default_factory=list)  # label -> Symbol object
    index: dict = field(default_factory=dict)  # name -> label

    def add(self, sym) -> int:
        lab = self.index.get(sym.name)
        if lab is not None:
            if self.symbols[lab].arity != sym.arity:
                raise UnsupportedNet(f"symbol {sym.name} used with two arities")
            return lab
        if sym.arity > MAX_ARITY:
            raise UnsupportedNet(f"{sym.name} has arity {sym.arity} > {MAX_ARITY}")
        if len(self.symbols) >= MAX_LABELS:
            raise UnsupportedNet(f"more than {MAX_LABELS} agent symbols")
        self.index[sym.name] = len(self.symbols)
        self.symbols.append(sym)
        return self.index[sym.name]

    def add_tree(self, term) -> None:
        """Number every symbol occurring in ``term``."""
        work = [term]
        while work:
            x = work.pop()
            if not is_var(x):
                if x.sym.name not in self.index:
                    self.add(x.sym)
                work.extend(x.children)

    @classmethod
    def of(cls, rules, configs=()) -> "Labels":
        """Declared symbols first (declaration order), then symbols that only
        occur on some rule's right-hand side (a RuleSet built in code declares
        only the pattern symbols, core.py:232-239), then those of the nets."""
        lab = cls()
        for s in rules.symbols.values():
            lab.add(s)
        for rule in rules.rules.values():
            for e in rule.rhs:
                lab.add_tree(e.lhs)
                lab.add_tree(e.rhs)
        for cfg in configs:
            for t in _roots(cfg):
                lab.add_tree(t)
        return lab


def _roots(cfg):
    yield from cfg.interface
    for e in cfg.equations:
        yield e.lhs
        yield e.rhs


def _term_key(t, ren):
    """Hashable skeleton of a rule term; variables through ``ren``."""
    if is_var(t):
        return (("v", ren(t.id)),)
    out = []
    work = [t]
    while work:  # preorder, iterative
        x = work.pop()
        if is_var(x):
            out.append(("v", ren(x.id)))
        else:
            out.append((x.sym.name, len(x.children)))
            work.extend(reversed(x.children))
    return tuple(out)


def same_symbol_rule_is_symmetric(rule) -> bool:
    """True if ``A(x..) >< A(y..) => rhs`` is unchanged when the two pattern
    agents trade places (x_k <-> y_k), up to renaming its bound variables and
    the order/orientation of its equations.

    The reference applies a same-symbol rule in the active equation's own
    orientation (core.py:287-298). The fast tiers form an active pair by a
    merge in arrival order, so nets with a rule whose result depends on the
    orientation run on tier R, which keeps the reference's order
    (engine.order_sensitive)."""
    swap = dict(zip(rule.a_vars, rule.b_vars))
    swap.update(zip(rule.b_vars, rule.a_vars))
    bound = list(rule.bound_vars)

    def eq_multiset(ren):
        return sorted(tuple(sorted((_term_key(e.lhs, ren), _term_key(e.rhs, ren)))) for e in rule.rhs)

    want = eq_multiset(lambda v: v)
    # try every renaming of the bound variables (a rule has at most 8; same-symbol
    # rules in practice 0-2, so this is a handful of comparisons)
    import itertools

    for perm in itertools.permutations(bound):
        m = dict(zip(bound, perm))
        if eq_multiset(lambda v: swap[v] if v in swap else m[v]) == want:
            return True
    return False


def compile_rules(rules, labels: Labels) -> np.ndarray:
    """RuleSet -> uint32 rule blob (layout in include/inet_b200.h)."""
    L = len(labels.symbols)
    rule_list = list(rules.rules.values())
    if len(rule_list) > MAX_RULES:
        raise UnsupportedNet(f"more than {MAX_RULES} rules")
    pair = np.full(L * L + (L * L) % 2, 0xFFFF, dtype=np.uint16)
    recs = np.zeros((len(rule_list), 16), dtype=np.uint32)
    for ri, rule in enumerate(rule_list):
        la = labels.add(rule.lhs_a)
        lb = labels.add(rule.lhs_b)
        pair[la * L + lb] = ri << 1
        if la != lb:
            pair[lb * L + la] = (ri << 1) | 1
        env = {}
        for k, v in enumerate(rule.a_vars):
            env[v] = k
        for k, v in enumerate(rule.b_vars):
            env[v] = 3 + k
        if len(rule.bound_vars) > MAX_FRESH:
            raise UnsupportedNet(f"rule {rule.lhs_a.name}><{rule.lhs_b.name}: too many fresh variables")
        for j, v in enumerate(rule.bound_vars):
            env[v] = SRC_FRESH + j
        new_agents: list[list[int]] = []  # [label, src0, src1, src2]

        def source(term) -> int:
            if is_var(term):
                return env[term.id]
            # allocate parent before children so reused slots go to outer agents
            slot = len(new_agents)
            if slot >= MAX_NEW:
                raise UnsupportedNet(f"rule {rule.lhs_a.name}><{rule.lhs_b.name}: too many rhs agents")
            rec = [labels.add(term.sym), SRC_NONE, SRC_NONE, SRC_NONE]
            new_agents.append(rec)
            work = [(term, rec)]
            while work:
                t, r = work.pop()
                for k, ch in enumerate(t.children):
                    if is_var(ch):
                        r[1 + k] = env[ch.id]
                    else:
                        s = len(new_agents)
                        if s >= MAX_NEW:
                            raise UnsupportedNet(
                                f"rule {rule.lhs_a.name}><{rule.lhs_b.name}: too many rhs agents")
                        cr = [labels.add(ch.sym), SRC_NONE, SRC_NONE, SRC_NONE]
                        new_agents.append(cr)
                        r[1 + k] = SRC_NEW + s
                        work.append((ch, cr))
            return SRC_NEW + slot

        if len(rule.rhs) > MAX_EQ:
            raise UnsupportedNet(f"rule {rule.lhs_a.name}><{rule.lhs_b.name}: rhs has > {MAX_EQ} equations")
        eq_src = [(source(e.lhs), source(e.rhs)) for e in rule.rhs]
        recs[ri, 0] = len(new_agents) | (len(eq_src) << 8) | (len(rule.bound_vars) << 16)
        for m, (lab, s0, s1, s2) in enumerate(new_agents):
            recs[ri, 1 + m] = lab | (s0 << 8) | (s1 << 16) | (s2 << 24)
        for e, (sl, sr) in enumerate(eq_src):
            recs[ri, 9 + e // 2] |= (sl | (sr << 8)) << (16 * (e & 1))
    head = np.array([MAGIC, L, len(rule_list), 0], dtype=np.uint32)
    return np.concatenate([head, pair.view(np.uint32), recs.reshape(-1)]).astype(np.uint32)


@dataclass
class FlatNet:
    agents: np.ndarray  # (n, 4) uint32
    eqs: np.ndarray  # (m, 2) uint32
    iface: np.ndarray  # (k,) uint32
    var_ids: list  # dense id -> original id
    fresh_base: int  # first id for fresh variables on the way back


def flatten(config, labels: Labels) -> FlatNet:
    """Configuration -> flat device input (net-local refs)."""
    agents: list[tuple] = []
    dense: dict[int, int] = {}
    var_ids: list[int] = []
    index = labels.index

    def ref(term) -> int:
        if is_var(term):
            d = dense.get(term.id)
            if d is None:
                d = dense[term.id] = len(var_ids)
                var_ids.append(term.id)
            return VAR | d
        # iterative: reserve the record, fill ports afterwards
        root = len(agents)
        agents.append(None)
        work = [(term, root)]
        while work:
            t, slot = work.pop()
            if len(t.children) > MAX_ARITY:
                raise UnsupportedNet(f"{t.sym.name} has arity {len(t.children)} > {MAX_ARITY}")
            ports = [NONE, NONE, NONE]
            for k, ch in enumerate(t.children):
                if is_var(ch):
                    d = dense.get(ch.id)
                    if d is None:
                        d = dense[ch.id] = len(var_ids)
                        var_ids.append(ch.id)
                    ports[k] = VAR | d
                else:
                    s = len(agents)
                    agents.append(None)
                    ports[k] = s
                    work.append((ch, s))
            lab = index.get(t.sym.name)
            if lab is None:
                lab = labels.add(t.sym)
            agents[slot] = (lab, ports[0], ports[1], ports[2])
        return root

    iface = [ref(t) for t in config.interface]
    eqs = [(ref(e.lhs), ref(e.rhs)) for e in config.equations]
    max_id = max(var_ids) if var_ids else -1
    ag = np.array(agents, dtype=np.uint32).reshape(-1, 4)
    eq = np.array(eqs, dtype=np.uint32).reshape(-1, 2)
    fc = np.array(iface, dtype=np.uint32)
    # dense ids in the order of the original ids: the device compares input
    # variables by id where the reference keys var = var on the smaller id
    # (engine.py:150-153)
    if any(var_ids[i] > var_ids[i + 1] for i in range(len(var_ids) - 1)):
        order = np.argsort(np.asarray(var_ids, dtype=np.int64), kind="stable")
        rank = np.empty(len(var_ids), dtype=np.uint32)
        rank[order] = np.arange(len(var_ids), dtype=np.uint32)
        for arr in (ag, eq, fc):
            m = (arr != NONE) & ((arr & VAR) != 0)
            arr[m] = VAR | rank[arr[m] & ~np.uint32(VAR)]
        var_ids = [var_ids[i] for i in order]
    return FlatNet(agents=ag, eqs=eq, iface=fc, var_ids=var_ids, fresh_base=max_id + 1)


@dataclass
class FlatInfo:
    """What unflatten needs of a flattened net (FlatNet without the arrays)."""

    var_ids: list
    fresh_base: int


try:  # native term walks (csrc/hostpy.cpp); the Python ones below are the fallback
    from . import _hostpy
except ImportError:  # pragma: no cover - the extension is built with the library
    _hostpy = None


def flatten_many(configs, labels: Labels):
    """Flatten a batch: (agents, agent_off, eqs, eq_off, iface, iface_off, n_vars, infos).

    Same layout and numbering as ``flatten`` per net, concatenated; the native
    walk handles the reference's classes, anything it cannot (a symbol the
    label table lacks, arity > 3) takes the Python path.
    """
    configs = list(configs)
    if _hostpy is not None and configs:
        try:
            ag, ao, eq, eo, fc, fo, nv, vids, fb = _hostpy.flatten_batch(
                configs, labels.index, _core.Var, _core.Agent, _core.Symbol)
        except LookupError:
            pass
        else:
            u32 = lambda b: np.frombuffer(b, dtype=np.uint32)
            u64 = lambda b: np.frombuffer(b, dtype=np.uint64)
            infos = [FlatInfo(v, f) for v, f in zip(vids, fb)]
            return (u32(ag).reshape(-1, 4), u64(ao), u32(eq).reshape(-1, 2), u64(eo), u32(fc), u64(fo), u32(nv),
                    infos)
    flats = [flatten(c, labels) for c in configs]
    cat = lambda arrs, w: (np.concatenate([a.reshape(-1, w) for a in arrs]) if arrs else np.zeros((0, w), np.uint32))
    offs = lambda arrs: np.concatenate([[0], np.cumsum([len(a) for a in arrs])]).astype(np.uint64)
    return (cat([f.agents for f in flats], 4), offs([f.agents for f in flats]), cat([f.eqs for f in flats], 2),
            offs([f.eqs for f in flats]),
            np.concatenate([f.iface for f in flats]) if flats else np.zeros(0, np.uint32),
            offs([f.iface for f in flats]), np.array([len(f.var_ids) for f in flats], dtype=np.uint32),
            [FlatInfo(f.var_ids, f.fresh_base) for f in flats])


def term_classes(config):
    """(Var, Agent, Equation, Configuration) classes of the caller's objects."""
    mod = sys.modules.get(type(config).__module__)
    if mod is not None and all(hasattr(mod, n) for n in ("Var", "Agent", "Equation", "Configuration")):
        return mod.Var, mod.Agent, mod.Equation, mod.Configuration
    return _core.Var, _core.Agent, _core.Equation, _core.Configuration


def unflatten(agents: np.ndarray, iface: np.ndarray, eqs: np.ndarray, labels: Labels, flat, classes) -> object:
    """Device normal form (preorder agents) -> Configuration of ``classes``."""
    Var, Agent, Equation, Configuration = classes
    if _hostpy is not None:
        return _hostpy.unflatten(np.ascontiguousarray(agents, dtype=np.uint32).tobytes(),
                                 np.ascontiguousarray(iface, dtype=np.uint32).tobytes(),
                                 np.ascontiguousarray(eqs, dtype=np.uint32).tobytes(),
                                 labels.symbols, flat.var_ids, flat.fresh_base, Var, Agent, Equation, Configuration)
    n_in = len(flat.var_ids)
    var_ids = flat.var_ids
    base = flat.fresh_base
    vcache: dict[int, object] = {}

    def var(d: int):
        v = vcache.get(d)
        if v is None:
            v = vcache[d] = Var(var_ids[d] if d < n_in else base + (d - n_in))
        return v

    syms = labels.symbols
    built: list = [None] * len(agents)
    rows = agents.tolist()
    # preorder numbering puts children after parents: build back to front
    for a in range(len(rows) - 1, -1, -1):
        lab, p0, p1, p2 = rows[a]
        sym = syms[lab]
        kids = []
        for p in (p0, p1, p2)[: sym.arity]:
            kids.append(var(p & ~VAR) if p & VAR else built[p])
        built[a] = Agent(sym, tuple(kids))

    def term(r: int):
        return var(r & ~VAR) if r & VAR else built[r]

    return Configuration(
        tuple(term(int(r)) for r in iface),
        tuple(Equation(term(int(l)), term(int(r))) for l, r in eqs.reshape(-1, 2)),
    )
