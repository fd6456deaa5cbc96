"""Host-side domain model of the lightweight interaction calculus.

This is the Python surface the device engine consumes and produces. It keeps
the reference's names and attribute layout (src/inet/core.py:19-312) so that
user code written against the reference — ``Var(id)``, ``Agent(sym,
children)``, ``Equation(lhs, rhs)``, ``Configuration(interface, equations)``,
``Rule``/``RuleSet`` — works unchanged, and so that the engine can equally be
handed the reference's own objects (it only reads ``.id``, ``.sym.name``,
``.sym.arity``, ``.children``, ``.lhs``, ``.rhs``).

Terms are immutable trees whose leaves are variables; every variable id occurs
at most twice in a configuration. All traversals are iterative: normal forms
such as the Ackermann(3,10) result are 8,190-deep successor towers.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Iterator, Optional, Union

from .errors import NoRuleForPair, RuleShapeError


@dataclass(frozen=True, slots=True)
class Symbol:
    """Agent label plus auxiliary-port count (src/inet/core.py:19-30)."""

    name: str
    arity: int

    def __post_init__(self):
        if not self.name or not self.name[0].isupper():
            raise ValueError(f"agent name must start upper-case: {self.name!r}")
        if self.arity < 0:
            raise ValueError("arity must be non-negative")


class Var:
    """Variable leaf; identity is the integer id alone."""

    __slots__ = ("id",)

    def __init__(self, id: int):
        self.id = id

    def __repr__(self):
        return f"Var({self.id})"

    def __eq__(self, other):
        return type(other) is Var and other.id == self.id

    def __hash__(self):
        return hash(("var", self.id))


class Agent:
    """A symbol applied to exactly ``sym.arity`` subterms."""

    __slots__ = ("sym", "children")

    def __init__(self, sym: Symbol, children: tuple = ()):
        if len(children) != sym.arity:
            raise ValueError(
                f"{sym.name} has arity {sym.arity}, got {len(children)} children"
            )
        self.sym = sym
        self.children = children

    def __repr__(self):
        return f"Agent({self.sym.name}, {self.children!r})"

    def __eq__(self, other):
        return type(other) is Agent and terms_equal(self, other)

    def __hash__(self):
        return hash(("agent", self.sym, self.children))


Term = Union[Var, Agent]


def is_var(t) -> bool:
    """Duck-typed variable test: accepts this package's and the reference's terms."""
    return not hasattr(t, "sym")


def terms_equal(a: Term, b: Term) -> bool:
    """Structural equality without recursion."""
    work = [(a, b)]
    while work:
        x, y = work.pop()
        xv, yv = is_var(x), is_var(y)
        if xv != yv:
            return False
        if xv:
            if x.id != y.id:
                return False
            continue
        if x.sym != y.sym or len(x.children) != len(y.children):
            return False
        work.extend(zip(x.children, y.children))
    return True


def iter_vars(term: Term) -> Iterator[int]:
    """Variable ids of ``term`` in left-to-right preorder."""
    work = [term]
    while work:
        t = work.pop()
        if is_var(t):
            yield t.id
        else:
            for c in reversed(t.children):
                work.append(c)


@dataclass(slots=True)
class Equation:
    """``lhs = rhs``; unordered in the calculus."""

    lhs: Term
    rhs: Term

    def sides(self) -> tuple[Term, Term]:
        return (self.lhs, self.rhs)


class EqClass(Enum):
    ACTIVE = "active"
    VAR_HEADED = "var-headed"
    VAR_VAR = "var-var"


def classify(eq: Equation) -> EqClass:
    """ACTIVE (agent = agent), VAR_VAR, or VAR_HEADED (src/inet/core.py:124-132)."""
    lv, rv = is_var(eq.lhs), is_var(eq.rhs)
    if lv and rv:
        return EqClass.VAR_VAR
    if lv or rv:
        return EqClass.VAR_HEADED
    return EqClass.ACTIVE


@dataclass(slots=True)
class Configuration:
    """Interface terms plus a multiset of equations."""

    interface: tuple[Term, ...]
    equations: tuple[Equation, ...]

    def _all_terms(self) -> Iterator[Term]:
        yield from self.interface
        for eq in self.equations:
            yield eq.lhs
            yield eq.rhs

    def max_var_id(self) -> int:
        """Largest variable id, or -1 when the net has none (src/inet/core.py:142-149)."""
        best = -1
        for t in self._all_terms():
            for v in iter_vars(t):
                if v > best:
                    best = v
        return best


@dataclass(slots=True)
class Rule:
    """Interaction rule for one unordered pair (src/inet/core.py:158-208).

    ``a_vars``/``b_vars`` are the rule-local ids bound to the auxiliary ports
    of ``lhs_a``/``lhs_b``; every other id in ``rhs`` is a bound variable that
    is renamed fresh at each application. ``bound_vars`` lists them in
    first-occurrence (preorder) order.
    """

    lhs_a: Symbol
    a_vars: tuple[int, ...]
    lhs_b: Symbol
    b_vars: tuple[int, ...]
    rhs: tuple[Equation, ...]
    bound_vars: tuple[int, ...] = field(init=False)

    def __post_init__(self):
        if len(self.a_vars) != self.lhs_a.arity or len(self.b_vars) != self.lhs_b.arity:
            raise RuleShapeError("pattern variable count must match arity")
        pattern = tuple(self.a_vars) + tuple(self.b_vars)
        if len(set(pattern)) != len(pattern):
            raise RuleShapeError("pattern variables must be pairwise distinct")
        seen: dict[int, int] = {}
        for eq in self.rhs:
            for side in (eq.lhs, eq.rhs):
                for v in iter_vars(side):
                    seen[v] = seen.get(v, 0) + 1
        for v in pattern:
            if seen.get(v, 0) != 1:
                raise RuleShapeError(
                    f"pattern variable {v} must occur exactly once in the rhs"
                )
        pset = set(pattern)
        bound = []
        for v, n in seen.items():  # dict order == first occurrence
            if v in pset:
                continue
            if n != 2:
                raise RuleShapeError(
                    f"bound rule variable {v} must occur exactly twice in the rhs"
                )
            bound.append(v)
        self.bound_vars = tuple(bound)

    @property
    def pair(self) -> tuple[str, str]:
        return (self.lhs_a.name, self.lhs_b.name)


def pair_key(a: str, b: str) -> tuple[str, str]:
    return (a, b) if a <= b else (b, a)


class RuleSet:
    """Declared symbols plus at most one rule per unordered pair."""

    def __init__(self):
        self.symbols: dict[str, Symbol] = {}
        self.rules: dict[tuple[str, str], Rule] = {}

    def declare(self, sym: Symbol) -> Symbol:
        old = self.symbols.get(sym.name)
        if old is None:
            self.symbols[sym.name] = sym
            return sym
        if old.arity != sym.arity:
            raise RuleShapeError(
                f"symbol {sym.name} used with arities {old.arity} and {sym.arity}"
            )
        return old

    def add(self, rule: Rule) -> None:
        self.declare(rule.lhs_a)
        self.declare(rule.lhs_b)
        key = pair_key(rule.lhs_a.name, rule.lhs_b.name)
        if key in self.rules:
            raise RuleShapeError(f"duplicate rule for pair {key[0]} >< {key[1]}")
        self.rules[key] = rule

    def lookup(self, a: str, b: str) -> Optional[Rule]:
        return self.rules.get(pair_key(a, b))

    @property
    def max_rhs_size(self) -> int:
        return max((len(r.rhs) for r in self.rules.values()), default=0)

    @property
    def max_fresh(self) -> int:
        return max((len(r.bound_vars) for r in self.rules.values()), default=0)


class FreshIdAllocator:
    """Monotone variable-id source (src/inet/core.py:254-272)."""

    def __init__(self, start: int = 0):
        self.next_id = start

    def fresh(self) -> int:
        v = self.next_id
        self.next_id += 1
        return v

    def reserve(self, count: int) -> int:
        base = self.next_id
        self.next_id += count
        return base


def find_rule(rules: RuleSet, eq: Equation) -> Rule:
    """Rule of an active equation or ``NoRuleForPair`` in equation orientation."""
    rule = rules.lookup(eq.lhs.sym.name, eq.rhs.sym.name)
    if rule is None:
        raise NoRuleForPair(eq.lhs.sym.name, eq.rhs.sym.name)
    return rule
