"""Random rule sets and nets for differential tests.

Rule sets are complete (a rule for every unordered pair of symbols) and
terminating by construction: a rule's right-hand side creates at most one
agent, so every interaction lowers the agent count. Rules for a symbol with
itself annihilate port by port (symmetric, as a same-symbol rule must be for
the result not to depend on the pair's orientation). Nets obey the name
discipline (every variable occurs exactly twice).
"""

from inet.core import Agent, Configuration, Equation, Rule, RuleSet, Symbol, Var


def random_signature(rng, n=None):
    n = n or rng.randint(3, 6)
    arities = [0, 2] + [rng.randint(0, 3) for _ in range(n - 2)]
    rng.shuffle(arities)
    return [Symbol(f"A{i}", a) for i, a in enumerate(arities)]


def _rule(rng, a, b, syms):
    a_vars = list(range(a.arity))
    b_vars = list(range(a.arity, a.arity + b.arity))
    if a.name == b.name:
        return Rule(a, tuple(a_vars), b, tuple(b_vars),
                    tuple(Equation(Var(x), Var(y)) for x, y in zip(a_vars, b_vars)))
    pattern = a_vars + b_vars
    rng.shuffle(pattern)
    nxt = len(pattern)
    # parity: the ends (pattern variables not in the new agent, plus the agent
    # itself) must pair up
    options = [None] + [s for s in syms if s.arity <= len(pattern)]
    rng.shuffle(options)
    for s in options:
        n_ends = len(pattern) - (s.arity if s else 0) + (1 if s else 0)
        if n_ends % 2 == 0:
            break
    ends = []
    agent = None
    pool = list(pattern)
    if s is not None:
        ports = []
        for _ in range(s.arity):
            if rng.random() < 0.3:  # a bound variable: one end in the agent, one in an equation
                v = Var(nxt)
                nxt += 1
                ports.append(v)
                ends.append(Var(v.id))
            else:
                ports.append(Var(pool.pop()))
        agent = Agent(s, tuple(ports))
        ends.append(agent)
    ends.extend(Var(v) for v in pool)
    rng.shuffle(ends)
    rhs = tuple(Equation(ends[i], ends[i + 1]) for i in range(0, len(ends), 2))
    return Rule(a, tuple(a_vars), b, tuple(b_vars), rhs)


def random_rules(rng, syms):
    rs = RuleSet()
    for i, a in enumerate(syms):
        for b in syms[i:]:
            rs.add(_rule(rng, a, b, syms))
    return rs


def to_golden(rules):
    """RuleSet -> the flat rule format of tests/golden/programs.json (oracle input)."""
    symbols = [[n, s.arity] for n, s in rules.symbols.items()]
    label = {n: i for i, (n, _) in enumerate(symbols)}
    out = []
    for r in rules.rules.values():
        agents = []

        def ref(t):
            if not hasattr(t, "sym"):
                return -(t.id + 1)
            kids = [ref(c) for c in t.children]
            agents.append([label[t.sym.name]] + kids)
            return len(agents) - 1

        rhs = [[ref(e.lhs), ref(e.rhs)] for e in r.rhs]
        out.append({"a": r.lhs_a.name, "a_vars": list(r.a_vars), "b": r.lhs_b.name, "b_vars": list(r.b_vars),
                    "agents": agents, "rhs": rhs, "bound_vars": list(r.bound_vars)})
    return {"symbols": symbols, "rules": out, "max_rhs_size": rules.max_rhs_size, "max_fresh": rules.max_fresh}


def random_net(rng, syms, n_eqs, depth):
    pending = []
    nxt = [0]

    def leaf():
        if pending and rng.random() < 0.5:
            return pending.pop(rng.randrange(len(pending)))
        v = Var(nxt[0])
        nxt[0] += 1
        pending.append(v)
        return v

    def tree(d):
        if d <= 0 or rng.random() < 0.25:
            return leaf()
        return root(d)

    def root(d):
        s = rng.choice(syms)
        return Agent(s, tuple(tree(d - 1) for _ in range(s.arity)))

    eqs = []
    for _ in range(n_eqs):
        lhs = root(depth)
        rhs = root(depth) if rng.random() < 0.7 else tree(depth)
        eqs.append(Equation(lhs, rhs))
    iface = list(pending)
    rng.shuffle(iface)
    return Configuration(tuple(iface), tuple(eqs))
