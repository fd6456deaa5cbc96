"""Port-graph canonical form of a configuration (test helper).

Two configurations denote the same net when their port graphs are isomorphic
with the interface order kept: agents are nodes with ports 0 (principal) ..
arity, and variables and equations are wires. Port graphs are rigid (fixing
one node fixes its whole connected component), so a breadth-first numbering
from the interface, and for closed components the least numbering over all
start agents, is a canonical form. Used where the printed text may differ
without the net differing: a normal form that keeps cyclic equations is
written from wherever finalize cut each cycle.
"""


def _wires(config):
    """Endpoint pairing: ('i', k) interface slot k, (a, p) port p of agent a."""
    agents = []  # label name per agent
    link = {}  # node -> list of neighbours (wire graph before contraction)

    def add(u, v):
        link.setdefault(u, []).append(v)
        link.setdefault(v, []).append(u)

    def place(slot, term):
        # the wire leaving `slot` reaches `term`
        if not hasattr(term, "sym"):
            add(slot, ("v", term.id))
            return
        a = len(agents)
        agents.append(term.sym.name)
        add(slot, (a, 0))
        for p, child in enumerate(term.children, start=1):
            place((a, p), child)

    for k, t in enumerate(config.interface):
        place(("i", k), t)
    for e, eq in enumerate(config.equations):
        place(("e", e, 0), eq.lhs)
        place(("e", e, 1), eq.rhs)
        add(("e", e, 0), ("e", e, 1))
    # contract pass-through nodes (variables and equation sides have degree 2)
    partner = {}

    def endpoint(n):
        return n[0] == "i" or isinstance(n[0], int)

    for n in list(link):
        if not endpoint(n) or n in partner:
            continue
        prev, cur = n, link[n][0]
        while not endpoint(cur):
            a, b = link[cur]
            prev, cur = cur, (b if a == prev else a)
        partner[n] = cur
        partner[cur] = n
    return agents, partner


def _bfs(starts, agents, partner, arity, order):
    """Number agents breadth-first from `starts` (appending to `order`); encode them."""
    seq = []
    for a in starts:
        if a not in order:
            order[a] = len(order)
            seq.append(a)
    out = []
    i = 0
    while i < len(seq):
        a = seq[i]
        i += 1
        out.append(agents[a])
        for p in range(arity[a] + 1):
            q = partner[(a, p)]
            if q[0] == "i":
                out.append(("i", q[1]))
                continue
            if q[0] not in order:
                order[q[0]] = len(order)
                seq.append(q[0])
            out.append((order[q[0]], q[1]))
    return out


def canonical(config):
    """Canonical form of the net denoted by `config` (see the module docstring)."""
    agents, partner = _wires(config)
    arity = [0] * len(agents)
    for k in partner:
        if isinstance(k[0], int):
            arity[k[0]] = max(arity[k[0]], k[1])
    order = {}
    head = []
    starts = []
    for k in range(len(config.interface)):
        q = partner[("i", k)]
        if q[0] == "i":
            head.append(("i", q[1]))
        else:
            if q[0] not in order and q[0] not in starts:
                starts.append(q[0])
            head.append(("a", starts.index(q[0]) if q[0] in starts else -1, q[1]))
    body = _bfs(starts, agents, partner, arity, order)
    closed = []
    for a in range(len(agents)):
        if a in order:
            continue
        comp = {}
        _bfs([a], agents, partner, arity, comp)
        best = min(tuple(map(repr, _bfs([s], agents, partner, arity, {}))) for s in comp)
        for s in comp:
            order[s] = -1
        closed.append(best)
    return tuple(map(repr, head)), tuple(map(repr, body)), tuple(sorted(closed))
