"""State spaces of the paper's network-flow formulations as node-form problems.

The paper writes the multi-commodity problem over *states* (§3.2, eq:multicommodity P:659-683): a state
is a directed edge, transitions i -> j are allowed when C_ij < inf ("C_ij = 0 if edge i leads to edge
j"), commodities pay C_L[l, i] for being on state i at the intermediate times, and the capacities bound
the state marginals, P_t(M) <= d_t.  §3.3 adds staying on an edge, vertex storage (states E u V) and
the traffic-routing state space (E u S+ u S-).  Every one of them is the library's node form on a *state graph*:
nodes = states, arcs = allowed transitions (cost C_ij), node costs = C_L (NEXT-2), node capacities = d (NEXT-3),
sources / sinks = point masses or distributions on states.  This module builds those state graphs from a road
network; it holds no arithmetic of the method (graph combinatorics only) and is shared by the oracle tests and the
GPU runs like workloads/configs.py.

Readings (reading R-S):
- edges:           e -> f iff head(e) = tail(f)                                   ("leads to")
- edges+stay:      edges, plus e -> e with the staying cost (may be negative)
- vertex_storage:  E u V; e -> f as above, e -> head(e), v -> out-edges(v), v -> v ("a vertex is adjacent
                   to all edges it connects to, and to itself", directed along the edges)
- traffic:         E u S+ u S-; Source(v) -> {Source(v), out-edges(v)}, e -> {successor edges, e, Sink(head(e))},
                   Sink(v) -> {Sink(v)}: sinks absorbing (the prose of P:714-720 / SPEC S:86, not the garbled formula)
"""
from __future__ import annotations

import numpy as np

from .configs import Problem


def street_map(seed: int = 0, rows: int = 8, cols: int = 8, drop_nodes: int = 7, n_undirected: int = 75):
    """A synthetic street network in the size of the paper's §5.3 map (57 vertices, 150 directed edges, P:1224-1230;
    the map itself is unpublished): a jittered rows x cols grid with ``drop_nodes`` junctions removed and
    two-way streets removed at random down to ``n_undirected`` while staying connected.  Returns (N, tail, head,
    length, xy) with lengths = Euclidean distances of the jittered coordinates."""
    rng = np.random.default_rng(seed)
    xy = np.array([(c, r) for r in range(rows) for c in range(cols)], float)
    xy += rng.uniform(-0.25, 0.25, size=xy.shape)
    keep = np.ones(rows * cols, bool)
    keep[rng.choice(rows * cols, size=drop_nodes, replace=False)] = False
    und = []
    for r in range(rows):
        for c in range(cols):
            u = r * cols + c
            for v in ((u + 1) if c + 1 < cols else -1, (u + cols) if r + 1 < rows else -1):
                if v >= 0 and keep[u] and keep[v]:
                    und.append((u, v))
    und = np.array(und)
    ids = -np.ones(rows * cols, int)
    ids[keep] = np.arange(keep.sum())
    N = int(keep.sum())

    def connected(edges):
        adj = [[] for _ in range(N)]
        for a, b in edges:
            adj[ids[a]].append(ids[b])
            adj[ids[b]].append(ids[a])
        seen = {0}
        stack = [0]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if y not in seen:
                    seen.add(y)
                    stack.append(y)
        return len(seen) == N

    assert connected(und), "grid minus the dropped junctions must stay connected"
    order = rng.permutation(len(und))
    cur = list(map(tuple, und))
    for k in order:
        if len(cur) <= n_undirected:
            break
        trial = [e for e in cur if e != tuple(und[k])]
        if connected(trial):
            cur = trial
    und = np.array(cur)
    tail = np.concatenate([ids[und[:, 0]], ids[und[:, 1]]]).astype(np.int32)
    head = np.concatenate([ids[und[:, 1]], ids[und[:, 0]]]).astype(np.int32)
    pos = xy[keep]
    length = np.linalg.norm(pos[tail] - pos[head], axis=1)
    return N, tail, head, length, pos


def state_graph(N: int, tail, head, policy: str, stay_cost: float = 0.0, sources=(), sinks=()):
    """States and allowed transitions of a road network (N vertices, directed edges tail -> head) under ``policy``
    (module docstring).  Returns (n_states, st_tail, st_head, st_cost, kind, ref) where kind[s] in {"E", "V", "S+",
    "S-"} and ref[s] is the edge id (kind E) or vertex id of state s; transition costs are 0 except staying on an
    edge (edges+stay, traffic: stay_cost).  Traffic routing needs the source / sink vertices (S+, S- states)."""
    tail = np.asarray(tail)
    head = np.asarray(head)
    E = tail.size
    kind = ["E"] * E
    ref = list(range(E))
    out_edges = [[] for _ in range(N)]
    for e in range(E):
        out_edges[tail[e]].append(e)
    st_t, st_h, st_c = [], [], []

    def tr(a, b, c=0.0):
        st_t.append(a)
        st_h.append(b)
        st_c.append(c)

    for e in range(E):  # edge -> successor edges (head(e) = tail(f); u-turns included)
        for f in out_edges[head[e]]:
            tr(e, f)
    if policy in ("edges+stay", "traffic"):
        for e in range(E):
            tr(e, e, stay_cost)
    if policy == "vertex_storage":
        base = E
        kind += ["V"] * N
        ref += list(range(N))
        for e in range(E):
            tr(e, base + head[e])
        for v in range(N):
            tr(base + v, base + v)
            for f in out_edges[v]:
                tr(base + v, f)
    elif policy == "traffic":
        sp = {v: E + k for k, v in enumerate(sorted(set(sources)))}
        sm = {v: E + len(sp) + k for k, v in enumerate(sorted(set(sinks)))}
        kind += ["S+"] * len(sp) + ["S-"] * len(sm)
        ref += sorted(sp) + sorted(sm)
        for v, s in sp.items():
            tr(s, s)
            for f in out_edges[v]:
                tr(s, f)
        for e in range(E):
            if head[e] in sm:
                tr(e, sm[head[e]])
        for v, s in sm.items():
            tr(s, s)
    elif policy not in ("edges", "edges+stay"):
        raise ValueError(policy)
    n = len(kind)
    return n, np.array(st_t, np.int32), np.array(st_h, np.int32), np.array(st_c, float), np.array(kind), np.array(ref)


def state_problem(policy: str, T: int, eps: float, seed: int = 0, L: int = None, edge_cap=(0.5, 1.5),
                  vertex_cap: float = None, commodity_costs: bool = True, stay_cost: float = 0.0,
                  net=None) -> Problem:
    """A dynamic multi-commodity problem over the states of a (synthetic) street map, P:1224-1303 in synthetic form:
    L point-mass commodities between random vertex pairs with unit mass (traffic: Source(s) -> Sink(g); vertex
    storage: vertex states; edges / edges+stay: an out-edge of s -> an in-edge of g), commodity state costs
    C_L[l, s] = edge length * U[0.5, 1.5] (per commodity and edge; 0 on vertex / source / sink states) charged at the
    intermediate layers (node costs), state capacities d = U[edge_cap] on edge states (vertex states: vertex_cap,
    default free), transitions free except staying."""
    N, tail, head, length, pos = net if net is not None else street_map(seed)
    rng = np.random.default_rng(seed + 1000)
    L = N if L is None else L
    # OD pairs: distinct vertices within T - 2 hops (the traffic / edge states add up to two boundary steps)
    adj = [[] for _ in range(N)]
    for a, b in zip(tail, head):
        adj[a].append(b)

    def hops(s):
        d = np.full(N, 10 ** 9)
        d[s] = 0
        q = [s]
        for x in q:
            for y in adj[x]:
                if d[y] > d[x] + 1:
                    d[y] = d[x] + 1
                    q.append(y)
        return d

    src, dst = [], []
    while len(src) < L:
        s, g = rng.integers(0, N, size=2)
        if s != g and 1 <= hops(s)[g] <= T - 3:
            src.append(int(s))
            dst.append(int(g))
    n, st_t, st_h, st_c, kind, ref = state_graph(N, tail, head, policy, stay_cost, src, dst)
    is_edge = kind == "E"
    if policy == "traffic":
        sp = {int(v): k for k, v in zip(np.flatnonzero(kind == "S+"), ref[kind == "S+"])}
        sm = {int(v): k for k, v in zip(np.flatnonzero(kind == "S-"), ref[kind == "S-"])}
        s_state = [sp[s] for s in src]
        g_state = [sm[g] for g in dst]
    elif policy == "vertex_storage":
        s_state = [int(np.flatnonzero((kind == "V") & (ref == s))[0]) for s in src]
        g_state = [int(np.flatnonzero((kind == "V") & (ref == g))[0]) for g in dst]
    else:
        s_state = [int(rng.choice(np.flatnonzero(is_edge & (tail[np.minimum(ref, tail.size - 1)] == s)))) for s in src]
        g_state = [int(rng.choice(np.flatnonzero(is_edge & (head[np.minimum(ref, tail.size - 1)] == g)))) for g in dst]
    node_cost = np.zeros((L, n))
    if commodity_costs:
        node_cost[:, is_edge] = length[ref[is_edge]][None, :] * rng.uniform(0.5, 1.5, size=(L, int(is_edge.sum())))
    node_cap = np.full(n, np.inf)
    node_cap[is_edge] = rng.uniform(edge_cap[0], edge_cap[1], size=int(is_edge.sum()))
    if vertex_cap is not None:
        node_cap[kind == "V"] = vertex_cap
    A = st_t.size
    return Problem(name=f"{policy}-street{N}-T{T}-L{L}", N=n, tail=st_t, head=st_h, T=T, eps=eps, cost=st_c,
                   cap=np.full(A, np.inf), L=L, src=np.array(s_state, np.int32), dst=np.array(g_state, np.int32),
                   mass=np.ones(L), node_cost=node_cost, node_cap=node_cap, prec="fp32", sweeps=10,
                   meta={"policy": policy, "readings": "R-S", "vertices": N, "edges": int(tail.size)})
