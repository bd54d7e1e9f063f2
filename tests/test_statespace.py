"""NEXT-3: the paper's state spaces as node-form state graphs (workloads/statespace.py), host logic.

SPEC build_structure_matrix examples and invariants, the §5.3-sized synthetic street map, and an oracle
run on each state space (feasible, capacities and marginals met after convergence-length runs)."""
import numpy as np
import pytest

from workloads.statespace import street_map, state_graph, state_problem


def _support(n, t, h):
    return set(zip(t.tolist(), h.tolist()))


def test_spec_triangle_edges_only():
    """triangle cycle a->b->c->a, EdgesOnly -> support {(ab,bc),(bc,ca),(ca,ab)} (SPEC, head/tail matching)."""
    n, t, h, c, kind, ref = state_graph(3, [0, 1, 2], [1, 2, 0], "edges")
    assert n == 3 and _support(n, t, h) == {(0, 1), (1, 2), (2, 0)} and np.all(c == 0)


def test_spec_chain_traffic_routing():
    """chain Source(s) -> e -> Sink(t), TrafficRouting -> {(s,s),(s,e),(e,e),(e,t),(t,t)} (SPEC, textual rules)."""
    n, t, h, c, kind, ref = state_graph(2, [0], [1], "traffic", sources=[0], sinks=[1])
    s = int(np.flatnonzero(kind == "S+")[0])
    g = int(np.flatnonzero(kind == "S-")[0])
    assert _support(n, t, h) == {(s, s), (s, 0), (0, 0), (0, g), (g, g)}


def test_edges_support_is_brute_force_adjacency_and_traffic_invariants():
    N, tail, head, length, pos = street_map(0)
    assert (N, tail.size) == (57, 150)  # the §5.3 sizes
    n, t, h, c, kind, ref = state_graph(N, tail, head, "edges")
    brute = {(e, f) for e in range(tail.size) for f in range(tail.size) if head[e] == tail[f]}
    assert _support(n, t, h) == brute
    src, dst = [0, 5, 9], [3, 5, 40]
    n, t, h, c, kind, ref = state_graph(N, tail, head, "traffic", sources=src, sinks=dst)
    assert n == tail.size + 3 + 3
    for a, b in zip(t, h):
        if kind[a] == "S-":
            assert b == a  # sinks absorbing
        if kind[b] == "S+":
            assert a == b  # nothing enters a source
    n, t, h, c, kind, ref = state_graph(N, tail, head, "vertex_storage")
    assert n == tail.size + N
    V = np.flatnonzero(kind == "V")
    assert all((v, v) in _support(n, t, h) for v in V)


@pytest.mark.parametrize("policy", ["edges+stay", "vertex_storage", "traffic"])
def test_state_problem_oracle_feasible_and_capacities_bind(policy):
    from oracle import oracle_run, readout_flows, stats
    p = state_problem(policy, T=12, eps=0.1, seed=1, L=6, edge_cap=(0.3, 0.9))
    st = oracle_run(p, 40)
    s = stats(st)
    assert abs(s["mass"] - 6.0) < 1e-9 and s["src_mismatch"] < 1e-3 * 6
    assert np.min(np.exp(st.nu)) < 0.999  # (state capacities bind)
