"""ORACLE PIN (test infrastructure only): exact LP on the time-expanded network.

The unregularised dynamic multi-commodity min-cost flow (eq:flow_dynamic_multi-commodity P:273-280,
equivalent to eq:multicommodity by thm:equiv_mc) written in node-arc form on the
time-expanded network N_exp: one variable x[l, t, a] >= 0 per commodity, step and arc;
conservation at every time-expanded node (t, v), 1 <= t <= T-1; sources at layer 0 and sinks at
layer T; capacity sum_l x[l, t, a] <= d_t[a] on capacitated arcs.  Solved by SciPy's HiGHS.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog


def time_expanded_counts(problem) -> tuple:
    """(#vertices, #edges) of N_exp: (T+1)|V| and T|A|."""
    return (problem.T + 1) * problem.N, problem.T * problem.A


def build_lp(problem):
    p = problem
    L, T, A, N = p.L, p.T, p.A, p.N
    nv = L * T * A

    def var(l, t):
        return (l * T + t) * A + np.arange(A)

    rows, cols, vals, rhs = [], [], [], []
    r = 0
    mu0, muT = p.mu0, p.muT
    for l in range(L):
        # layer 0: out-flow of node v = mu0[l, v]
        v0 = var(l, 0)
        rows.append(r + p.tail)
        cols.append(v0)
        vals.append(np.ones(A))
        rhs.append(mu0[l])
        r += N
        # layers 1..T-1: in-flow(t-1) - out-flow(t) = 0
        for t in range(1, T):
            rows.append(r + p.head)
            cols.append(var(l, t - 1))
            vals.append(np.ones(A))
            rows.append(r + p.tail)
            cols.append(var(l, t))
            vals.append(-np.ones(A))
            rhs.append(np.zeros(N))
            r += N
        # layer T: in-flow = muT[l, v]
        rows.append(r + p.head)
        cols.append(var(l, T - 1))
        vals.append(np.ones(A))
        rhs.append(muT[l])
        r += N
    A_eq = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(r, nv))
    b_eq = np.concatenate(rhs)
    urows, ucols, ub = [], [], []
    ru = 0
    for t in range(T):
        cap = np.asarray(p.cap_t(t), float)
        capped = np.flatnonzero(np.isfinite(cap))
        for k, a in enumerate(capped):
            for l in range(L):
                urows.append(ru + k)
                ucols.append(var(l, t)[a])
        ub.append(cap[capped])
        ru += capped.size
    A_ub = sp.csr_matrix((np.ones(len(urows)), (urows, ucols)), shape=(ru, nv)) if ru else None
    b_ub = np.concatenate(ub) if ru else None
    c = np.concatenate([np.tile(np.asarray(p.cost_t(t), float), 1) for l in range(L) for t in range(T)])
    return c, A_eq, b_eq, A_ub, b_ub


def solve_lp(problem) -> dict:
    c, A_eq, b_eq, A_ub, b_ub = build_lp(problem)
    res = linprog(c, A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    return {"status": res.status, "opt": float(res.fun) if res.status == 0 else None, "x": res.x,
            "n_var": c.size, "n_eq": A_eq.shape[0], "n_ub": 0 if A_ub is None else A_ub.shape[0]}


def count_walks(problem) -> int:
    """P = number of (commodity, walk) pairs on which the LP / entropic tensor can be nonzero:
    sum_l (A_0 A_1 ... A_{T-1})[s_l, g_l] with integer adjacency matrices (exact Python ints)."""
    p = problem
    total = 0
    adj = [np.zeros((p.N, p.N), dtype=object) for _ in range(p.T)]
    for t in range(p.T):
        cap = np.asarray(p.cap_t(t), float)
        for a in range(p.A):
            if cap[a] != 0:
                adj[t][p.tail[a], p.head[a]] = 1
    mu0, muT = p.mu0, p.muT
    for l in range(p.L):
        v = np.array([1 if x > 0 else 0 for x in mu0[l]], dtype=object)
        for t in range(p.T):
            v = v.dot(adj[t])
        total += int(sum(int(v[j]) for j in range(p.N) if muT[l, j] > 0))
    return total
