"""ORACLE PIN (test infrastructure only): brute-force full transport tensor on micro instances.

Builds M in R_+^{L x N^(T+1)} literally as M = K ⊙ U (eq:MKU P:357-358, thm:solution P:777-781,
node form SURVEY §8.0):

    M[l, v_0, ..., v_T] = U0[l, v_0] * prod_t KW_t[v_t, v_{t+1}] * UT[l, v_T]

with KW_t the dense N x N matrix exp(-C_t/eps) * W_t on arcs and 0 off the graph (C = inf).
Projections are literal sums over all other modes (eq:proj_discrete P:319-321,
eq:proj_discrete_bi P:469-471).  ``brute_sweep`` runs the Sinkhorn scheme of prp:sinkhorn
(eq:sinkhorn_graph_E / _Vineq) with every projection taken from the full tensor,
in the Gauss-Seidel order of Algorithm 2 (U0 block, W_0..W_{T-1} blocks, UT block).
Linear domain float64: only for instances where no product under- or overflows (micro sizes).
"""
from __future__ import annotations

import numpy as np


def dense_kernel(problem, t: int, W_t: np.ndarray) -> np.ndarray:
    """N x N matrix with exp(-C_t[a]/eps) * W_t[a] at (tail_a, head_a), 0 elsewhere."""
    p = problem
    K = np.zeros((p.N, p.N))
    K[p.tail, p.head] = np.exp(-np.asarray(p.cost_t(t), float) / p.eps) * W_t
    return K


def full_tensor(problem, U0: np.ndarray, W: np.ndarray, UT: np.ndarray, Un: np.ndarray = None) -> np.ndarray:
    """M with shape (L, N, ..., N) (T+1 node modes).  With commodity node costs c[l, j] (NEXT-2, reading R-N) every
    intermediate mode t = 1..T-1 is also multiplied by exp(-c[l, v_t]/eps) (the commodity-dependent K_L of
    eq:K_multicommodity)."""
    p = problem
    nc = getattr(p, "node_cost", None)
    M = U0.copy()                                   # (L, N)
    for t in range(p.T):
        KW = dense_kernel(p, t, W[t])
        M = M[..., :, None] * KW.reshape((1,) * (M.ndim - 1) + KW.shape)
        if nc is not None and t + 1 <= p.T - 1:     # mode t + 1 is an intermediate layer
            Dl = np.exp(-np.asarray(nc, float) / p.eps)          # (L, N)
            M = M * Dl.reshape((p.L,) + (1,) * (M.ndim - 2) + (p.N,))
        if Un is not None and t + 1 <= p.T - 1:     # node-capacity duals u_{t+1} (NEXT-3)
            M = M * np.asarray(Un[t + 1], float).reshape((1,) * (M.ndim - 1) + (p.N,))
    return M * UT.reshape((p.L,) + (1,) * (p.T) + (p.N,))


def commodity_marginal(M: np.ndarray, mode: int) -> np.ndarray:
    """P_{c,mode}(M): [L, N], summing every node mode except ``mode`` (0..T)."""
    axes = tuple(k for k in range(1, M.ndim) if k != mode + 1)
    return M.sum(axis=axes)


def bimarginal(M: np.ndarray, t: int) -> np.ndarray:
    """P_{t,t+1}(M) per commodity: [L, N, N]."""
    axes = tuple(k for k in range(1, M.ndim) if k not in (t + 1, t + 2))
    return M.sum(axis=axes)


def arc_flows(problem, M: np.ndarray) -> np.ndarray:
    """Aggregate arc flows F_t[a] = sum_l P_{t,t+1}(M^l)[tail_a, head_a]: [T, A]."""
    p = problem
    return np.stack([bimarginal(M, t).sum(axis=0)[p.tail, p.head] for t in range(p.T)])


def commodity_arc_flows(problem, M: np.ndarray, t: int) -> np.ndarray:
    p = problem
    return bimarginal(M, t)[:, p.tail, p.head].T      # [A, L]


def _ratio(num: np.ndarray, den: np.ndarray) -> np.ndarray:
    """num/den with 0/0 := 0 and x/0 := +inf (x > 0)."""
    out = np.zeros_like(num, dtype=float)
    pos = den > 0
    out[pos] = num[pos] / den[pos]
    out[(~pos) & (num > 0)] = np.inf
    return out


class BruteState:
    def __init__(self, problem):
        p = problem
        self.p = p
        self.U0 = np.ones((p.L, p.N))
        self.W = np.ones((p.T, p.A))
        self.UT = (p.muT > 0).astype(float)     # Q7: all-ones on the support
        self.Un = np.ones((p.T + 1, p.N)) if getattr(p, "node_cap", None) is not None else None
        self.sweeps = 0

    def tensor(self):
        return full_tensor(self.p, self.U0, self.W, self.UT, self.Un)


def _brute_w_block(bs: BruteState, t: int) -> None:
    """u_t <- min(u_t ⊙ d ./ P_t(K⊙U), 1) with the step-t bimarginals of the full tensor (eq:sinkhorn_graph_Vineq)."""
    p = bs.p
    F = arc_flows(p, bs.tensor())[t]
    cap = np.asarray(p.cap_t(t), float)
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio = np.where(F > 0, cap / np.where(F > 0, F, 1.0), np.inf)
    with np.errstate(invalid="ignore"):
        neww = np.minimum(bs.W[t] * ratio, 1.0)
    neww = np.where(cap == 0, 0.0, neww)
    neww = np.where(np.isinf(cap), 1.0, neww)
    bs.W[t] = neww


def _brute_node_block(bs: BruteState, t: int) -> None:
    """u_t <- min(u_t ⊙ d_t ./ P_t(K⊙U), 1) on the node marginal of layer t summed over the commodities."""
    p = bs.p
    P = commodity_marginal(bs.tensor(), t).sum(axis=0)
    nc = np.asarray(p.node_cap, float)
    d = nc if nc.ndim == 1 else nc[t]
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio = np.where(P > 0, d / np.where(P > 0, P, 1.0), np.inf)
    with np.errstate(invalid="ignore"):
        new = np.minimum(bs.Un[t] * ratio, 1.0)
    new = np.where(d == 0, 0.0, new)
    new = np.where(np.isinf(d), 1.0, new)
    bs.Un[t] = new


def brute_sweep_symmetric(bs: BruteState) -> None:
    """Symmetric GS (NEXT-1): the GS sweep's blocks, then W_{T-1} .. W_0 again, every projection from the full tensor."""
    brute_sweep(bs)
    for t in range(bs.p.T - 1, -1, -1):
        _brute_w_block(bs, t)


def brute_sweep(bs: BruteState) -> None:
    """One GS sweep of eq:sinkhorn_graph with projections of the full tensor."""
    p = bs.p
    # U^(0,1) block: U <- U ⊙ R ./ P_{0,1}(K⊙U)   (eq:sinkhorn_graph_E)
    P0 = commodity_marginal(bs.tensor(), 0)
    r = _ratio(p.mu0, P0)
    if np.isinf(r).any():
        raise RuntimeError("infeasible source")
    bs.U0 = bs.U0 * r
    # u_t blocks: u <- min(u ⊙ d ./ P_t(K⊙U), 1)   (eq:sinkhorn_graph_Vineq)
    for t in range(p.T):
        _brute_w_block(bs, t)
        if bs.Un is not None and t + 1 <= p.T - 1:  # node-capacity block of layer t + 1 (NEXT-3)
            _brute_node_block(bs, t + 1)
    # U^(0,T) block
    PT = commodity_marginal(bs.tensor(), p.T)
    r = _ratio(p.muT, PT)
    if np.isinf(r).any():
        raise RuntimeError("infeasible sink")
    bs.UT = bs.UT * r
    bs.sweeps += 1


# ---------------------------------------------------------------------------------------------------------------
# NEXT-4 entry / exit times (rem:multi_tensor_scheme P:1139-1149): one transport tensor per commodity l
# over its own layers t_in[l] .. t_out[l] (eq:multicommodity_tensor_problem), the capacity duals shared.

def commodity_window_tensor(problem, l: int, U0_l, W, UT_l) -> np.ndarray:
    """M^l[v_{t_in}, ..., v_{t_out}] = U0[v_{t_in}] prod_{t = t_in}^{t_out - 1} KW_t[v_t, v_{t+1}]
    (x exp(-c[l, v_s]/eps) at every layer s of the window that is an intermediate layer 1..T-1 of the horizon)
    UT[v_{t_out}]."""
    p = problem
    t0, t1 = int(p.t_in[l]), int(p.t_out[l])
    nc = getattr(p, "node_cost", None)
    M = np.asarray(U0_l, float).copy()
    if nc is not None and 1 <= t0 <= p.T - 1:  # (the entry layer is an intermediate layer of the horizon)
        M = M * np.exp(-np.asarray(nc[l], float) / p.eps)
    for t in range(t0, t1):
        KW = dense_kernel(p, t, W[t])
        M = M[..., :, None] * KW.reshape((1,) * (M.ndim - 1) + KW.shape)
        if nc is not None and t + 1 <= p.T - 1:
            M = M * np.exp(-np.asarray(nc[l], float) / p.eps).reshape((1,) * (M.ndim - 1) + (p.N,))
    return M * np.asarray(UT_l, float).reshape((1,) * (M.ndim - 1) + (p.N,))


class BruteTimes:
    """Gauss-Seidel Sinkhorn (prp:sinkhorn; the order of eq:Sinkhorn_multi_tensor P:1141-1145: u_1^l, u_t, u_T^l) on
    the per-commodity window tensors, every projection a literal sum."""

    def __init__(self, problem):
        p = problem
        self.p = p
        self.U0 = np.ones((p.L, p.N))
        self.W = np.ones((p.T, p.A))
        self.UT = (p.muT > 0).astype(float)

    def tensors(self):
        return [commodity_window_tensor(self.p, l, self.U0[l], self.W, self.UT[l]) for l in range(self.p.L)]

    def flows(self):
        """Aggregate arc flows F_t[a] (zero outside each commodity's window): [T, A]."""
        p = self.p
        F = np.zeros((p.T, p.A))
        for l, M in enumerate(self.tensors()):
            t0 = int(p.t_in[l])
            for t in range(t0, int(p.t_out[l])):
                k = t - t0
                axes = tuple(x for x in range(M.ndim) if x not in (k, k + 1))
                B = M.sum(axis=axes)
                F[t] += B[p.tail, p.head]
        return F

    def sweep(self):
        p = self.p
        for l, M in enumerate(self.tensors()):       # u_1^l blocks: source marginal at layer t_in
            P0 = M.sum(axis=tuple(range(1, M.ndim)))
            r = _ratio(p.mu0[l], P0)
            if np.isinf(r).any():
                raise RuntimeError("infeasible source")
            self.U0[l] = self.U0[l] * r
        for t in range(p.T):                          # u_t blocks: shared capacity duals
            F = self.flows()[t]
            cap = np.asarray(p.cap_t(t), float)
            with np.errstate(invalid="ignore", divide="ignore"):
                ratio = np.where(F > 0, cap / np.where(F > 0, F, 1.0), np.inf)
            with np.errstate(invalid="ignore"):
                neww = np.minimum(self.W[t] * ratio, 1.0)
            neww = np.where(cap == 0, 0.0, neww)
            neww = np.where(np.isinf(cap), 1.0, neww)
            self.W[t] = neww
        for l, M in enumerate(self.tensors()):       # u_T^l blocks: sink marginal at layer t_out
            PT = M.sum(axis=tuple(range(M.ndim - 1)))
            r = _ratio(p.muT[l], PT)
            if np.isinf(r).any():
                raise RuntimeError("infeasible sink")
            self.UT[l] = self.UT[l] * r
