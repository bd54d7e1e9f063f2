"""ORACLE (test infrastructure only): float64 log-domain Gauss-Seidel Sinkhorn sweep, node form.

Transcribes SURVEY.md §8(c) steps 1-5, which follow Algorithm 2 (alg:multi_commodity, PAPER.md
P:1085-1107) pushed through the node form of SURVEY.md §8.0:

    a = log alpha  (forward messages  Psi-hat, eq:psi_hat P:1031-1036)
    b = log beta   (backward messages Psi,     eq:psi     P:1038-1043)
    lam0 = log U0 (U^(0,1)), lamT = log UT (U^(0,T)), omega = log W (u_t)

State arrays:  lK [T, A] = -C_t/eps ; omega [T, A] ; lam0, lamT [L, N] ; a, b [T+1, L, N].
LSE = log-sum-exp with max shift; -inf encodes an exact zero (thm:solution_extension's zero
entries, eq:u_augment P:843-848).  No blocking, fusion or reordering beyond the algorithm: every
step is a whole-array numpy expression over arcs and commodities (segment sums over the arcs
of a node are a sparse 0/1 incidence-matrix product, a library primitive).

The capacity-dual update is written in Algorithm 2's own form
    u_t <- min( d ./ ((Psi-hat_t ⊙ Psi_t ⊙ K)^T 1), 1 )
i.e. omega_t[a] <- min(log d[a] - LSE_l(a_t[i_a,l] + lK_t[a] + b_{t+1}[j_a,l]), 0), which does not
involve the previous W (prp:sinkhorn P:861 with u_t cancelled).  Zero conventions (SURVEY Q6/Q8,
P:109 "0 * inf = 0"): d = +inf -> W = 1; d = 0 -> W = 0; flow-without-W = 0 and d > 0 -> W = 1;
0/0 := 0 at the boundary scalings; x/0 with x > 0 raises OracleInfeasible.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np
import scipy.sparse as sp

NEG_INF = -np.inf


class OracleInfeasible(RuntimeError):
    """Boundary scaling x/0 with x > 0: a commodity's source (sink) node cannot reach any sink
    (source) node through the current kernel."""

    def __init__(self, where: str, commodity: int, node: int):
        super().__init__(f"infeasible at {where}: commodity {commodity}, node {node}")
        self.where, self.commodity, self.node = where, commodity, node


def _segments(keys: np.ndarray, n: int):
    """Segment structure of arcs grouped by ``keys`` (head for in-arcs, tail for out-arcs):
    arc order sorted by key, per-node counts, start offsets, and the 0/1 incidence matrix S [n, A]
    with S[v, a] = 1 iff keys[a] = v (used as the segment sum, a plain sparse matmul)."""
    order = np.argsort(keys, kind="stable")
    counts = np.bincount(keys, minlength=n)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    S = sp.csr_matrix((np.ones(keys.size), (keys[order], np.arange(keys.size))), shape=(n, keys.size))
    # ELL table of each segment's (sorted) arc positions, padded with A (an appended -inf column),
    # for the segment max
    D = int(counts.max()) if n else 0
    ell = np.full((D, n), keys.size, np.int64)
    pos = np.arange(keys.size) - starts[keys[order]]
    ell[pos, keys[order]] = np.arange(keys.size)
    return order, counts, starts, S, ell


def seg_lse(X: np.ndarray, seg: tuple) -> np.ndarray:
    """out[l, v] = log sum_{a in segment v} exp(X[l, a]) for X [L, A] whose arcs are already in
    segment order; empty segment -> -inf.  Max-shifted per (l, v)."""
    order, counts, starts, S, ell = seg
    n = counts.size
    Xp = np.concatenate([X, np.full((X.shape[0], 1), NEG_INF)], axis=1)
    mx = np.full((X.shape[0], n), NEG_INF)
    for k in range(ell.shape[0]):
        np.maximum(mx, Xp[:, ell[k]], out=mx)
    shift = np.where(np.isfinite(mx), mx, 0.0)
    E = np.exp(X - np.repeat(shift, counts, axis=1))
    s = (S @ E.T).T
    with np.errstate(divide="ignore"):
        out = shift + np.log(s)
    return out


def _lse_rows(X: np.ndarray) -> np.ndarray:
    """LSE over axis 0 (commodities) of an [L, A] array; all -inf column -> -inf."""
    mx = X.max(axis=0)
    shift = np.where(np.isfinite(mx), mx, 0.0)
    with np.errstate(divide="ignore"):
        return shift + np.log(np.exp(X - shift[None, :]).sum(axis=0))


def _log(x: np.ndarray) -> np.ndarray:
    with np.errstate(divide="ignore"):
        return np.log(x)


@dataclasses.dataclass
class OracleState:
    problem: object
    lK: np.ndarray      # [T, A]   log K_t = -C_t / eps           (eq K_multicommodity)
    logd: np.ndarray    # [T, A]   log d_t (+inf free, -inf closed)
    omega: np.ndarray   # [T, A]   log W_t <= 0
    lam0: np.ndarray    # [L, N]   log U0
    lamT: np.ndarray    # [L, N]   log UT
    a: np.ndarray       # [T+1, L, N] log alpha_t (kept from the last forward pass)
    b: np.ndarray       # [T+1, L, N] log beta_t  (from the last backward pass)
    log_mu0: np.ndarray  # [L, N]
    log_muT: np.ndarray  # [L, N]
    in_seg: tuple        # arcs grouped by head (forward recursion)
    out_seg: tuple       # arcs grouped by tail (backward recursion)
    sweeps: int = 0
    keep_forward: bool = True   # False: ``a`` holds only the two latest layers (see _TwoLayers)
    lD: Optional[np.ndarray] = None  # [L, N] -c[l, j]/eps, commodity node costs (NEXT-2), or None
    t_in: Optional[np.ndarray] = None   # [L] entry layer of each commodity (NEXT-4 entry/exit times), or None = 0
    t_out: Optional[np.ndarray] = None  # [L] exit layer, or None = T
    logdn: Optional[np.ndarray] = None  # [T+1, N] log node (state) capacities (NEXT-3), +inf at layers 0 and T; or None
    nu: Optional[np.ndarray] = None     # [T+1, N] log u_t of the node capacities (0 where free)


def _at_layers(arr, layers: np.ndarray) -> np.ndarray:
    """[L, N] slice of a [T+1, L, N] message store taking commodity l at layer layers[l]."""
    return arr[layers, np.arange(layers.size)]


def _src_layer(st) -> np.ndarray:
    return st.t_in if st.t_in is not None else np.zeros(st.problem.L, np.int64)


def _sink_layer(st) -> np.ndarray:
    return st.t_out if st.t_out is not None else np.full(st.problem.L, st.problem.T, np.int64)


def _layer_cost(st: "OracleState", t: int, nu: bool = True):
    """log of the node factors of layer t that multiply every walk through (t, j):
    - the commodity node factor D[l, j] = exp(-c[l, j]/eps) (SURVEY §8(f) NEXT-2 in the form of DESIGN.md reading R-N:
      charged at the intermediate layers 1..T-1 only, so the boundary layers 0 and T carry the marginals alone; the
      commodity-dependent kernel K_L of eq:K_multicommodity P:1010-1013 restricted to costs that depend on the head);
    - (nu) the node-capacity dual u_t[j] = exp(nu_t[j]) (NEXT-3: the capacity of the state marginal P_t(M) <= d_t of
      eq:multicommodity P:676-683, Algorithm 2's u_t), also at the intermediate layers only."""
    T = st.problem.T
    if t < 1 or t > T - 1:
        return 0.0
    out = 0.0
    if st.lD is not None:
        out = st.lD
    if nu and st.nu is not None:
        out = out + st.nu[t][None, :]
    return out


class _TwoLayers:
    """Storage-only variant of the forward-message store ``a`` for instances whose [T+1, L, N] float64
    arrays do not fit in host memory (configs [4], [5] at full size): the sweep reads a_t and writes
    a_{t+1} only, so two layers suffice; layer t lives in slot t % 2.  Readouts recompute the kept
    layers (``forward_layers``) with the same arithmetic.  No step of the method changes."""

    def __init__(self, L: int, N: int):
        self.buf = np.full((2, L, N), NEG_INF)

    def __getitem__(self, t):
        return self.buf[t % 2]

    def __setitem__(self, t, v):
        self.buf[t % 2] = v


def oracle_init(problem, b_store: Optional[np.ndarray] = None, keep_forward: bool = True) -> OracleState:
    """Step 1-2 of SURVEY §8(c): lK = -C/eps (fp64), W = 1, UT = 1 on supp(muT) (Q7),
    then one backward pass (Alg. 2 "Initialize ... Compute Psi_t").

    Storage options (no effect on any value; pinned bitwise by tests/test_oracle_pins.py
    test_storage_options_bitwise_equal): ``b_store`` a caller-provided float64 [T+1, L, N] array for the
    backward messages (e.g. an np.memmap on disk: [4]'s store is 66 GB); ``keep_forward=False`` keeps
    only two forward layers and recomputes the others for readouts."""
    p = problem
    T, A, N, L = p.T, p.A, p.N, p.L
    cost = np.broadcast_to(p.cost, (T, A)) if p.cost.ndim == 1 else p.cost
    cap = np.broadcast_to(p.cap, (T, A)) if p.cap.ndim == 1 else p.cap
    lK = -np.asarray(cost, np.float64) / float(p.eps)
    logd = _log(np.asarray(cap, np.float64))
    mu0 = p.mu0
    muT = p.muT
    if b_store is None:
        b = np.full((T + 1, L, N), NEG_INF)
    else:
        assert b_store.shape == (T + 1, L, N) and b_store.dtype == np.float64
        b = b_store
        for t in range(T + 1):
            b[t] = NEG_INF
    st = OracleState(
        problem=p, lK=lK, logd=logd, omega=np.zeros((T, A)),
        lam0=np.full((L, N), NEG_INF), lamT=np.where(muT > 0, 0.0, NEG_INF),
        a=np.full((T + 1, L, N), NEG_INF) if keep_forward else _TwoLayers(L, N), b=b,
        log_mu0=_log(mu0), log_muT=_log(muT),
        in_seg=_segments(p.head.astype(np.int64), N), out_seg=_segments(p.tail.astype(np.int64), N),
        keep_forward=keep_forward,
        lD=None if getattr(p, "node_cost", None) is None else -np.asarray(p.node_cost, np.float64) / float(p.eps))
    if getattr(p, "node_cap", None) is not None:
        # NEXT-3 state capacities: d_t[j] on the node marginal at the intermediate layers 1..T-1
        nc = np.asarray(p.node_cap, np.float64)
        dn = np.broadcast_to(nc, (T + 1, N)).copy() if nc.ndim == 1 else nc.copy()
        dn[0] = np.inf
        dn[T] = np.inf
        st.logdn = _log(dn)
        st.nu = np.zeros((T + 1, N))
    if getattr(p, "t_in", None) is not None or getattr(p, "t_out", None) is not None:
        # NEXT-4 entry / exit times (rem:multi_tensor_scheme P:1139-1149): commodity l's transport tensor
        # spans the layers t_in[l] .. t_out[l]; its source scaling sits at layer t_in[l], its sink scaling at t_out[l]
        assert keep_forward, "commodity times need the kept forward store"
        st.t_in = np.zeros(L, np.int64) if p.t_in is None else np.asarray(p.t_in, np.int64)
        st.t_out = np.full(L, T, np.int64) if p.t_out is None else np.asarray(p.t_out, np.int64)
        assert np.all((0 <= st.t_in) & (st.t_in < st.t_out) & (st.t_out <= T))
    backward(st)
    return st


def backward(st: OracleState) -> None:
    """Backward recursion (eq:psi P:1038-1043; Alg. 2), node form:
    b_T = lamT ; b_t[l,i] = LSE_{a: i_a = i}( lK_t[a] + omega_t[a] + b_{t+1}[l, j_a] )."""
    p = st.problem
    o = st.out_seg[0]
    head_o = p.head[o]
    tout = _sink_layer(st)
    st.b[p.T] = np.where((tout == p.T)[:, None], st.lamT, NEG_INF)
    for t in range(p.T - 1, -1, -1):
        X = (st.lK[t][o] + st.omega[t][o])[None, :] + (st.b[t + 1] + _layer_cost(st, t + 1))[:, head_o]
        st.b[t] = seg_lse(X, st.out_seg)
        if st.t_out is not None and np.any(tout == t):  # commodities leaving at layer t: beta_t = UT there
            sel = tout == t
            st.b[t][sel] = st.lamT[sel]


def _boundary(log_mu: np.ndarray, msg: np.ndarray, where: str) -> np.ndarray:
    """U = mu ./ msg in logs ([L, N]): 0/0 := 0 (mu = 0 -> -inf); mu > 0 with msg = 0 -> infeasible."""
    with np.errstate(invalid="ignore"):
        lam = np.where(np.isfinite(log_mu), log_mu - msg, NEG_INF)
    bad = np.isfinite(log_mu) & ~np.isfinite(msg)
    if bad.any():
        l, v = np.argwhere(bad)[0]
        raise OracleInfeasible(where, int(l), int(v))
    return lam


def capacity_update(logd_t: np.ndarray, log_ks: np.ndarray) -> np.ndarray:
    """Algorithm 2 line P:1093: omega = min(log d - log(K-weighted bimarginal without W), 0),
    with d = +inf -> 0, d = 0 -> -inf, (d > 0 and flow 0) -> 0."""
    with np.errstate(invalid="ignore"):
        om = np.minimum(logd_t - log_ks, 0.0)
    om = np.where(np.isposinf(logd_t), 0.0, om)
    om = np.where(np.isneginf(logd_t), NEG_INF, om)
    om = np.where(np.isfinite(logd_t) & np.isneginf(log_ks), 0.0, om)
    return om


def _enter(st: OracleState, t: int, nu: bool = True) -> None:
    """Commodities entering at layer t (t_in = t > 0): alpha_t = U0 there (their alpha below t_in is zero, so the
    recursion left -inf in place), times the layer's node factor: a commodity pays its node cost at every
    intermediate layer 1..T-1 of its window, the boundary layers of the window included (reading R-N with times;
    at a boundary layer the factor only rescales U0 / UT, the flows do not depend on it)."""
    if st.t_in is not None and np.any(st.t_in == t):
        sel = st.t_in == t
        lc = np.broadcast_to(_layer_cost(st, t, nu), st.lam0.shape)
        st.a[t][sel] = st.lam0[sel] + lc[sel]


def _src_msg(st: OracleState) -> np.ndarray:
    """log beta-hat at each commodity's entry layer: beta_{t_in} times the node factor of that layer (the source
    marginal at t_in is U0 beta-hat; alpha_{t_in} = U0 times the factor, so alpha_{t_in} beta_{t_in} = mu0 after a2)."""
    b = _at_layers(st.b, st.t_in).copy()
    for t in np.unique(st.t_in):
        sel = st.t_in == t
        b[sel] = b[sel] + np.broadcast_to(_layer_cost(st, int(t)), b.shape)[sel]
    return b


def _mass_now(st: OracleState, t: int, X: Optional[np.ndarray] = None) -> float:
    """Mass <K, U> of the current tensor during a sweep (after the U0 block: t = -1; after W_t: t; after UT: T), per
    commodity from the layer where its messages are current: before its window (t < t_in) lam0 + beta_{t_in}; inside,
    the step-t flows sum_a F^l_t[a] (X are the step's log terms without W); after it (t >= t_out) alpha_{t_out} + lamT."""
    p = st.problem
    tin, tout = _src_layer(st), _sink_layer(st)
    m = np.zeros(p.L)
    pre = np.exp(st.lam0 + (_src_msg(st) if st.t_in is not None else st.b[0])).sum(axis=1)
    if t < 0:
        return float(pre.sum())
    post = np.exp(_at_layers(st.a, tout) + st.lamT).sum(axis=1)
    if t >= p.T:
        return float(post.sum())
    inside = np.exp(X + st.omega[t][None, :]).sum(axis=1)
    m = np.where(t < tin, pre, np.where(t >= tout, post, inside))
    return float(m.sum())


def _node_update(st: OracleState, t: int, on_block: Optional[Callable] = None) -> None:
    """NEXT-3 node (state) capacity block at layer t (1..T-1), Algorithm 2's u_t update on the node marginal:
    nu_t = min(log d_t - LSE_l(a_t + b_t), 0) with a_t without the node factor (the current tensor's marginal at layer t
    up to u_t), the zero conventions of capacity_update; then a_t += nu_t."""
    if st.nu is None or t < 1 or t > st.problem.T - 1:
        return
    X = st.a[t] + st.b[t]
    st.nu[t] = capacity_update(st.logdn[t], _lse_rows(X))
    st.a[t] = st.a[t] + st.nu[t][None, :]
    if on_block is not None:
        assert st.t_in is None and st.t_out is None
        on_block("N", t, float(np.exp(X + st.nu[t][None, :]).sum()))


def oracle_sweep(st: OracleState, on_block: Optional[Callable] = None,
                 reduce_lse: Optional[Callable] = None, _backward: bool = True) -> None:
    """One Gauss-Seidel sweep in Algorithm 2's order.

    on_block(kind, t, mass) is called after every dual block update (kind in {"U0", "W", "UT"}),
    with the tensor mass <K, U> at that moment, for the BCA-monotonicity pin (prp:sinkhorn).

    reduce_lse(v) -> v_global: when the state holds only a slice of the commodities, combines the
    per-arc log flow sums log sum_l exp(X[l, a]) over all slices (the commodities couple only
    through this sum in the capacity update, rem:multi_tensor_scheme P:1139-1147)."""
    p = st.problem
    oi = st.in_seg[0]
    tail_i = p.tail[oi]
    tin, tout = _src_layer(st), _sink_layer(st)
    # a2: U^(0,1) <- R^(0,1) ./ Psi_1, at each commodity's entry layer
    st.lam0 = _boundary(st.log_mu0, _src_msg(st) if st.t_in is not None else st.b[0], "source")
    st.a[0] = st.lam0 if st.t_in is None else np.where((tin == 0)[:, None], st.lam0, NEG_INF)
    if on_block is not None:
        on_block("U0", -1, _mass_now(st, -1))
    # a3: forward loop
    for t in range(p.T):
        X = st.a[t][:, p.tail] + st.lK[t][None, :] + (st.b[t + 1] + _layer_cost(st, t + 1))[:, p.head]  # no W
        lse = _lse_rows(X)
        if reduce_lse is not None:
            lse = reduce_lse(lse)
        st.omega[t] = capacity_update(st.logd[t], lse)
        if on_block is not None:
            on_block("W", t, float(np.exp(X + st.omega[t][None, :]).sum()) if st.t_in is None and st.t_out is None
                     else _mass_now(st, t, X))
        Y = st.a[t][:, tail_i] + (st.lK[t][oi] + st.omega[t][oi])[None, :]
        st.a[t + 1] = seg_lse(Y, st.in_seg) + _layer_cost(st, t + 1, nu=False)  # Psi-hat_{t+1}
        _enter(st, t + 1, nu=False)
        _node_update(st, t + 1, on_block)                                       # u_{t+1} (states)
    # a4: U^(0,T) <- R^(0,T) ./ Psi-hat_T, at each commodity's exit layer
    st.lamT = _boundary(st.log_muT, _at_layers(st.a, tout) if st.t_out is not None else st.a[p.T], "sink")
    if on_block is not None:
        on_block("UT", p.T, _mass_now(st, p.T))
    # a5: backward recompute
    if _backward:
        backward(st)
    st.sweeps += 1


def damped_update(omega_old: np.ndarray, omega_full: np.ndarray, theta: float) -> np.ndarray:
    """W <- W^(1 - theta) * min(W d / F, 1)^theta, in logs; an exact zero stays zero
    (0^x = 0 for x > 0), theta = 1 is the undamped update."""
    if theta == 1.0:
        return omega_full.copy()
    with np.errstate(invalid="ignore"):
        om = (1.0 - theta) * omega_old + theta * omega_full
    return np.where(np.isneginf(omega_old) | np.isneginf(omega_full), NEG_INF, om)


def oracle_sweep_jacobi(st: OracleState, theta: float) -> None:
    """One sweep of the bulk-coupled (Jacobi) schedule of SURVEY §8(f) NEXT-1: every W_t is updated from the
    same alpha/beta pair — the forward pass computes alpha_{t+1} with the W_t of the previous sweep and the
    flows F_t from (alpha_t, beta_{t+1}) — then damped, W <- W^(1 - theta) min(W d / F, 1)^theta; then the
    sink scaling and the backward pass as in Algorithm 2."""
    p = st.problem
    oi = st.in_seg[0]
    tail_i = p.tail[oi]
    assert st.nu is None, "node capacities: Gauss-Seidel schedules only"
    tin, tout = _src_layer(st), _sink_layer(st)
    st.lam0 = _boundary(st.log_mu0, _src_msg(st) if st.t_in is not None else st.b[0], "source")
    st.a[0] = st.lam0 if st.t_in is None else np.where((tin == 0)[:, None], st.lam0, NEG_INF)
    new_omega = np.empty_like(st.omega)
    for t in range(p.T):
        X = st.a[t][:, p.tail] + st.lK[t][None, :] + (st.b[t + 1] + _layer_cost(st, t + 1))[:, p.head]
        full = capacity_update(st.logd[t], _lse_rows(X))
        new_omega[t] = damped_update(st.omega[t], full, theta)
        Y = st.a[t][:, tail_i] + (st.lK[t][oi] + st.omega[t][oi])[None, :]   # (the previous W_t)
        st.a[t + 1] = seg_lse(Y, st.in_seg) + _layer_cost(st, t + 1)
        _enter(st, t + 1)
    st.omega = new_omega
    st.lamT = _boundary(st.log_muT, _at_layers(st.a, tout) if st.t_out is not None else st.a[p.T], "sink")
    backward(st)
    # readouts (edge flows, mass) are projections of the end-of-sweep tensor M(U0, W, UT): keep the forward
    # messages of that tensor, i.e. recomputed with the new W (under Gauss-Seidel the pass's own messages
    # already are; DESIGN.md §2 reading R-J)
    # (unchanged in the kept store; the two-layer store has overwritten slot 0)
    st.a[0] = st.lam0 if st.t_in is None else np.where((tin == 0)[:, None], st.lam0, NEG_INF)
    for t in range(p.T):
        Y = st.a[t][:, tail_i] + (st.lK[t][oi] + st.omega[t][oi])[None, :]
        st.a[t + 1] = seg_lse(Y, st.in_seg) + _layer_cost(st, t + 1)
        _enter(st, t + 1)
    st.sweeps += 1


def oracle_sweep_symmetric(st: OracleState, on_block: Optional[Callable] = None) -> None:
    """One sweep of the symmetric Gauss-Seidel schedule: Algorithm 2's forward pass (U0 block,
    W_0 .. W_{T-1} blocks, UT block), then a backward pass that updates every W_t again before forming
    beta_t (blocks W_{T-1} .. W_0): each update is the same exact block maximisation (prp:sinkhorn P:861, in
    Algorithm 2's form P:1093) on the current tensor, so any such cyclic block order is a valid BCA order
    (P:853-891).  Readouts use forward messages recomputed with the final W (reading R-J)."""
    p = st.problem
    oracle_sweep(st, on_block=on_block, _backward=False)
    o = st.out_seg[0]
    head_o = p.head[o]
    tout = _sink_layer(st)
    st.b[p.T] = np.where((tout == p.T)[:, None], st.lamT, NEG_INF)
    for t in range(p.T - 1, -1, -1):
        bh = st.b[t + 1] + _layer_cost(st, t + 1)
        X = st.a[t][:, p.tail] + st.lK[t][None, :] + bh[:, p.head]            # current tensor, no W
        st.omega[t] = capacity_update(st.logd[t], _lse_rows(X))
        if on_block is not None:
            on_block("W", t, _mass_now(st, t, X) if st.t_in is not None or st.t_out is not None
                     else float(np.exp(X + st.omega[t][None, :]).sum()))
        Xb = (st.lK[t][o] + st.omega[t][o])[None, :] + bh[:, head_o]
        st.b[t] = seg_lse(Xb, st.out_seg)                                        # Psi_t with the new W_t
        if st.t_out is not None and np.any(tout == t):
            sel = tout == t
            st.b[t][sel] = st.lamT[sel]
    # forward messages of the end-of-sweep tensor (every W_t changed after its alpha_{t+1} was formed)
    oi = st.in_seg[0]
    tail_i = p.tail[oi]
    st.a[0] = st.lam0 if st.t_in is None else np.where((_src_layer(st) == 0)[:, None], st.lam0, NEG_INF)
    for t in range(p.T):
        Y = st.a[t][:, tail_i] + (st.lK[t][oi] + st.omega[t][oi])[None, :]
        st.a[t + 1] = seg_lse(Y, st.in_seg) + _layer_cost(st, t + 1)
        _enter(st, t + 1)


def oracle_run(problem, sweeps: int, schedule: str = "gs", theta: float = 1.0) -> OracleState:
    """sweeps of Algorithm 2 (schedule "gs"), of the damped Jacobi schedule ("jacobi") or of the symmetric
    Gauss-Seidel schedule ("sym"), SURVEY §8(f) NEXT-1."""
    st = oracle_init(problem)
    for _ in range(sweeps):
        if schedule == "gs":
            oracle_sweep(st)
        elif schedule == "sym":
            oracle_sweep_symmetric(st)
        else:
            oracle_sweep_jacobi(st, theta)
    return st


def forward_layers(st: OracleState, t_stop: Optional[int] = None):
    """Yields (t, a_t) for t = 0..t_stop (default T): the forward messages of the end-of-sweep tensor.
    Kept store: the last pass's own layers.  Two-layer store: recomputed from (lam0, omega) by the
    forward recursion a_{t+1} = LSE_{a -> j}(a_t[i_a] + lK_t[a] + omega_t[a]) (eq:psi_hat P:1031-1036),
    the sweep's own expression on the same operands (under Gauss-Seidel omega_t is final once alpha_{t+1}
    is formed; under Jacobi the sweep recomputes them with the new omega, reading R-J), hence bitwise
    the same layers."""
    p = st.problem
    t_stop = p.T if t_stop is None else t_stop
    if st.keep_forward:
        for t in range(t_stop + 1):
            yield t, st.a[t]
        return
    assert st.t_in is None, "commodity times need the kept forward store"
    cur = st.lam0                       # a_0 = lam0 (all -inf before the first sweep)
    oi = st.in_seg[0]
    tail_i = p.tail[oi]
    for t in range(t_stop + 1):
        yield t, cur
        if t < t_stop:
            Y = cur[:, tail_i] + (st.lK[t][oi] + st.omega[t][oi])[None, :]
            cur = seg_lse(Y, st.in_seg) + _layer_cost(st, t + 1)


def _commodity_flows_at(st: OracleState, t: int, a_t: np.ndarray) -> np.ndarray:
    p = st.problem
    return np.exp(a_t[:, p.tail] + (st.lK[t] + st.omega[t])[None, :] + (st.b[t + 1] + _layer_cost(st, t + 1))[:, p.head]).T


def readout_commodity_flows(st: OracleState, t: int) -> np.ndarray:
    """Per-commodity arc flow F^l_t[a] = alpha_t[i_a,l] K_t[a] W_t[a] beta_{t+1}[j_a,l]
    (cor:proj P:1078 in node form), from the kept forward messages and the latest backward pass."""
    if st.keep_forward:
        return _commodity_flows_at(st, t, st.a[t])
    for tt, a_t in forward_layers(st, t):
        if tt == t:
            return _commodity_flows_at(st, t, a_t)


def readout_flows(st: OracleState) -> tuple:
    """(F [T, A], W [T, A]) : aggregate edge flows F_t[a] = sum_l F^l_t[a] and capacity duals."""
    p = st.problem
    F = np.stack([_commodity_flows_at(st, t, a_t).sum(axis=1)
                  for t, a_t in forward_layers(st, p.T - 1)]) if p.T else np.zeros((0, p.A))
    return F, np.exp(st.omega)


def dual_terms(st: OracleState) -> tuple:
    """The three linear terms of the dual objective (eq:omt_multi_graph_dual P:786-788, node form,
    lambda = -eps log u): (sum mu0*lam0, sum muT*lamT, sum d*omega), with 0 * (+-inf) = 0."""
    p = st.problem
    mu0, muT = p.mu0, p.muT
    cap = np.broadcast_to(p.cap, st.omega.shape)
    s0 = np.where(mu0 > 0, mu0 * np.where(np.isfinite(st.lam0), st.lam0, 0.0), 0.0).sum()
    sT = np.where(muT > 0, muT * np.where(np.isfinite(st.lamT), st.lamT, 0.0), 0.0).sum()
    fin = np.isfinite(cap) & (cap > 0)
    sd = (np.where(fin, cap, 0.0) * np.where(fin, st.omega, 0.0)).sum()
    if st.nu is not None:  # node capacities (NEXT-3): sum_t <d_t, log u_t> over the finite positive ones
        dn = np.exp(st.logdn)
        finn = np.isfinite(dn) & (dn > 0)
        sd = sd + (np.where(finn, dn, 0.0) * np.where(finn, st.nu, 0.0)).sum()
    return s0, sT, sd


def dual_objective(st: OracleState, mass: float) -> float:
    """Dual objective of thm:solution (eq:omt_multi_graph_dual P:786-788) in node form with
    U = exp(-Lambda/eps):  Phi = -eps*mass + eps*[sum mu0*lam0 + sum muT*lamT + sum d*omega],
    with 0 * (+-inf) = 0."""
    s0, sT, sd = dual_terms(st)
    return float(st.problem.eps * (-mass + s0 + sT + sd))


def stats(st: OracleState) -> dict:
    """End-of-sweep statistics."""
    p = st.problem
    F, W = readout_flows(st)
    cost = np.broadcast_to(p.cost, F.shape)
    cap = np.broadcast_to(p.cap, F.shape)
    # source / sink marginals of the end-of-sweep tensor (at each commodity's entry / exit layer)
    P0 = np.exp(st.lam0 + (_src_msg(st) if st.t_in is not None else st.b[0]))
    PT = np.exp((_at_layers(st.a, st.t_out) if st.t_out is not None else st.a[p.T]) + st.lamT)
    mass = float(PT.sum())
    return {
        "mass": mass,
        "primal": float((cost * F).sum()),
        "dual": dual_objective(st, mass),
        "src_mismatch": float(np.abs(P0 - p.mu0).sum()),
        "sink_mismatch": float(np.abs(PT - p.muT).sum()),
        "cap_violation": float(np.maximum(F - cap, 0.0)[np.isfinite(cap)].max(initial=0.0)),
        "cap_excess": float(np.maximum(F - cap, 0.0)[np.isfinite(cap)].sum()),
        "sweeps": st.sweeps,
    }


def solve_error(st: OracleState) -> float:
    """Convergence error of the end-of-sweep state (SPEC solve, as defined in
    include/mmf.h mmf_solve): (source + sink marginal L1 mismatch + total capacity excess) / tensor mass."""
    s = stats(st)
    return (s["src_mismatch"] + s["sink_mismatch"] + s["cap_excess"]) / s["mass"]


def oracle_solve(problem, tol: float, max_sweeps: int, check_every: int = 1, schedule: str = "gs",
                 theta: float = 1.0) -> tuple:
    """Sweeps until solve_error < tol, checked every check_every sweeps (at most max_sweeps).
    Returns (state, converged, sweeps, err, history)."""
    st = oracle_init(problem)
    done, err, hist = 0, float("inf"), []
    while True:
        if done > 0:
            err = solve_error(st)
            hist.append(err)
            if err < tol:
                break
        if done >= max_sweeps:
            break
        for _ in range(min(check_every, max_sweeps - done)):
            if schedule == "gs":
                oracle_sweep(st)
            elif schedule == "sym":
                oracle_sweep_symmetric(st)
            else:
                oracle_sweep_jacobi(st, theta)
        done = st.sweeps
    return st, err < tol, done, err, hist
