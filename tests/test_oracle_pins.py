"""Pins of the float64 log-domain oracle against things other than itself.

Every test here is CPU-only (-m "not gpu").  A plausible mistake anywhere in oracle/sweep.py (a
dropped K, a transposed message, a wrong sign in the capacity update, a wrong GS order, a wrong
zero convention) fails at least one of: brute-force tensor projections (P1), the closed-form
Schroedinger bridge (P2), textbook bimarginal Sinkhorn (P3), exact identities (P4), dual-ascent
monotonicity (P5), the LP bracket (P6) and the extended-precision twins (P9).
"""
import numpy as np
import pytest

from oracle import (oracle_init, oracle_sweep, oracle_run, readout_flows, readout_commodity_flows,
                    dual_objective, stats, OracleInfeasible)
from oracle.brute import BruteState, brute_sweep, full_tensor, arc_flows, commodity_marginal, BruteTimes
from oracle.lp import solve_lp, count_walks, time_expanded_counts
from oracle.twins import LinearTwin, MpTwin
from workloads import gen, grid_problem, fig1_problem
from tests._metrics import max_rel_err

MICROS = [
    dict(rows=2, cols=2, T=3, L=2, eps=0.5, seed=1),
    dict(rows=2, cols=3, T=4, L=3, eps=0.7, seed=2),
    dict(rows=2, cols=2, T=1, L=2, eps=0.4, seed=3),                                  # T = 1 (P7)
    dict(rows=2, cols=3, T=3, L=1, eps=0.5, seed=4),                                  # L = 1 (P7)
    dict(rows=2, cols=2, T=4, L=3, eps=0.6, seed=5, marginals="dense"),
    dict(rows=2, cols=3, T=3, L=2, eps=0.5, seed=6, time_varying=True),
    dict(rows=2, cols=3, T=4, L=2, eps=0.5, seed=8, closed_arcs=3, marginals="dense"),  # d = 0 arcs
]


def _micro(kw):
    kw = dict(kw)
    return grid_problem(kw.pop("rows"), kw.pop("cols"), kw.pop("T"), kw.pop("L"), kw.pop("eps"), **kw)


# ---------------------------------------------------------------------------------------------
# P1 brute force

@pytest.mark.parametrize("kw", MICROS)
def test_p1_structured_projections_equal_full_tensor(kw):
    """cor:proj / thm:biproj in node form == literal sums of M = K ⊙ U (eq:proj_discrete)."""
    p = _micro(kw)
    st = oracle_run(p, 3)
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    F_brute = arc_flows(p, M)
    F, W = readout_flows(st)
    assert max_rel_err(F, F_brute, 1e-300) < 1e-12
    for t in range(p.T):
        from oracle.brute import commodity_arc_flows
        assert max_rel_err(readout_commodity_flows(st, t), commodity_arc_flows(p, M, t), 1e-300) < 1e-12
    # end-of-sweep marginals: P_{c,T} = muT exactly after a4, P_{c,0} from the new backward pass
    assert max_rel_err(commodity_marginal(M, p.T), p.muT, 1e-300) < 1e-12
    P0 = np.exp(st.lam0 + st.b[0])
    assert max_rel_err(commodity_marginal(M, 0), P0, 1e-300) < 1e-12


@pytest.mark.parametrize("kw", MICROS)
def test_p1_iterates_identical_to_full_tensor_sinkhorn(kw):
    """10 GS sweeps of prp:sinkhorn with projections of the full tensor (W*d/F form)
    == the oracle's message-passing sweeps (P:1093 form): U0, W, UT after every sweep."""
    p = _micro(kw)
    st = oracle_init(p)
    bs = BruteState(p)
    for k in range(10):
        oracle_sweep(st)
        brute_sweep(bs)
        assert max_rel_err(np.exp(st.lam0), bs.U0, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.omega), bs.W, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.lamT), bs.UT, 1e-300) < 1e-12, k


# ---------------------------------------------------------------------------------------------
# P2 closed-form bridge

def _dense_K(p, t):
    K = np.zeros((p.N, p.N))
    for a in range(p.A):
        K[p.tail[a], p.head[a]] = np.exp(-p.cost_t(t)[a] / p.eps)
    return K


@pytest.mark.parametrize("tv", [False, True])
def test_p2_schroedinger_bridge_closed_form(tv):
    """d = inf, point masses: after one sweep F^l_t[a] = m_l (PK)_{0:t}[s,i] K_t[a] (PK)_{t+1:T}[j,g]
    / (PK)_{0:T}[s,g] (remark P:922-928: a discrete Schroedinger bridge) and it is a fixed point."""
    p = grid_problem(3, 3, 6, 3, 0.3, seed=11, cap=None, time_varying=tv, mass=[1.0, 2.0, 0.5])
    Ks = [_dense_K(p, t) for t in range(p.T)]

    def prod(r, q):
        P = np.eye(p.N)
        for t in range(r, q):
            P = P @ Ks[t]
        return P

    st = oracle_init(p)
    for sweep in range(3):
        oracle_sweep(st)
        for t in range(p.T):
            Fl = readout_commodity_flows(st, t)
            pre, post, tot = prod(0, t), prod(t + 1, p.T), prod(0, p.T)
            for l in range(p.L):
                s, g = p.src[l], p.dst[l]
                ref = p.mass[l] * pre[s, p.tail] * Ks[t][p.tail, p.head] * post[p.head, g] / tot[s, g]
                assert max_rel_err(Fl[:, l], ref, 1e-300) < 1e-12


# ---------------------------------------------------------------------------------------------
# P3 textbook Sinkhorn

def test_p3_textbook_bimarginal_sinkhorn():
    """d = inf, dense mu: the GS sweep's (U0, UT) equal classical Sinkhorn scalings (u, v) for
    the kernel Kbar = prod_t K_t (eq:omt P:305-311 regularised), iterate by iterate."""
    p = grid_problem(3, 3, 5, 2, 0.5, seed=12, cap=None, marginals="dense")
    Kbar = np.eye(p.N)
    for t in range(p.T):
        Kbar = Kbar @ _dense_K(p, t)
    v = (p.muT > 0).astype(float)
    st = oracle_init(p)
    for k in range(8):
        with np.errstate(divide="ignore", invalid="ignore"):
            u = np.where(p.mu0 > 0, p.mu0 / (v @ Kbar.T), 0.0)
            v = np.where(p.muT > 0, p.muT / (u @ Kbar), 0.0)
        oracle_sweep(st)
        assert max_rel_err(np.exp(st.lam0), u, 1e-300) < 1e-12
        assert max_rel_err(np.exp(st.lamT), v, 1e-300) < 1e-12


# ---------------------------------------------------------------------------------------------
# P4 exact identities

@pytest.mark.parametrize("which", ["tiny", "dense-micro", "closed-micro"])
def test_p4_conservation_marginals_capacity(which):
    if which == "tiny":
        p = gen(1)
    elif which == "dense-micro":
        p = grid_problem(3, 4, 6, 3, 0.3, seed=13, marginals="dense")
    else:
        p = grid_problem(3, 3, 5, 2, 0.3, seed=15, closed_arcs=4)
    st = oracle_init(p)
    in_step = []

    def hook(kind, t, mass):
        if kind == "W":
            # F_t <= d_t right after W_t's own update (prp:sinkhorn, the min(.,1) block)
            Fl = readout_commodity_flows(st, t)  # uses a_t and W_t new, b_{t+1} old: the current tensor
            in_step.append((t, Fl.sum(axis=1)))

    for k in range(5):
        in_step.clear()
        oracle_sweep(st, on_block=hook)
        for t, F in in_step:
            cap = p.cap_t(t)
            fin = np.isfinite(cap)
            assert np.all(F[fin] <= cap[fin] * (1 + 1e-12) + 1e-300)
        m = stats(st)["mass"]
        Fagg, W = readout_flows(st)
        assert np.all(W >= 0) and np.all(W <= 1)
        assert np.all(Fagg >= 0)
        # (ii) every time slice carries the whole mass
        assert np.allclose(Fagg.sum(axis=1), m, rtol=1e-12, atol=0)
        for t in range(1, p.T):
            fin_prev = readout_commodity_flows(st, t - 1)
            fout = readout_commodity_flows(st, t)
            inflow = np.zeros((p.N, p.L))
            outflow = np.zeros((p.N, p.L))
            np.add.at(inflow, p.head, fin_prev)
            np.add.at(outflow, p.tail, fout)
            # (i) per-commodity conservation at every node and step
            assert max_rel_err(inflow, outflow, 1e-14 * m) < 1e-11
        # (iii) sink marginal exact after a4
        lastin = np.zeros((p.N, p.L))
        np.add.at(lastin, p.head, readout_commodity_flows(st, p.T - 1))
        assert max_rel_err(lastin.T, p.muT, 1e-14) < 1e-11
        # (iv) point masses: source marginal exact too
        if p.is_point:
            firstout = np.zeros((p.N, p.L))
            np.add.at(firstout, p.tail, readout_commodity_flows(st, 0))
            assert max_rel_err(firstout.T, p.mu0, 1e-14) < 1e-11
        closed = np.isfinite(p.cap) & (p.cap == 0) if p.cap.ndim == 1 else None
        if closed is not None and closed.any():
            assert np.all(W[:, closed] == 0) and np.all(Fagg[:, closed] == 0)


# ---------------------------------------------------------------------------------------------
# P5 block-coordinate ascent

@pytest.mark.parametrize("which", ["tiny", "micro-dense", "grid-tight"])
def test_p5_dual_nondecreasing_after_every_block(which):
    """prp:sinkhorn: each update is an exact block maximisation of the dual, so
    the dual objective never decreases -- after U0, after every W_t and after UT."""
    if which == "tiny":
        p = gen(1)
    elif which == "micro-dense":
        p = grid_problem(3, 3, 5, 3, 0.3, seed=15, marginals="dense")
    else:
        p = grid_problem(4, 4, 8, 4, 0.2, seed=16, cap=(0.05, 0.4))
    st = oracle_init(p)
    vals = []
    st_ref = st

    def hook(kind, t, mass):
        vals.append(dual_objective(st_ref, mass))

    for k in range(15):
        oracle_sweep(st, on_block=hook)
    v = np.array(vals)
    scale = np.abs(v).max()
    assert np.all(np.diff(v) >= -1e-12 * scale), np.diff(v).min()
    if which != "tiny":            # Tiny's capacities do not bind (W stays 1): dual constant
        assert v[-1] > v[0]


# ---------------------------------------------------------------------------------------------
# P6 LP bracket

def _converge(p, max_sweeps=20000, tol=1e-10):
    st = oracle_init(p)
    prev = None
    for k in range(max_sweeps):
        oracle_sweep(st)
        w = st.omega.copy()
        if prev is not None and np.nanmax(np.abs(np.exp(w) - np.exp(prev))) < tol:
            break
        prev = w
    return st


@pytest.mark.parametrize("which", ["tiny", "tight-micro"])
def test_p6_lp_bracket_and_eps_monotone(which):
    """thm:equiv_mc + entropic bound: 0 <= <C,F_eps> - OPT_LP <= eps m_tot log(P m_max / m_tot),
    and <C,F_eps> is non-increasing as eps decreases.  "tight-micro" has binding caps
    (its LP optimum exceeds the uncapacitated one)."""
    import dataclasses
    if which == "tiny":
        base = gen(1)
    else:
        base = grid_problem(3, 3, 6, 3, 1.0, seed=35, cap=(0.3, 0.6))
    lp = solve_lp(base)
    assert lp["status"] == 0, "instance must be LP-feasible"
    if which == "tiny":
        # Tiny LP size: 3150 variables, 825 equalities, 800 capacity rows
        assert (lp["n_var"], lp["n_eq"], lp["n_ub"]) == (3150, 825, 800)
    else:
        free = solve_lp(dataclasses.replace(base, cap=np.full_like(base.cap, np.inf)))
        assert lp["opt"] > free["opt"] + 0.05
    P = count_walks(base)
    mtot = float(base.mass.sum())
    mmax = float(base.mass.max())
    prims = []
    for eps in [1.0, 0.3, 0.1, 0.03]:
        p = dataclasses.replace(base, eps=eps)
        st = _converge(p)
        s = stats(st)
        assert s["cap_violation"] < 1e-7
        gap = s["primal"] - lp["opt"]
        assert -1e-7 <= gap <= eps * mtot * np.log(P * mmax / mtot) + 1e-7, (eps, gap)
        prims.append(s["primal"])
    assert all(prims[i + 1] <= prims[i] + 1e-9 for i in range(len(prims) - 1)), prims


def test_p8_conditioning_probe():
    """P8: the oracle disagrees with itself, on inputs perturbed at 1e-15 relative, by far less than
    the fp64 parity tolerance 1e-10 after the parity sweep count -- so 1e-10 is attainable."""
    import dataclasses
    from tests._metrics import flow_floor
    for base, sweeps in [(grid_problem(3, 3, 6, 3, 0.1, seed=35, cap=(0.3, 0.6)), 200), (gen(2, L=4, T=12), 30)]:
        rng = np.random.default_rng(0)
        pert = dataclasses.replace(base, cost=base.cost * (1 + 1e-15 * rng.uniform(-1, 1, base.cost.shape)))
        F1, W1 = readout_flows(oracle_run(base, sweeps))
        F2, W2 = readout_flows(oracle_run(pert, sweeps))
        assert max_rel_err(F2, F1, flow_floor(base)) < 1e-11
        assert max_rel_err(W2, W1, 1e-30) < 1e-11


def test_lp_builder_on_fig1_counts():
    """Golden: Fig. time_exp: 3 nodes, 4 edges, T=3 -> 12 vertices, 12 edges."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "fig1_time_expansion.txt")
    gold = dict(line.split() for line in open(path) if line.strip() and not line.startswith("#"))
    p = fig1_problem(int(gold["T"]))
    assert p.N == int(gold["nodes"]) and p.A == int(gold["edges"])
    assert time_expanded_counts(p) == (int(gold["expanded_vertices"]), int(gold["expanded_edges"]))
    lp = solve_lp(p)
    assert lp["n_var"] == int(gold["expanded_edges"]) * p.L


def test_lp_tiny_optimum_matches_walk_enumeration():
    """The LP itself pinned on an uncapacitated micro instance: OPT = sum_l m_l * (min-cost T-step
    walk s_l -> g_l), by brute-force dynamic programming over walks."""
    p = grid_problem(3, 3, 4, 3, 1.0, seed=17, cap=None)
    lp = solve_lp(p)
    best = 0.0
    for l in range(p.L):
        d = np.full(p.N, np.inf)
        d[p.src[l]] = 0.0
        for t in range(p.T):
            nd = np.full(p.N, np.inf)
            for a in range(p.A):
                nd[p.head[a]] = min(nd[p.head[a]], d[p.tail[a]] + p.cost_t(t)[a])
            d = nd
        best += p.mass[l] * d[p.dst[l]]
    assert abs(lp["opt"] - best) < 1e-9


# ---------------------------------------------------------------------------------------------
# P9 representation twins

@pytest.mark.parametrize("which,sweeps", [("tiny", 200), ("micro-dense", 30), ("grid2-lite", 5)])
def test_p9_longdouble_linear_twin(which, sweeps):
    if which == "tiny":
        p = gen(1)
    elif which == "micro-dense":
        p = grid_problem(3, 4, 6, 3, 0.3, seed=18, marginals="dense", closed_arcs=2)
    else:
        p = gen(2, L=4, T=12)
    st = oracle_init(p)
    tw = LinearTwin(p, np.longdouble)
    for k in range(sweeps):
        oracle_sweep(st)
        tw.sweep()
    F, W = readout_flows(st)
    from tests._metrics import flow_floor
    assert max_rel_err(F, tw.flows().astype(np.float64), flow_floor(p)) < 1e-12
    assert max_rel_err(W, tw.W.astype(np.float64), 1e-30) < 1e-12


def test_p9_mpmath_twin_micro():
    p = grid_problem(2, 2, 3, 2, 0.5, seed=19)
    st = oracle_init(p)
    tw = MpTwin(p, dps=40)
    for k in range(4):
        oracle_sweep(st)
        tw.sweep()
    F, W = readout_flows(st)
    assert max_rel_err(F, tw.flows(), 1e-300) < 1e-13
    assert max_rel_err(W, np.array([[float(x) for x in row] for row in tw.W]), 1e-300) < 1e-13


# ---------------------------------------------------------------------------------------------
# conventions

def test_infeasible_source_raises():
    """x/0 with x > 0 at the boundary scaling: a sink unreachable within T steps."""
    p = grid_problem(3, 3, 2, 1, 0.5, seed=20)
    p.src = np.array([0], np.int32)
    p.dst = np.array([8], np.int32)   # Manhattan distance 4 > T = 2
    st = oracle_init(p)
    with pytest.raises(OracleInfeasible):
        oracle_sweep(st)


def test_tiny_runs_200_sweeps_and_satisfies_capacities_approximately():
    p = gen(1)
    st = oracle_run(p, p.sweeps)
    s = stats(st)
    assert abs(s["mass"] - 3.0) < 1e-9
    assert s["src_mismatch"] < 1e-6
    assert s["cap_violation"] < 1e-3


# ---------------------------------------------------------------------------------------------
# NEXT-1: the damped Jacobi schedule, W <- W^(1-theta) min(W d / F, 1)^theta from one
# alpha/beta pair

from oracle import oracle_sweep_jacobi  # noqa: E402


@pytest.mark.parametrize("kw", [MICROS[0], MICROS[1], MICROS[6]])
@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_jacobi_update_equals_full_tensor_projection(kw, theta):
    """Every W_t of a Jacobi sweep is the damped update evaluated on the SAME tensor: the flows are the
    bimarginals of M(U0 new, W old, UT old) summed literally over the full tensor (brute force), and the
    sink scaling then matches P_T = muT of M(U0 new, W new, UT new)."""
    from oracle.brute import bimarginal
    p = _micro(kw)
    st = oracle_init(p)
    for _ in range(2):
        oracle_sweep(st)
    for _ in range(3):
        W_old, lamT_old = np.exp(st.omega), st.lamT.copy()
        oracle_sweep_jacobi(st, theta)
        M = full_tensor(p, np.exp(st.lam0), W_old, np.exp(lamT_old))
        F = arc_flows(p, M)
        cap = np.broadcast_to(p.cap, F.shape)
        with np.errstate(divide="ignore", invalid="ignore"):
            full = np.where(np.isinf(cap), 1.0, np.where(cap == 0, 0.0,
                            np.where(F > 0, np.minimum(W_old * cap / np.where(F > 0, F, 1.0), 1.0), 1.0)))
        W_ref = W_old ** (1.0 - theta) * full ** theta
        assert max_rel_err(np.exp(st.omega), W_ref, 1e-300) < 1e-12
        M_new = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
        # the end-of-sweep sink marginal is exact only for the alpha that a4 used: alpha_T of the pass with
        # W old, i.e. the tensor M(U0 new, W old, UT new)
        M_a4 = full_tensor(p, np.exp(st.lam0), W_old, np.exp(st.lamT))
        assert max_rel_err(commodity_marginal(M_a4, p.T), p.muT, 1e-300) < 1e-12
        # readout = projections of the end-of-sweep tensor
        F_end, _ = readout_flows(st)
        assert max_rel_err(F_end, arc_flows(p, M_new), 1e-300) < 1e-12


@pytest.mark.parametrize("theta", [0.3, 1.0])
def test_jacobi_equals_gs_without_capacities(theta):
    """d = inf: W stays 1, so the Jacobi schedule reduces to the plain Sinkhorn of Algorithm 2 iterate by
    iterate (the schedules differ only in when W is updated)."""
    p = grid_problem(3, 3, 5, 3, 0.3, seed=12, cap=None)
    a = oracle_init(p)
    b = oracle_init(p)
    for _ in range(4):
        oracle_sweep(a)
        oracle_sweep_jacobi(b, theta)
        assert max_rel_err(np.exp(b.lam0), np.exp(a.lam0), 1e-300) < 1e-13
        assert max_rel_err(np.exp(b.lamT), np.exp(a.lamT), 1e-300) < 1e-13


def test_jacobi_fixed_point_is_the_gs_optimum():
    """Damped Jacobi converges to the same optimum as Gauss-Seidel (the unique minimiser of the strictly convex
    problem, pinned independently by the LP bracket P6): capacity duals and flows agree after convergence."""
    p = grid_problem(3, 3, 4, 2, 0.5, seed=13, cap=(0.15, 0.4))
    gs = oracle_run(p, 400)
    jb = oracle_run(p, 400, schedule="jacobi", theta=0.5)
    Fg, Wg = readout_flows(gs)
    Fj, Wj = readout_flows(jb)
    assert max_rel_err(Wj, Wg, 1e-12) < 1e-7
    assert max_rel_err(Fj, Fg, 1e-12) < 1e-7
    assert np.any(Wg < 0.99)  # (capacities bind: the schedules differ along the way)


def test_jacobi_theta_zero_keeps_w():
    """theta = 0 never moves W: after any number of sweeps the state is Algorithm 2's on the uncapacitated
    copy of the instance."""
    import dataclasses
    p = grid_problem(3, 3, 4, 2, 0.5, seed=14, cap=(0.15, 0.4))
    q = dataclasses.replace(p, cap=np.full_like(p.cap, np.inf))
    a = oracle_run(q, 3)
    b = oracle_run(p, 3, schedule="jacobi", theta=0.0)
    assert np.all(b.omega == 0.0)
    assert max_rel_err(np.exp(b.lam0), np.exp(a.lam0), 1e-300) < 1e-13


# ---------------------------------------------------------------------------------------------
# NEXT-4: solve to tolerance

from oracle import oracle_solve, solve_error  # noqa: E402


def test_solve_error_equals_full_tensor_marginals_and_excess():
    """The solve error is the literal marginal L1 mismatch + capacity excess of the full tensor."""
    p = _micro(MICROS[4])  # (dense marginals, capacities bind)
    st = oracle_run(p, 3)
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    F = arc_flows(p, M)
    cap = np.broadcast_to(p.cap, F.shape)
    ex = np.maximum(F - cap, 0.0)[np.isfinite(cap)].sum()
    ref = (np.abs(commodity_marginal(M, 0) - p.mu0).sum() + np.abs(commodity_marginal(M, p.T) - p.muT).sum()
           + ex) / M.sum()
    assert abs(solve_error(st) - ref) <= 1e-12 * max(ref, 1e-300) + 1e-15


def test_solve_converges_and_satisfies_constraints():
    """tol = 1e-8 on a tiny capacitated instance: converged, and the brute-force tensor of the returned state
    meets the marginals and capacities to the tolerance; max_sweeps = 0 returns the initial state, not
    converged (SPEC solve examples)."""
    p = grid_problem(3, 3, 4, 2, 0.5, seed=13, cap=(0.15, 0.4))
    st, conv, k, err, hist = oracle_solve(p, 1e-8, 2000)
    assert conv and err < 1e-8 and len(hist) == k
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    mass = M.sum()
    assert np.abs(commodity_marginal(M, 0) - p.mu0).sum() / mass < 1e-8
    F = arc_flows(p, M)
    cap = np.broadcast_to(p.cap, F.shape)
    assert np.maximum(F - cap, 0.0)[np.isfinite(cap)].sum() / mass < 1e-8
    st0, conv0, k0, err0, hist0 = oracle_solve(p, 1e-8, 0)
    assert not conv0 and k0 == 0 and hist0 == [] and st0.sweeps == 0


# ---------------------------------------------------------------------------------------------
# round 2: the dual objective pinned completely (thm:solution P:777-788), storage options, sharding combine,
# fp32-level conditioning probe, a negative control of the parity metric

def _cost_tensor(p):
    """C[l, v_0, ..., v_T] = sum_t C_t[v_t, v_{t+1}] (+inf off the graph), the cost tensor of eq:omt_multi_graph_reg
    in node form, built literally by broadcasting."""
    Ct = []
    for t in range(p.T):
        D = np.full((p.N, p.N), np.inf)
        D[p.tail, p.head] = p.cost_t(t)
        Ct.append(D)
    C = np.zeros((1,) * 1 + (p.N,))
    for t in range(p.T):
        C = C[..., :, None] + Ct[t].reshape((1,) * (C.ndim - 1) + Ct[t].shape)
    return np.broadcast_to(C, (p.L,) + C.shape[1:])


@pytest.mark.parametrize("kw", [MICROS[0], MICROS[4], MICROS[6]])
def test_dual_objective_equals_brute_force_dual(kw):
    """eq:omt_multi_graph_dual: Phi = -eps <K, U> - sum <lambda_t, mu_t> - sum <lambda_t, d_t> with
    u = exp(-lambda/eps), evaluated on the brute-force Sinkhorn's OWN scalings (oracle/brute.py, full-tensor
    projections) and the full tensor's mass, equals the oracle's dual_objective after every sweep."""
    p = _micro(kw)
    st = oracle_init(p)
    bs = BruteState(p)
    cap = np.broadcast_to(p.cap, (p.T, p.A))
    for k in range(6):
        oracle_sweep(st)
        brute_sweep(bs)
        M = bs.tensor()
        with np.errstate(divide="ignore"):
            lam0, lamT, lamW = -p.eps * np.log(bs.U0), -p.eps * np.log(bs.UT), -p.eps * np.log(bs.W)
        # <lambda, mu> with 0 * inf = 0; lambda_t on capacitated arcs only (V_<=)
        t0 = np.where(p.mu0 > 0, p.mu0 * lam0, 0.0).sum()
        tT = np.where(p.muT > 0, p.muT * lamT, 0.0).sum()
        fin = np.isfinite(cap) & (cap > 0)
        tW = np.where(fin, cap * np.where(fin, lamW, 0.0), 0.0).sum()
        phi = -p.eps * M.sum() - t0 - tT - tW
        got = dual_objective(st, float(np.exp(st.a[p.T] + st.lamT).sum()))
        assert abs(got - phi) <= 1e-11 * max(1.0, abs(phi)), (k, got, phi)


@pytest.mark.parametrize("which", ["tight-micro", "tight-grid", "dense-slack"])
def test_strong_duality_at_convergence(which):
    """thm:solution (strong duality, the proof's Lagrangian): at the optimum the regularised primal
    <C, M> + eps sum (M log M - M) of the brute-force tensor equals the dual objective.  With binding capacities
    the capacity term sum d * log W carries a sizeable share of Phi (dropping it fails this pin)."""
    if which == "tight-micro":
        p = grid_problem(2, 3, 4, 2, 0.5, seed=2, cap=(0.3, 0.6))
    elif which == "tight-grid":
        p = grid_problem(3, 3, 4, 2, 0.5, seed=13, cap=(0.15, 0.4))
    else:
        p = grid_problem(2, 3, 4, 2, 0.6, seed=5, cap=(0.3, 0.7), marginals="dense")
    st = oracle_init(p)
    for _ in range(3000):
        oracle_sweep(st)
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    C = _cost_tensor(p)
    pos = M > 0
    primal = (C[pos] * M[pos]).sum() + p.eps * (M[pos] * np.log(M[pos]) - M[pos]).sum()
    mass = float(np.exp(st.a[p.T] + st.lamT).sum())
    phi = dual_objective(st, mass)
    from oracle.sweep import dual_terms
    sd = dual_terms(st)[2]
    assert stats(st)["cap_violation"] < 1e-12          # (a feasible instance, converged)
    assert abs(primal - phi) <= 1e-9 * abs(phi), (primal, phi)
    # complementary slackness behind it: F_t[a] = d_t[a] wherever W_t[a] < 1
    F, W = readout_flows(st)
    cap = np.broadcast_to(p.cap, F.shape)
    bind = W < 1 - 1e-9
    if which != "dense-slack":
        assert abs(p.eps * sd) > 0.1 * abs(phi)        # (capacities bind: the term matters)
        assert bind.any() and np.max(np.abs(F[bind] - cap[bind]) / cap[bind]) < 1e-8
    else:
        assert not bind.any() and sd == 0.0


@pytest.mark.parametrize("schedule", ["gs", "jacobi"])
def test_storage_options_bitwise_equal(schedule):
    """oracle_init's storage options (an np.memmap backward store, two forward layers recomputed for readouts —
    used for the full-size [4]/[5] fixtures) change no value: F, W and every statistic are bitwise equal to the
    in-memory oracle's, for both schedules and at 0 sweeps."""
    import os
    import tempfile
    from oracle import oracle_sweep_jacobi
    for kw in [dict(), dict(marginals="dense", closed_arcs=2, time_varying=True)]:
        p = grid_problem(4, 5, 6, 5, 0.3, seed=3, cap=(0.2, 0.6), **kw)
        ref = oracle_init(p)
        with tempfile.TemporaryDirectory() as d:
            mm = np.lib.format.open_memmap(os.path.join(d, "b.npy"), mode="w+", dtype=np.float64,
                                           shape=(p.T + 1, p.L, p.N))
            st = oracle_init(p, b_store=mm, keep_forward=False)
            for k in range(4):
                F1, W1 = readout_flows(ref)
                F2, W2 = readout_flows(st)
                assert np.array_equal(F1, F2) and np.array_equal(W1, W2)
                assert stats(ref) == stats(st)
                for t in (0, p.T - 1):
                    assert np.array_equal(readout_commodity_flows(ref, t), readout_commodity_flows(st, t))
                if schedule == "gs":
                    oracle_sweep(ref)
                    oracle_sweep(st)
                else:
                    oracle_sweep_jacobi(ref, 0.5)
                    oracle_sweep_jacobi(st, 0.5)
            del st, mm


def test_sharded_oracle_combine_equals_unsharded():
    """oracle.shard (the commodity sharding the full-size fixtures use): G = 3 shards run in lock step in one
    process, their per-arc log flow sums combined by combine_lse before every W_t update, and their statistics by
    combine_stats, reproduce the unsharded oracle (rem:multi_tensor_scheme P:1139-1147) to rounding."""
    import threading
    from oracle.shard import combine_lse, shard_pieces, combine_stats
    p = grid_problem(4, 5, 6, 7, 0.2, seed=41, cap=(0.2, 0.6))
    G = 3
    bounds = [(0, 3), (3, 5), (5, 7)]
    shards = [oracle_init(p.commodity_slice(a, b)) for a, b in bounds]
    bar = threading.Barrier(G)
    box = [None] * G
    out = {}

    def worker(g):
        def reduce_lse(v):
            box[g] = np.array(v)
            bar.wait()
            r = combine_lse(np.stack(box))
            bar.wait()
            return r
        for _ in range(5):
            oracle_sweep(shards[g], reduce_lse=reduce_lse)
        out[g] = shard_pieces(shards[g])

    th = [threading.Thread(target=worker, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    s = combine_stats(p, [out[g] for g in range(G)], shards[0].omega, 5)
    ref = oracle_run(p, 5)
    F, W = readout_flows(ref)
    so = stats(ref)
    assert max_rel_err(s["F"], F, 1e-300) < 1e-12 and max_rel_err(s["W"], W, 1e-300) < 1e-12
    for k in ("mass", "primal", "dual", "src_mismatch", "sink_mismatch", "cap_violation", "cap_excess"):
        assert abs(s[k] - so[k]) <= 1e-11 * max(abs(so[k]), 1e-3), (k, s[k], so[k])
    assert np.min(W) < 0.999


def test_p8_conditioning_probe_fp32_inputs():
    """P8 at the fp32 parity bar: the oracle on inputs perturbed as the fp32 path rounds them (K = exp(-C/eps) by
    a relative 2^-24, capacities to float32) disagrees with itself by far less than 1e-4 after the Q21 sweep count,
    on the BASELINE graphs and horizons at small L — so 1e-4 is attainable (an ill-conditioned config would show
    here)."""
    import dataclasses
    from tests._metrics import flow_floor
    cases = [(gen(1), 200), (gen(2, L=4, T=60), 100), (gen(4, L=2, T=40), 3), (gen(5, L=8, T=40), 3),
             (gen(3, L=2, T=40), 10)]
    for base, sweeps in cases:
        rng = np.random.default_rng(0)
        dK = rng.uniform(-2.0 ** -24, 2.0 ** -24, base.cost.shape)
        pert = dataclasses.replace(base, cost=base.cost - base.eps * np.log1p(dK),
                                   cap=base.cap.astype(np.float32).astype(np.float64))
        F1, W1 = readout_flows(oracle_run(base, sweeps))
        F2, W2 = readout_flows(oracle_run(pert, sweeps))
        ef, ew = max_rel_err(F2, F1, flow_floor(base)), max_rel_err(W2, W1, 1e-30)
        assert ef < 1e-5 and ew < 1e-5, (base.name, ef, ew)


def test_parity_metric_negative_control():
    """SURVEY §4 negative control of the parity metric itself (Q11): an oracle result with ONE capacity dual moved
    by k ulp fails the fp64 bar once k ulp exceed 1e-10 relative, and one flow moved by 2e-4 relative fails fp32."""
    p = grid_problem(3, 3, 5, 3, 0.3, seed=15, cap=(0.1, 0.4))
    F, W = readout_flows(oracle_run(p, 5))
    from tests._metrics import flow_floor
    i = np.unravel_index(np.argmin(W), W.shape)
    assert W[i] < 1
    W2 = W.copy()
    W2[i] = W[i] + 2 ** 20 * np.spacing(W[i])           # 2^20 ulp = 2.3e-10 relative
    assert max_rel_err(W2, W, 1e-30) > 1e-10
    W2[i] = W[i] + 2 ** 10 * np.spacing(W[i])           # 2^10 ulp = 2.3e-13: passes
    assert max_rel_err(W2, W, 1e-30) < 1e-10
    F2 = F.copy()
    j = np.unravel_index(np.argmax(F), F.shape)
    F2[j] *= 1 + 2e-4
    assert max_rel_err(F2, F, flow_floor(p)) > 1e-4


# ---------------------------------------------------------------------------------------------
# NEXT-2: commodity-dependent node costs c[l, j] at the intermediate layers (reading R-N)

def _with_node_cost(p, seed, scale=1.0, kind="random"):
    import dataclasses
    rng = np.random.default_rng(seed)
    if kind == "random":
        c = rng.uniform(0.0, scale, size=(p.L, p.N))
    elif kind == "const":
        c = np.full((p.L, p.N), scale)
    elif kind == "per-commodity":
        c = np.repeat(rng.uniform(0.0, scale, size=(p.L, 1)), p.N, axis=1)
    else:  # "per-node": the same for every commodity
        c = np.repeat(rng.uniform(0.0, scale, size=(1, p.N)), p.L, axis=0)
    return dataclasses.replace(p, node_cost=c)


@pytest.mark.parametrize("kw", [MICROS[0], MICROS[1], MICROS[4], MICROS[5], MICROS[6]])
def test_node_costs_iterates_identical_to_full_tensor_sinkhorn(kw):
    """P1 with commodity node costs: 10 GS sweeps of prp:sinkhorn whose projections are literal sums of the full
    tensor M[l, v] = U0 prod_t K_t W_t prod_{t=1}^{T-1} exp(-c[l, v_t]/eps) UT (oracle/brute.py) equal the oracle's
    message-passing sweeps iterate by iterate, and the readout equals the tensor's projections."""
    p = _with_node_cost(_micro(kw), seed=7, scale=0.8)
    st = oracle_init(p)
    bs = BruteState(p)
    for k in range(10):
        oracle_sweep(st)
        brute_sweep(bs)
        assert max_rel_err(np.exp(st.lam0), bs.U0, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.omega), bs.W, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.lamT), bs.UT, 1e-300) < 1e-12, k
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    F, _ = readout_flows(st)
    assert max_rel_err(F, arc_flows(p, M), 1e-300) < 1e-12
    for t in (0, p.T - 1):
        from oracle.brute import commodity_arc_flows
        assert max_rel_err(readout_commodity_flows(st, t), commodity_arc_flows(p, M, t), 1e-300) < 1e-12
    assert abs(stats(st)["mass"] - M.sum()) <= 1e-12 * M.sum()


@pytest.mark.parametrize("kind", ["const", "per-commodity"])
def test_node_costs_gauge_invariance(kind):
    """A node cost that is the same at every node for a commodity (c[l, j] = g_l) charges every walk of commodity l the
    same (T-1) g_l: the optimal tensor of each commodity is unchanged up to its scalings, so the flows and capacity
    duals equal those without node costs after every sweep (to rounding)."""
    p = grid_problem(3, 4, 6, 3, 0.3, seed=16, cap=(0.1, 0.5))
    q = _with_node_cost(p, seed=3, scale=0.7, kind=kind)
    a, b = oracle_init(p), oracle_init(q)
    for _ in range(6):
        oracle_sweep(a)
        oracle_sweep(b)
        Fa, Wa = readout_flows(a)
        Fb, Wb = readout_flows(b)
        assert max_rel_err(Fb, Fa, 1e-300) < 1e-11 and max_rel_err(Wb, Wa, 1e-300) < 1e-11
    assert np.min(Wa) < 0.99


def test_node_costs_commodity_independent_reduce_to_arc_costs():
    """A node cost that does not depend on the commodity (c[l, j] = g_j) is an arc cost: it equals the problem with
    time-varying arc costs C_t[a] + g[head(a)] for t = 0..T-2 (and C_{T-1}[a] on the last step, reading R-N), which
    the oracle solves through the already pinned commodity-independent path: identical flows and duals."""
    import dataclasses
    p = grid_problem(3, 4, 6, 3, 0.3, seed=17, cap=(0.1, 0.5))
    q = _with_node_cost(p, seed=5, scale=0.9, kind="per-node")
    g = q.node_cost[0]
    cost = np.broadcast_to(p.cost, (p.T, p.A)).copy()
    cost[: p.T - 1] += g[p.head][None, :]
    r = dataclasses.replace(p, cost=cost)
    a, b = oracle_run(q, 6), oracle_run(r, 6)
    Fa, Wa = readout_flows(a)
    Fb, Wb = readout_flows(b)
    assert max_rel_err(Fa, Fb, 1e-300) < 1e-11 and max_rel_err(Wa, Wb, 1e-300) < 1e-11
    assert np.min(Wa) < 0.99


def test_node_costs_dual_monotone_and_strong_duality():
    """prp:sinkhorn with K_L: the dual objective (now with the commodity-dependent kernel in <K, U>) is non-decreasing
    after every block, and at convergence equals the regularised primal of the brute-force tensor whose cost includes
    the node costs (thm:solution P:777-788)."""
    p = _with_node_cost(grid_problem(3, 3, 4, 2, 0.5, seed=13, cap=(0.15, 0.4)), seed=9, scale=0.6)
    st = oracle_init(p)
    vals = []
    for _ in range(20):
        oracle_sweep(st, on_block=lambda kind, t, mass: vals.append(dual_objective(st, mass)))
    v = np.array(vals)
    assert np.all(np.diff(v) >= -1e-12 * np.abs(v).max())
    for _ in range(3000):
        oracle_sweep(st)
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT))
    C = np.array(_cost_tensor(p))
    for t in range(1, p.T):  # node cost of mode t
        C = C + p.node_cost.reshape((p.L,) + (1,) * t + (p.N,) + (1,) * (p.T - t))
    pos = M > 0
    primal = (C[pos] * M[pos]).sum() + p.eps * (M[pos] * np.log(M[pos]) - M[pos]).sum()
    phi = dual_objective(st, float(np.exp(st.a[p.T] + st.lamT).sum()))
    assert stats(st)["cap_violation"] < 1e-12
    assert abs(primal - phi) <= 1e-9 * abs(phi), (primal, phi)


# ---------------------------------------------------------------------------------------------
# NEXT-4: per-commodity entry / exit times (rem:multi_tensor_scheme P:1139-1149)

def _times_problem(seed=0, T=6, L=3, node_cost=False, marginals="point", cap=(0.15, 0.5), rows=2, cols=3):
    import dataclasses
    p = grid_problem(rows, cols, T, L, 0.5, seed=seed, cap=cap, marginals=marginals)
    rng = np.random.default_rng(seed)
    t_in = rng.integers(0, 2, size=L)
    t_out = np.maximum(t_in + 3, T - rng.integers(0, 2, size=L))
    t_out = np.minimum(t_out, T)
    q = dataclasses.replace(p, t_in=t_in, t_out=t_out)
    if node_cost:
        q = dataclasses.replace(q, node_cost=rng.uniform(0, 0.5, size=(L, p.N)))
    return q


@pytest.mark.parametrize("kw", [dict(seed=1), dict(seed=2, marginals="dense"), dict(seed=3, node_cost=True),
                                dict(seed=4, L=2, T=5)])
def test_commodity_times_iterates_identical_to_window_tensors(kw):
    """P1 with entry / exit times: 8 GS sweeps of the per-commodity window tensors (oracle/brute.py BruteTimes, every
    projection a literal sum) equal the oracle's sweeps iterate by iterate (U0, W, UT), and its flows vanish outside
    each commodity's window."""
    p = _times_problem(**kw)
    assert np.any(p.t_in > 0) and np.any(p.t_out < p.T)
    st = oracle_init(p)
    bt = BruteTimes(p)
    for k in range(8):
        oracle_sweep(st)
        bt.sweep()
        assert max_rel_err(np.exp(st.lam0), bt.U0, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.omega), bt.W, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.lamT), bt.UT, 1e-300) < 1e-12, k
    F, _ = readout_flows(st)
    assert max_rel_err(F, bt.flows(), 1e-300) < 1e-12
    for l in range(p.L):
        for t in list(range(0, p.t_in[l])) + list(range(p.t_out[l], p.T)):
            assert np.all(readout_commodity_flows(st, t)[:, l] == 0.0)
    s = stats(st)
    assert abs(s["mass"] - sum(M.sum() for M in bt.tensors())) <= 1e-12 * s["mass"]


def test_commodity_times_full_window_equals_plain():
    """t_in = 0 and t_out = T for every commodity is Algorithm 2 itself (to rounding)."""
    import dataclasses
    p = grid_problem(3, 3, 5, 3, 0.3, seed=12, cap=(0.1, 0.4))
    q = dataclasses.replace(p, t_in=np.zeros(3, int), t_out=np.full(3, 5))
    a, b = oracle_run(p, 5), oracle_run(q, 5)
    Fa, Wa = readout_flows(a)
    Fb, Wb = readout_flows(b)
    assert max_rel_err(Fb, Fa, 1e-300) < 1e-14 and max_rel_err(Wb, Wa, 1e-300) < 1e-14


def test_commodity_times_shifted_window_is_a_shorter_horizon():
    """Time shift: with time-invariant costs and no capacities, a commodity present on layers [t_in, t_out] moves
    exactly like the same commodity on a horizon of t_out - t_in steps (the Schroedinger bridge of remark P:922-928
    only sees the window): its flows are the shorter problem's, shifted by t_in."""
    import dataclasses
    p = grid_problem(3, 3, 7, 1, 0.4, seed=11, cap=None)
    q = dataclasses.replace(p, t_in=np.array([2]), t_out=np.array([6]))
    r = dataclasses.replace(p, T=4)
    Fq, _ = readout_flows(oracle_run(q, 3))
    Fr, _ = readout_flows(oracle_run(r, 3))
    assert max_rel_err(Fq[2:6], Fr, 1e-300) < 1e-12
    assert np.all(Fq[:2] == 0) and np.all(Fq[6:] == 0)


def test_commodity_times_dual_monotone():
    """prp:sinkhorn on the multi-tensor form (eq:Sinkhorn_multi_tensor P:1141-1145): the dual objective is
    non-decreasing after every block (U0, each W_t, UT) with the per-commodity windows."""
    p = _times_problem(seed=5, L=3, T=6, cap=(0.1, 0.3))
    st = oracle_init(p)
    vals = []
    for _ in range(15):
        oracle_sweep(st, on_block=lambda kind, t, mass: vals.append(dual_objective(st, mass)))
    v = np.array(vals)
    assert np.all(np.diff(v) >= -1e-12 * np.abs(v).max()), np.diff(v).min()
    assert v[-1] > v[0]


# ---------------------------------------------------------------------------------------------
# NEXT-1 remainder: symmetric Gauss-Seidel (W updated in the forward and the backward pass)

from oracle import oracle_sweep_symmetric  # noqa: E402
from oracle.brute import brute_sweep_symmetric  # noqa: E402


@pytest.mark.parametrize("kw", [MICROS[0], MICROS[1], MICROS[4], MICROS[6]])
def test_symmetric_gs_iterates_identical_to_full_tensor(kw):
    """Every block of the symmetric sweep (U0, W_0..W_{T-1}, UT, W_{T-1}..W_0) is prp:sinkhorn's update with the
    projections of the full tensor: 8 sweeps iterate-identical to the brute-force symmetric sweep, and the readout
    equals the end-of-sweep tensor's projections."""
    p = _micro(kw)
    st = oracle_init(p)
    bs = BruteState(p)
    for k in range(8):
        oracle_sweep_symmetric(st)
        brute_sweep_symmetric(bs)
        assert max_rel_err(np.exp(st.lam0), bs.U0, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.omega), bs.W, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.lamT), bs.UT, 1e-300) < 1e-12, k
    F, _ = readout_flows(st)
    assert max_rel_err(F, arc_flows(p, bs.tensor()), 1e-300) < 1e-12


def test_symmetric_gs_dual_monotone_and_same_optimum():
    """BCA with the symmetric block order: the dual never decreases after any block, and the iteration
    reaches the Gauss-Seidel optimum (the unique minimiser)."""
    p = grid_problem(3, 3, 4, 2, 0.5, seed=13, cap=(0.15, 0.4))
    st = oracle_init(p)
    vals = []
    for _ in range(20):
        oracle_sweep_symmetric(st, on_block=lambda kind, t, mass: vals.append(dual_objective(st, mass)))
    v = np.array(vals)
    assert np.all(np.diff(v) >= -1e-12 * np.abs(v).max())
    sym = oracle_run(p, 300, schedule="sym")
    gs = oracle_run(p, 300)
    Fs, Ws = readout_flows(sym)
    Fg, Wg = readout_flows(gs)
    assert max_rel_err(Ws, Wg, 1e-12) < 1e-8 and max_rel_err(Fs, Fg, 1e-12) < 1e-8
    assert np.any(Wg < 0.99)


# ---------------------------------------------------------------------------------------------
# NEXT-3: node (state) capacities, Algorithm 2's u_t on the states (eq:multicommodity P:676-683)

def _node_caps(p, seed, frac=0.5, lo=0.2, hi=0.6, tv=False):
    import dataclasses
    rng = np.random.default_rng(seed)
    shape = (p.T + 1, p.N) if tv else (p.N,)
    d = rng.uniform(lo, hi, size=shape)
    d[rng.random(shape) > frac] = np.inf
    return dataclasses.replace(p, node_cap=d)


@pytest.mark.parametrize("kw,tv", [(MICROS[0], False), (MICROS[1], True), (MICROS[4], False), (MICROS[6], False)])
def test_node_caps_iterates_identical_to_full_tensor(kw, tv):
    """P1 with node capacities: the GS blocks U0, W_0, u_1, W_1, ..., u_{T-1}, W_{T-1}, UT (prp:sinkhorn with the state
    marginals' inequality constraints) with every projection a literal sum of the full tensor M = K ⊙ U
    (U including prod_t u_t[v_t]) equal the oracle's sweeps iterate by iterate."""
    p = _node_caps(_micro(kw), seed=3, tv=tv)
    st = oracle_init(p)
    bs = BruteState(p)
    for k in range(8):
        oracle_sweep(st)
        brute_sweep(bs)
        assert max_rel_err(np.exp(st.lam0), bs.U0, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.omega), bs.W, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.nu), bs.Un, 1e-300) < 1e-12, k
        assert max_rel_err(np.exp(st.lamT), bs.UT, 1e-300) < 1e-12, k
    F, _ = readout_flows(st)
    assert max_rel_err(F, arc_flows(p, bs.tensor()), 1e-300) < 1e-12
    assert np.min(np.exp(st.nu)) < 0.99


def test_node_cap_on_a_single_in_arc_node_equals_the_arc_capacity():
    """A node whose only in-arc is a: its marginal at layer t is the flow of a at step t - 1, so a node capacity d on it
    (layers 1..T-1) is the arc capacity d on a at steps 0..T-2 — the already pinned arc-capacity path: same flows."""
    import dataclasses
    from workloads.configs import Problem
    # 0 -> 1 -> 2 -> 3 and 0 -> 4 -> 3 (loops at 0, 2, 3, 4; node 1's only in-arc is 0 -> 1)
    tail = np.array([0, 1, 2, 0, 4, 0, 2, 3, 4], np.int32)
    head = np.array([1, 2, 3, 4, 3, 0, 2, 3, 4], np.int32)
    T, A = 5, tail.size
    cost = np.array([0.2, 0.3, 0.1, 0.6, 0.5, 0.05, 0.05, 0.05, 0.05])
    p = Problem("chain", 5, tail, head, T, 0.3, cost, np.full(A, np.inf), 2, src=np.array([0, 0], np.int32),
                dst=np.array([3, 3], np.int32), mass=np.array([1.0, 0.7]))
    dn = np.full(5, np.inf)
    dn[1] = 0.6
    q = dataclasses.replace(p, node_cap=dn)
    cap = np.full((T, A), np.inf)
    cap[: T - 1, 0] = 0.6
    r = dataclasses.replace(p, cap=cap)
    Fq, _ = readout_flows(oracle_run(q, 6))
    Fr, _ = readout_flows(oracle_run(r, 6))
    assert max_rel_err(Fq, Fr, 1e-300) < 1e-12
    assert Fq[: T - 1, 0].max() > 0.3


def test_node_caps_dual_monotone_and_strong_duality():
    """BCA with the node blocks: the dual (now with sum <d_t, log u_t>) never decreases after any block, and
    at convergence equals the regularised primal of the brute-force tensor (thm:solution P:777-788)."""
    p = _node_caps(grid_problem(2, 3, 4, 2, 0.5, seed=2, cap=(0.3, 0.6)), seed=5, lo=0.3, hi=0.8, frac=0.6)
    st = oracle_init(p)
    vals = []
    for _ in range(15):
        oracle_sweep(st, on_block=lambda kind, t, mass: vals.append(dual_objective(st, mass)))
    v = np.array(vals)
    assert np.all(np.diff(v) >= -1e-12 * np.abs(v).max())
    for _ in range(3000):
        oracle_sweep(st)
    M = full_tensor(p, np.exp(st.lam0), np.exp(st.omega), np.exp(st.lamT), np.exp(st.nu))
    C = _cost_tensor(p)
    pos = M > 0
    primal = (C[pos] * M[pos]).sum() + p.eps * (M[pos] * np.log(M[pos]) - M[pos]).sum()
    phi = dual_objective(st, float(np.exp(st.a[p.T] + st.lamT).sum()))
    assert abs(primal - phi) <= 1e-9 * abs(phi), (primal, phi)
    assert np.min(np.exp(st.nu)) < 0.99
    P = np.stack([commodity_marginal(M, t).sum(axis=0) for t in range(p.T + 1)])
    dn = np.broadcast_to(p.node_cap, P.shape)
    assert np.all(P[1:p.T] <= dn[1:p.T] * (1 + 1e-8))
