"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle, element by element.

Tolerances are BASELINE.json north_star's: max relative error 1e-10 on edge flows and capacity
duals in fp64 mode, 1e-4 in fp32 mode (metric: SURVEY §8(c) Q11, tests/_metrics.py).
"""
import numpy as np
import pytest

from oracle import oracle_run, readout_flows, stats as oracle_stats
from oracle.sweep import dual_terms
from workloads import gen, grid_problem
from tests._metrics import max_rel_err, flow_floor, W_FLOOR

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-10, "fp32": 1e-4}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_14485_b200.build import build
    build()


def run_gpu(p, sweeps, prec, **kw):
    from paper_2106_14485_b200 import Solver
    with Solver(p, prec=prec, **kw) as s:
        s.sweep(sweeps)
        s.sync()
        F, W = s.edge_flows(), s.cap_duals()
        st = s.stats()
    return F, W, st


def run_oracle(p, sweeps, **kw):
    st = oracle_run(p, sweeps, **kw)
    F, W = readout_flows(st)
    so = oracle_stats(st)
    so["dual_scale"] = p.eps * (so["mass"] + sum(abs(x) for x in dual_terms(st)))
    return F, W, so


def assert_stats(sg, so, prec, F=None):
    """Every mmf_read_stats field against the oracle's end-of-sweep statistics.  The dual
    is a sum of large terms of both signs (eps * (-mass + <mu0, lam0> + <muT, lamT> + <d, omega>), thm:solution
    P:786-788): its tolerance scales with the sum of their magnitudes; marginal mismatches and the capacity
    violation are differences of near-equal numbers: absolute tolerances relative to the mass / flows."""
    tol = 10 * TOL[prec]
    m = abs(so["mass"])
    assert abs(sg["mass"] - so["mass"]) <= tol * m, ("mass", sg["mass"], so["mass"])
    assert abs(sg["primal"] - so["primal"]) <= tol * max(abs(so["primal"]), 1e-300), ("primal", sg["primal"], so["primal"])
    assert abs(sg["dual"] - so["dual"]) <= tol * so["dual_scale"], ("dual", sg["dual"], so["dual"])
    for k in ("src_mismatch", "sink_mismatch"):
        assert abs(sg[k] - so[k]) <= tol * m, (k, sg[k], so[k])
    fmax = float(np.max(F)) if F is not None and F.size else m
    assert abs(sg["cap_violation"] - so["cap_violation"]) <= tol * fmax, ("cap_violation", sg["cap_violation"],
                                                                          so["cap_violation"])


def assert_parity(p, sweeps, prec, oracle_kw=None, **kw):
    Fo, Wo, so = run_oracle(p, sweeps, **(oracle_kw or {}))
    Fg, Wg, sg = run_gpu(p, sweeps, prec, **kw)
    ef = max_rel_err(Fg, Fo, flow_floor(p))
    ew = max_rel_err(Wg, Wo, W_FLOOR)
    assert ef < TOL[prec] and ew < TOL[prec], (p.name, prec, ef, ew)
    assert sg["sweeps"] == so["sweeps"] == sweeps
    assert_stats(sg, so, prec, Fo)
    return ef, ew


MICROS = [
    dict(rows=2, cols=2, T=3, L=2, eps=0.5, seed=1),
    dict(rows=2, cols=3, T=4, L=3, eps=0.7, seed=2),
    dict(rows=2, cols=2, T=1, L=2, eps=0.4, seed=3),
    dict(rows=2, cols=3, T=3, L=1, eps=0.5, seed=4),
    dict(rows=2, cols=2, T=4, L=3, eps=0.6, seed=5, marginals="dense"),
    dict(rows=2, cols=3, T=3, L=2, eps=0.5, seed=6, time_varying=True),
    dict(rows=2, cols=3, T=4, L=2, eps=0.5, seed=8, closed_arcs=3, marginals="dense"),
]


def _micro(kw):
    kw = dict(kw)
    return grid_problem(kw.pop("rows"), kw.pop("cols"), kw.pop("T"), kw.pop("L"), kw.pop("eps"), **kw)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("kw", MICROS)
def test_micro_parity(kw, prec):
    assert_parity(_micro(kw), 10, prec)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tiny_config1(prec):
    p = gen(1)
    assert_parity(p, p.sweeps, prec)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("L,marg", [(37, "point"), (300, "point"), (45, "dense"), (1, "dense")])
def test_ragged_and_multi_group(L, marg, prec):
    """L not a multiple of the warp width (ragged tail) and L spanning several commodity groups."""
    p = grid_problem(6, 7, 9, L, 0.2, seed=21, cap=(0.3, 1.5), marginals=marg)
    assert_parity(p, 8, prec)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tight_capacities_long_run(prec):
    p = grid_problem(5, 5, 12, 6, 0.1, seed=22, cap=(0.1, 0.5))
    assert_parity(p, 40, prec)


def test_graph_capture_bitwise_equal_to_stream_launches():
    p = grid_problem(5, 6, 8, 20, 0.2, seed=23)
    F1, W1, _ = run_gpu(p, 5, "fp32", graph=True)
    F2, W2, _ = run_gpu(p, 5, "fp32", graph=False)
    assert np.array_equal(F1, F2) and np.array_equal(W1, W2)


def test_reorder_invisible():
    p = grid_problem(6, 6, 8, 12, 0.2, seed=24)
    F1, W1, _ = run_gpu(p, 6, "fp64", reorder=True)
    F2, W2, _ = run_gpu(p, 6, "fp64", reorder=False)
    assert max_rel_err(F1, F2, flow_floor(p)) < 1e-12 and max_rel_err(W1, W2, W_FLOOR) < 1e-12


def test_infeasible_is_sticky_error():
    from paper_2106_14485_b200 import MMFError
    p = grid_problem(3, 3, 2, 1, 0.5, seed=20)
    p.src = np.array([0], np.int32)
    p.dst = np.array([8], np.int32)
    with pytest.raises(MMFError) as e:
        run_gpu(p, 1, "fp64")
    assert e.value.name == "MMF_EINFEASIBLE"


def test_validation_errors():
    import dataclasses
    from paper_2106_14485_b200 import MMFError, Solver
    p = grid_problem(3, 3, 4, 2, 0.5, seed=25)
    bad = [
        dataclasses.replace(p, eps=0.0),
        dataclasses.replace(p, cap=np.where(np.isfinite(p.cap), -1.0, p.cap)),
        dataclasses.replace(p, tail=np.r_[p.tail, p.tail[:1]], head=np.r_[p.head, p.head[:1]],
                            cost=np.r_[p.cost, p.cost[:1]], cap=np.r_[p.cap, p.cap[:1]]),
        dataclasses.replace(p, mass=None, src=None, dst=None, mu0_dense=p.mu0, muT_dense=p.muT * 1.5),
        dataclasses.replace(p, cost=np.where(p.tail == p.head, np.nan, p.cost)),
    ]
    for q in bad:
        with pytest.raises(MMFError) as e:
            Solver(q, prec="fp64")
        assert e.value.name == "MMF_EINVAL"
    for key, val in [("kernels", 2), ("kernels", 7), ("bwd", 4), ("pexch", 2), ("fgw", 3)]:  # (removed / unknown values)
        with pytest.raises(MMFError) as e:
            Solver(p, prec="fp32", options={key: val})
        assert e.value.name == "MMF_EINVAL", (key, val)


@pytest.mark.parametrize("prec,opts", [("fp32", dict(kernels=1)), ("fp64", dict(kernels=1)), ("fp32", dict(kernels=5)),
                                       ("fp64", dict(kernels=5)), ("fp32", dict(kernels=5, tile=9)),
                                       ("fp32", dict(cpt=1)), ("fp32", dict(cpt=2)),
                                       ("fp32", dict(cpt=4)), ("fp32", dict(cpt=8)), ("fp64", dict(cpt=1)),
                                       ("fp64", dict(cpt=2)), ("fp32", dict(tile=1)), ("fp32", dict(tile=7)),
                                       ("fp64", dict(tile=128)), ("fp32", dict(reorder=0)),
                                       ("fp32", dict(kernels=3)), ("fp64", dict(kernels=3)),
                                       ("fp32", dict(kernels=3, cpt=8)), ("fp32", dict(kernels=4, cpt=8)),
                                       ("fp32", dict(kernels=6)), ("fp64", dict(kernels=6)),
                                       ("fp32", dict(order=1)), ("fp32", dict(order=3)), ("fp32", dict(stripw=4)),
                                       ("fp32", dict(bwd=2, wintma=0)), ("fp32", dict(bwd=3))])
def test_kernel_variants(prec, opts):
    """Every kernel configuration (reference per-node kernels, lane widths, tile sizes, no reordering)
    meets the same parity bar; several tiles, several chunks and a ragged commodity tail."""
    p = grid_problem(6, 7, 9, 150, 0.2, seed=26, cap=(0.3, 1.5))
    assert_parity(p, 6, prec, options=opts)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_dense_time_varying_closed(prec):
    p = grid_problem(5, 6, 7, 70, 0.25, seed=27, marginals="dense", time_varying=True, closed_arcs=2)
    assert_parity(p, 8, prec)


@pytest.mark.parametrize("prec,cpt", [("fp32", 1), ("fp32", 2), ("fp64", 1)])
def test_many_chunks_streaming_path(prec, cpt):
    """More than 8 commodity chunks per node: the forward kernel's warps loop over chunks and re-gather
    (no register-held rows); also nodes of in-degree above the register batch (the 3x3 grid has degree 5)."""
    p = grid_problem(5, 6, 7, 300, 0.25, seed=28, cap=(0.2, 0.8))
    assert_parity(p, 6, prec, options=dict(cpt=cpt))


FIXTURES = [("cfg3", 3, "fp32"), ("cfg3", 10, "fp32"), ("cfg4", 3, "fp32"), ("cfg5", 3, "fp32"),
            ("cfg4lite", 3, "fp32"), ("cfg4lite", 20, "fp32"), ("cfg5lite", 3, "fp32"), ("cfg5lite", 20, "fp32"),
            ("cfg5pipe", 3, "fp32"), ("cfg2", 100, "fp64"), ("cfg2", 100, "fp32")]


@pytest.mark.parametrize("name,k,prec", FIXTURES)
def test_config_parity_against_stored_oracle(name, k, prec):
    """BASELINE configs too slow for a live oracle: the GPU path (default launch configuration, as bench.py runs it)
    vs the float64 oracle's outputs stored by tests/golden/make_oracle_fixtures.py (which calls only oracle/ and
    workloads/), on uniformly sampled (t, a) entries (20,000; 100,000 for the full [4] / [5]), whole rows F_t, W_t at
    four steps where stored, and every end-of-sweep statistic.  cfg3 / cfg4 / cfg5 = configs [3] / [4] / [5] at full
    size and their SURVEY §8(c) Q21 sweep counts; cfg5pipe = the full [5] graph at L = 512 on a short horizon;
    *lite = the full [4] / [5] graphs and horizons at small L."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_{name}.npz")
    assert os.path.exists(path), f"fixture {name} missing"
    z = np.load(path)
    assert f"F_{k}" in z, f"fixture {name} has no snapshot {k}"
    from tests.golden.make_oracle_fixtures import JOBS
    cfg, kw, _ = JOBS[name]
    p = gen(cfg, **kw)
    assert (p.L, p.T, p.A, p.N) == (int(z["L"]), int(z["T"]), int(z["A"]), int(z["N"]))
    Fg, Wg, sg = run_gpu(p, k, prec)
    idx = z["idx"]
    ef = max_rel_err(Fg.reshape(-1)[idx], z[f"F_{k}"], flow_floor(p))
    ew = max_rel_err(Wg.reshape(-1)[idx], z[f"W_{k}"], W_FLOOR)
    assert ef < TOL[prec] and ew < TOL[prec], (name, k, ef, ew)
    if f"Frows_{k}" in z:
        rows = z["rows"]
        assert max_rel_err(Fg[rows], z[f"Frows_{k}"], flow_floor(p)) < TOL[prec]
        assert max_rel_err(Wg[rows], z[f"Wrows_{k}"], W_FLOOR) < TOL[prec]
    tol = 10 * TOL[prec]
    m = float(z[f"mass_{k}"])
    assert abs(sg["mass"] - m) <= tol * abs(m)
    assert abs(sg["primal"] - float(z[f"primal_{k}"])) <= tol * abs(float(z[f"primal_{k}"]))
    for key in ("src_mismatch", "sink_mismatch"):
        assert abs(sg[key] - float(z[f"{key}_{k}"])) <= tol * m, (key, sg[key], float(z[f"{key}_{k}"]))
    assert abs(sg["cap_violation"] - float(z[f"cap_violation_{k}"])) <= tol * float(np.max(Fg))
    if f"dual_scale_{k}" in z:
        assert abs(sg["dual"] - float(z[f"dual_{k}"])) <= tol * float(z[f"dual_scale_{k}"]), (sg["dual"], float(z[f"dual_{k}"]))


@pytest.mark.parametrize("bwd", [0, 1, 2, 3])
def test_pipelined_kernels_L1024_grid(bwd):
    """L = 1024 (the bench's commodity count on [4]: one 1024-commodity slice per node, 4 commodities per
    lane in the pipelined forward and backward kernels) on a 20 x 20 grid, live oracle; every backward
    variant (auto, three-pipeline TMA, sliding window, single-pipeline TMA)."""
    p = grid_problem(20, 20, 12, 1024, 0.1, seed=29, cap=(0.5, 3.0))
    assert_parity(p, 3, "fp32", options=dict(bwd=bwd))


def _hub_problem(L, nhub=22):
    """A 10 x 10 grid plus a hub (node 0 linked both ways to nhub other nodes: degree nhub + 3, above the
    pipelined kernels' register paths) and a node whose in-arcs and self-loop are all closed (no rows once its
    factors reach 0: the empty-item path).  nhub = 8 keeps the widest item small enough for 1024-commodity
    pipelined slices; nhub = 22 selects 512-commodity slices."""
    import dataclasses
    p = grid_problem(10, 10, 6, L, 0.1, seed=35, cap=(0.5, 3.0))
    hub = np.arange(30, 30 + nhub, dtype=np.int32)
    tail = np.r_[p.tail, hub, np.zeros_like(hub)].astype(np.int32)
    head = np.r_[p.head, np.zeros_like(hub), hub].astype(np.int32)
    cost = np.r_[p.cost, np.full(2 * hub.size, 0.7)]
    cap = np.r_[p.cap, np.full(2 * hub.size, 2.0)]
    cap[head == 55] = 0.0  # (node 55: closed in-arcs and loop)
    src, dst = p.src.copy(), p.dst.copy()
    dst[dst == 55] = 56
    src[src == dst] = 57
    # (OD pairs were drawn within 6 hops; 8 steps leave room for the detours around node 55)
    return dataclasses.replace(p, tail=tail, head=head, cost=cost, cap=cap, src=src, dst=dst, T=8, name=f"hub-L{L}")


@pytest.mark.parametrize("L,nhub,opts", [(1019, 22, {}), (1019, 22, dict(bwd=1, wrap=0)), (509, 22, {}),
                                         (1019, 8, {}), (1019, 8, dict(fgw=4, fng=2, fnp=2))])
def test_pipelined_hub_and_empty_items(L, nhub, opts):
    """High-degree items (streaming paths of the pipelined forward and backward) and empty items, live oracle."""
    assert_parity(_hub_problem(L, nhub), 3, "fp32", options=opts)


@pytest.mark.parametrize("L,marg,tv", [(1019, "dense", False), (1019, "point", True), (509, "dense", True),
                                       (251, "point", True)])
def test_pipelined_time_varying_and_dense(L, marg, tv):
    """The production (pipelined) path with per-step costs and capacities ([T][A] K, d: per-step records and
    dual-update operands), closed arcs, and dense marginals (a2 / a4 over every node)."""
    p = grid_problem(9, 9, 6, L, 0.2, seed=43, cap=(0.3, 1.2), marginals=marg, time_varying=tv,
                     closed_arcs=4 if marg == "dense" else 0)  # (closing arcs could cut a point OD pair's only path)
    assert_parity(p, 3, "fp32")


@pytest.mark.parametrize("L", [1019, 251])
def test_pipelined_forward_large_ratio_recompute(L):
    """Arcs with capacities 1e-14 of the flow they would carry: the first dual updates move W by more than 2^40,
    so the pipelined forward takes its recompute-from-shared-memory path for those items."""
    p = grid_problem(10, 10, 6, L, 0.2, seed=42, cap=(0.3, 1.2))
    moving = np.flatnonzero(p.tail != p.head)
    p.cap[moving[::7]] = 1e-14
    assert_parity(p, 3, "fp32")


@pytest.mark.parametrize("theta", [500, 1000, 200])
@pytest.mark.parametrize("which", ["grid", "hub"])
def test_jacobi_schedule(which, theta):
    """the damped Jacobi schedule (option schedule=1, theta_milli) in the pipelined
    forward against the oracle's Jacobi sweep (tests/test_oracle_pins.py pins it), 1024-commodity slices."""
    p = grid_problem(12, 12, 8, 1019, 0.1, seed=31, cap=(0.3, 1.5)) if which == "grid" else _hub_problem(1019, 8)
    assert_parity(p, 4, "fp32", oracle_kw=dict(schedule="jacobi", theta=theta / 1000.0),
                  options=dict(schedule=1, theta_milli=theta))


@pytest.mark.parametrize("prec,L,check", [("fp32", 1019, 1), ("fp64", 37, 1), ("fp32", 1019, 3)])
def test_solve_to_tolerance(prec, L, check):
    """mmf_solve (on-device marginal-mismatch and capacity-excess reductions) stops at the
    same sweep as the oracle's solve loop (tol placed between the oracle's errors of two consecutive checks),
    with the same state; the error history matches the oracle's."""
    from oracle import oracle_solve
    from paper_2106_14485_b200 import Solver
    # (total masses chosen so that capacities bind and the error decays geometrically over the 12 sweeps)
    p = grid_problem(8, 8, 6, L, 0.2, seed=37, cap=(0.1, 0.3), mass=np.full(L, (8.0 if L > 100 else 4.0) / L))
    _, _, _, _, hist = oracle_solve(p, 0.0, 12, check)
    floor = 1e-5 if prec == "fp32" else 1e-9  # (errors well above the arithmetic's own noise)
    k = next(i for i in range(1, len(hist)) if hist[i] < 0.95 * hist[i - 1] and hist[i] > floor)
    tol = (hist[k] * hist[k - 1]) ** 0.5
    st, conv, sweeps, err, hist_o = oracle_solve(p, tol, 12, check)
    assert conv
    with Solver(p, prec=prec) as s:
        r = s.solve(tol, 12, check)
        F, W = s.edge_flows(), s.cap_duals()
    assert r["converged"] and r["sweeps"] == sweeps
    assert np.all(np.abs(r["history"] - np.array(hist_o)) <= 1e-2 * np.array(hist_o) + 0.1 * floor), (r, hist_o)
    Fo, Wo = readout_flows(st)
    assert max_rel_err(F, Fo, flow_floor(p)) < TOL[prec] and max_rel_err(W, Wo, W_FLOOR) < TOL[prec]
    with Solver(p, prec=prec) as s:
        r0 = s.solve(tol, 0, check)
    assert not r0["converged"] and r0["sweeps"] == 0


@pytest.mark.parametrize("prec,L,opts_b", [("fp32", 1019, None), ("fp64", 37, None), ("fp32", 1019, dict(kernels=3)),
                                          ("fp32", 150, dict(cpt=1))])
def test_checkpoint_resume(prec, L, opts_b):
    """save after 3 sweeps, load into a fresh context, 2 more sweeps == 5 uninterrupted
    sweeps — bitwise with the same options, within the parity tolerance across kernel configurations — and
    equal to the oracle's 5 sweeps; a state of another problem is rejected."""
    from paper_2106_14485_b200 import MMFError, Solver
    p = grid_problem(9, 9, 7, L, 0.2, seed=38, cap=(0.3, 1.2))
    with Solver(p, prec=prec) as a:
        a.sweep(3)
        state = a.save_state()
        a.sweep(2)
        Fa, Wa = a.edge_flows(), a.cap_duals()
        sa = a.stats()
    with Solver(p, prec=prec, options=opts_b) as b:
        b.load_state(state)
        b.sweep(2)
        Fb, Wb = b.edge_flows(), b.cap_duals()
        sb = b.stats()
    assert sb["sweeps"] == sa["sweeps"] == 5
    if opts_b is None:
        assert np.array_equal(Fa, Fb) and np.array_equal(Wa, Wb)
    else:
        assert max_rel_err(Fb, Fa, flow_floor(p)) < TOL[prec] and max_rel_err(Wb, Wa, W_FLOOR) < TOL[prec]
    Fo, Wo, _ = run_oracle(p, 5)
    assert max_rel_err(Fb, Fo, flow_floor(p)) < TOL[prec] and max_rel_err(Wb, Wo, W_FLOOR) < TOL[prec]
    q = grid_problem(9, 8, 7, L, 0.2, seed=38, cap=(0.3, 1.2))
    with Solver(q, prec=prec) as c:
        with pytest.raises(MMFError) as e:
            c.load_state(state)
        assert e.value.name == "MMF_EINVAL"


@pytest.mark.parametrize("prec,L,opts", [("fp32", 1019, {}), ("fp64", 37, {}), ("fp32", 150, dict(kernels=1)),
                                        ("fp32", 70, dict(kernels=6))])
def test_commodity_flows_readout(prec, L, opts):
    """per-commodity arc flows F^l_t of the end-of-sweep state against the oracle's
    cor:proj readout, element by element, at the first, a middle and the last step; their commodity sum is the
    edge-flow readout."""
    from oracle import readout_commodity_flows
    from paper_2106_14485_b200 import Solver
    p = grid_problem(7, 7, 6, L, 0.2, seed=39, cap=(0.3, 1.2))
    st = oracle_run(p, 3)
    with Solver(p, prec=prec, options=opts) as s:
        s.sweep(3)
        F = s.edge_flows()
        for t in (0, 3, p.T - 1):
            Fl = s.commodity_flows(t)
            ref = readout_commodity_flows(st, t)
            assert Fl.shape == ref.shape == (p.A, p.L)
            assert max_rel_err(Fl, ref, 1e-30 * float(p.mass.max())) < TOL[prec], t
            assert max_rel_err(Fl.sum(axis=1), F[t], flow_floor(p)) < TOL[prec]


@pytest.mark.parametrize("prec,L,opts", [("fp64", 37, {}), ("fp32", 150, dict(kernels=3)), ("fp64", 20, dict(kernels=1)),
                                        ("fp32", 300, dict(kernels=5)), ("fp32", 60, dict(kernels=4))])
def test_jacobi_schedule_every_kernel_family(prec, L, opts):
    """The Jacobi sweep (one forward pass in readout mode, one bulk update, the backward pass) on every kernel
    family and both precisions, against the oracle."""
    p = grid_problem(6, 7, 6, L, 0.2, seed=40, cap=(0.3, 1.2), marginals="dense" if L == 20 else "point")
    assert_parity(p, 4, prec, oracle_kw=dict(schedule="jacobi", theta=0.5),
                  options=dict(schedule=1, theta_milli=500, **opts))


@pytest.mark.parametrize("wrap", [0, 1])
@pytest.mark.parametrize("L", [1024, 512])
def test_pipelined_backward_ring_wrap(L, wrap):
    """The three-pipeline backward with items that may wrap around the ring (per-row offsets) and with
    items that never wrap (the producer skips to slot 0), on a grid with a ragged commodity tail."""
    p = grid_problem(14, 14, 8, L - 3, 0.1, seed=33, cap=(0.5, 3.0))
    assert_parity(p, 2, "fp32", options=dict(bwd=1, wrap=wrap))


@pytest.mark.parametrize("L,fgw,fng,fnp", [(1024, 8, 1, 2), (1024, 4, 2, 2), (1024, 4, 3, 1), (512, 8, 1, 2),
                                           (512, 4, 2, 2), (256, 2, 4, 2)])
def test_pipelined_forward_groups(L, fgw, fng, fnp):
    """Every compiled consumer-group layout of the pipelined forward (fgw warps per group, fng groups per
    pipeline, fnp pipelines per CTA; 32 * fgw * CPT = the slice width) against the live oracle, on a grid
    whose in-degrees (2..5 plus the loop) exercise the register paths and a ragged commodity tail."""
    p = grid_problem(12, 12, 8, L - 5 if L > 256 else L, 0.1, seed=31, cap=(0.5, 3.0))
    assert_parity(p, 2, "fp32", options=dict(fgw=fgw, fng=fng, fnp=fnp))


def _invariants(p, F, W, rtol):
    """Properties of the end-of-sweep readout that hold at any size: F >= 0, W in [0, 1],
    per-step mass = total commodity mass (the sink marginal is exact after a4, and point-mass sources carry
    all of their commodity's mass), and node conservation of the aggregate flow between consecutive steps."""
    m_tot = float(np.sum(p.mass)) if p.is_point else float(p.mu0.sum())
    assert np.all(F >= 0) and np.all(np.isfinite(F))
    assert np.all((W >= 0) & (W <= 1))
    mass_t = F.sum(axis=1)
    assert np.max(np.abs(mass_t - m_tot)) <= rtol * m_tot, np.max(np.abs(mass_t - m_tot))
    into = np.zeros((p.T, p.N))
    outof = np.zeros((p.T, p.N))
    for t in range(p.T):
        into[t] = np.bincount(p.head, weights=F[t], minlength=p.N)
        outof[t] = np.bincount(p.tail, weights=F[t], minlength=p.N)
    lhs, rhs = into[:-1], outof[1:]
    scale = np.maximum(np.maximum(np.abs(lhs), np.abs(rhs)), 1e-6 * m_tot)
    assert np.max(np.abs(lhs - rhs) / scale) <= rtol, np.max(np.abs(lhs - rhs) / scale)


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_config_invariants(cfg):
    """The BASELINE configs at full size in the launch configuration bench.py times (default options,
    CUDA-graph sweeps): exact-identity checks of the readout after the parity sweep count."""
    p = gen(cfg)
    F, W, st = run_gpu(p, p.sweeps, "fp32")
    _invariants(p, F, W, 2e-4)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_nccl_jacobi_bulk_exchange_one_rank(prec):
    """The Jacobi schedule's single T x |A| flow all-reduce per sweep on a one-rank NCCL
    communicator, against the oracle's Jacobi sweep."""
    import torch
    torch.cuda.nccl.version()  # loads the NCCL the library resolves at run time
    from paper_2106_14485_b200 import _lib
    p = grid_problem(5, 6, 6, 40, 0.2, seed=41, cap=(0.3, 1.2))
    assert_parity(p, 4, prec, oracle_kw=dict(schedule="jacobi", theta=0.5), nccl_uid=_lib.mmf_nccl_unique_id(),
                  nranks=1, rank=0, options=dict(schedule=1, theta_milli=500))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_nccl_exchange_path_one_rank(prec):
    """The library's commodity-sharded sweep (per forward step: partial flows -> ncclAllReduce -> capacity-
    dual update) on a one-rank NCCL communicator: same kernels and exchange calls as the
    multi-GPU run, checked against the oracle."""
    import torch
    torch.cuda.nccl.version()  # loads the NCCL the library resolves at run time
    from paper_2106_14485_b200 import _lib
    uid = _lib.mmf_nccl_unique_id()
    p = grid_problem(6, 7, 9, 150, 0.2, seed=26, cap=(0.3, 1.5))
    assert_parity(p, 6, prec, nccl_uid=uid, nranks=1, rank=0)


# ---------------------------------------------------------------------------------------------
# round 2: readouts before any sweep / right after a state load, error paths, [5]'s wide-lane forward,
# the pipelined Jacobi bulk exchange, a negative control

@pytest.mark.parametrize("prec,L", [("fp32", 1019), ("fp64", 37)])
def test_readout_after_init_and_after_load_without_sweep(prec, L):
    """mmf_init leaves U0 = 0 (Alg. 2 computes U0 first; the oracle's lam0 = -inf), so a readout before
    any sweep returns the zero tensor's flows, equal to the oracle's 0-sweep readout; a state loaded into a fresh
    context reads out (flows, duals, stats) bitwise like the context that saved it, without a sweep."""
    from paper_2106_14485_b200 import Solver
    p = grid_problem(9, 9, 7, L, 0.2, seed=38, cap=(0.3, 1.2))
    Fo0, Wo0, so0 = run_oracle(p, 0)
    with Solver(p, prec=prec) as a:
        F0, W0 = a.edge_flows(), a.cap_duals()
        assert np.array_equal(F0, Fo0) and np.array_equal(W0, Wo0)
        assert a.stats()["mass"] == 0.0
        a.sweep(3)
        state = a.save_state()
        Fa, Wa, sa = a.edge_flows(), a.cap_duals(), a.stats()
    with Solver(p, prec=prec) as b:
        b.load_state(state)
        Fb, Wb, sb = b.edge_flows(), b.cap_duals(), b.stats()
    assert np.array_equal(Fa, Fb) and np.array_equal(Wa, Wb)
    for k in sa:  # (the device statistics reduce with atomics: equal up to summation order)
        assert abs(sa[k] - sb[k]) <= 1e-12 * max(abs(sa[k]), 1e-300), (k, sa[k], sb[k])
    Fo, Wo, so = run_oracle(p, 3)
    assert max_rel_err(Fb, Fo, flow_floor(p)) < TOL[prec] and max_rel_err(Wb, Wo, W_FLOOR) < TOL[prec]
    assert_stats(sb, so, prec, Fo)


def test_load_state_rejects_other_costs_and_corrupt_header():
    import dataclasses
    from paper_2106_14485_b200 import MMFError, Solver
    p = grid_problem(6, 6, 5, 40, 0.2, seed=38, cap=(0.3, 1.2))
    with Solver(p, prec="fp32") as a:
        a.sweep(1)
        state = a.save_state()
    for q in (dataclasses.replace(p, eps=0.21), dataclasses.replace(p, cost=p.cost * 1.01),
              dataclasses.replace(p, cap=p.cap * 0.5)):
        with Solver(q, prec="fp32") as c:
            with pytest.raises(MMFError) as e:
                c.load_state(state)
            assert e.value.name == "MMF_EINVAL"
    bad = bytearray(state)
    bad[:8] = b"MMFSTAT1"
    with Solver(p, prec="fp32") as c:
        with pytest.raises(MMFError):
            c.load_state(bytes(bad))
        with pytest.raises(MMFError):
            c.load_state(state[: len(state) // 2])


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_extended_exponent_overflow_is_sticky_erange(prec):
    """Every walk costs 12 (T = 12 unit-cost steps) at eps = 1e-3: the messages reach e^-12000 = 2^-17312, past the
    extended exponent's range (|e| <= 16000, xf.cuh): the sweep must raise MMF_ERANGE, not return
    garbage.  At eps = 2e-3 (2^-8656) the same instance is in range and matches the log-domain oracle."""
    from paper_2106_14485_b200 import MMFError
    p = grid_problem(3, 3, 12, 2, 1e-3, seed=44, move_cost=1.0, stay_cost=1.0, cap=None)
    with pytest.raises(MMFError) as e:
        run_gpu(p, 1, prec)
    assert e.value.name == "MMF_ERANGE"
    import dataclasses
    assert_parity(dataclasses.replace(p, eps=2e-3), 2, prec)


def test_out_of_order_calls_are_estate():
    """calling out of order returns MMF_ESTATE (sweep / readout before init, costs before graph,
    a pre-init option after init)."""
    import ctypes as C
    from paper_2106_14485_b200 import _lib as L
    lib = L.load()
    ctx = L.mmf_create(0, L.MMF_FP32, 0)
    try:
        assert lib.mmf_sweep(ctx, 1) == 8
        out = np.zeros(4)
        assert lib.mmf_read_edge_flows(ctx, out.ctypes.data_as(C.POINTER(C.c_double))) == 8
        cost = np.ones(4)
        assert lib.mmf_set_costs(ctx, 2, 0.1, cost.ctypes.data_as(C.POINTER(C.c_double)), 0) == 8
        assert lib.mmf_init(ctx) == 8
    finally:
        L.mmf_destroy(ctx)
    p = grid_problem(3, 3, 4, 2, 0.5, seed=25)
    from paper_2106_14485_b200 import MMFError, Solver
    with Solver(p, prec="fp32") as s:
        with pytest.raises(MMFError) as e:
            L.mmf_set_option(s.ctx, "kernels", 3)
        assert e.value.name == "MMF_ESTATE"


@pytest.mark.parametrize("bad", ["N0", "T0", "arc", "point"])
def test_setup_validation_einval(bad):
    """SURVEY §8(b) setup validation: N < 1, T < 1, out-of-range arc ids, out-of-range point-mass nodes."""
    import dataclasses
    from paper_2106_14485_b200 import MMFError, Solver
    p = grid_problem(3, 3, 4, 2, 0.5, seed=25)
    if bad == "N0":
        q = dataclasses.replace(p, N=0)
    elif bad == "T0":
        q = dataclasses.replace(p, T=0)
    elif bad == "arc":
        q = dataclasses.replace(p, head=np.where(np.arange(p.A) == 3, p.N, p.head).astype(np.int32))
    else:
        q = dataclasses.replace(p, dst=np.array([0, p.N], np.int32))
    with pytest.raises(MMFError) as e:
        Solver(q, prec="fp32")
    assert e.value.name == "MMF_EINVAL"


@pytest.mark.parametrize("L", [2051, 4099])
def test_wide_lane_multi_group_forward_fp32_default_options(L):
    """L > 1024: the forward of [5] (L = 8192) in its production configuration, the fp32 wide-lane kernel with 8
    commodities per lane and several 2048-commodity groups per node ("global partials + last arriver", wide.cuh),
    with the default options and a ragged commodity tail, against the live oracle element by element."""
    p = grid_problem(8, 8, 6, L, 0.1, seed=45, cap=(0.5 * L / 100, 3.0 * L / 100))
    assert_parity(p, 3, "fp32")


def test_nccl_jacobi_bulk_exchange_pipelined_one_rank():
    """The Jacobi schedule's bulk all-reduce with the pipelined readout-mode forward (MODE 3: fp32, L >= 256), on a
    one-rank NCCL communicator, against the oracle's Jacobi sweep (the fast path behind the 76 ms/sweep
    figure)."""
    import torch
    torch.cuda.nccl.version()
    from paper_2106_14485_b200 import _lib
    p = grid_problem(12, 12, 8, 1019, 0.1, seed=31, cap=(0.3, 1.5))
    assert_parity(p, 4, "fp32", oracle_kw=dict(schedule="jacobi", theta=0.5), nccl_uid=_lib.mmf_nccl_unique_id(),
                  nranks=1, rank=0, options=dict(schedule=1, theta_milli=500))


def test_negative_control_broken_kernel_fails_parity():
    """SURVEY §4 negative control: the parity harness must detect a wrong result.  (a) The GPU run on an input with
    ONE capacity changed by 0.1 % (a stand-in for a dropped or perturbed term) fails the fp32 comparison against the
    oracle of the original input, which the unchanged run passes; (b) the pipelined forward's diagnostic mode dry=3
    (skips the capacity-dual update: invalid by design) either fails the comparison or trips a sticky error."""
    from paper_2106_14485_b200 import MMFError
    p = grid_problem(12, 12, 8, 1019, 0.1, seed=31, cap=(0.3, 1.5))
    Fo, Wo, _ = run_oracle(p, 2)
    Fg, Wg, _ = run_gpu(p, 2, "fp32")
    assert max_rel_err(Wg, Wo, W_FLOOR) < TOL["fp32"] and max_rel_err(Fg, Fo, flow_floor(p)) < TOL["fp32"]
    a = int(np.argmin(Wo.min(axis=0)))
    assert Wo[:, a].min() < 0.99
    import dataclasses
    q = dataclasses.replace(p, cap=p.cap.copy())
    q.cap[a] *= 1.001
    Fg, Wg, _ = run_gpu(q, 2, "fp32")
    assert max_rel_err(Wg, Wo, W_FLOOR) > TOL["fp32"] and max_rel_err(Fg, Fo, flow_floor(p)) > TOL["fp32"]
    try:
        Fg, Wg, _ = run_gpu(p, 2, "fp32", options=dict(dry=3))
        assert max_rel_err(Wg, Wo, W_FLOOR) > 1e-2
    except MMFError:
        pass


# ---------------------------------------------------------------------------------------------
# NEXT-2: commodity-dependent node costs (the factor D = exp(-c/eps) at the intermediate layers)

def _node_cost(p, scale, seed=0):
    import dataclasses
    rng = np.random.default_rng(seed)
    return dataclasses.replace(p, node_cost=rng.uniform(0.0, scale, size=(p.L, p.N)))


@pytest.mark.parametrize("prec,L,marg,opts", [("fp64", 37, "point", {}), ("fp32", 1019, "point", {}),
                                              ("fp32", 150, "dense", {}), ("fp64", 20, "dense", dict(kernels=1)),
                                              ("fp32", 300, "point", dict(kernels=5)), ("fp32", 300, "point", dict(kernels=3)),
                                              ("fp32", 60, "point", dict(kernels=4)), ("fp32", 1019, "point", dict(bwd=2)),
                                              ("fp32", 2051, "point", {})])
def test_node_costs_parity(prec, L, marg, opts):
    """Commodity node costs on every kernel family (pipelined forward/backward, wide-lane incl. the L > 1024 multi-group
    forward, head-flow, tiles, per-node reference kernels, sliding window) against the oracle (pinned by brute force
    in tests/test_oracle_pins.py), flows, duals and every statistic."""
    p = _node_cost(grid_problem(7, 8, 6, L, 0.2, seed=46, cap=(0.3 * max(L, 100) / 100, 1.2 * max(L, 100) / 100),
                                marginals=marg), 0.5, seed=1)
    assert_parity(p, 4, prec, options=opts)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_node_costs_jacobi_readout_and_resume(prec):
    """Node costs with the Jacobi schedule, the per-commodity flow readout and checkpoint/resume (the state's problem
    hash covers the node costs: a state of the same problem without them is rejected)."""
    from oracle import readout_commodity_flows
    from paper_2106_14485_b200 import MMFError, Solver
    L = 1019 if prec == "fp32" else 37
    base = grid_problem(9, 9, 6, L, 0.2, seed=47, cap=(0.3, 1.2))
    p = _node_cost(base, 0.4, seed=2)
    assert_parity(p, 3, prec, oracle_kw=dict(schedule="jacobi", theta=0.5), options=dict(schedule=1, theta_milli=500))
    st = oracle_run(p, 3)
    with Solver(p, prec=prec) as s:
        s.sweep(3)
        Fl = s.commodity_flows(2)
        assert max_rel_err(Fl, readout_commodity_flows(st, 2), 1e-30 * float(p.mass.max())) < TOL[prec]
        state = s.save_state()
    with Solver(p, prec=prec) as s:
        s.load_state(state)
        s.sweep(1)
        F = s.edge_flows()
    Fo, _ = readout_flows(oracle_run(p, 4))
    assert max_rel_err(F, Fo, flow_floor(p)) < TOL[prec]
    with Solver(base, prec=prec) as s:
        with pytest.raises(MMFError):
            s.load_state(state)


@pytest.mark.parametrize("prec,L,G,marg", [("fp64", 37, 2, "point"), ("fp64", 45, 4, "dense"), ("fp32", 300, 3, "point"),
                                           ("fp32", 1019, 8, "point")])
def test_virtual_ranks_equal_unsharded(prec, L, G, marg):
    """G commodity shards on one GPU (mmf_sweep_group), each its own context, swept with the multi-GPU
    exchange path's kernels (shard partial flows -> device-side sum -> dual update, the coupling of rem:multi_tensor_scheme
    P:1139-1147): the capacity duals agree across shards and the summed flows equal the unsharded run (fp64 1e-12) and
    the oracle."""
    from paper_2106_14485_b200 import Solver, _lib
    sc = max(L, 100) / 100 if marg == "point" else 0.2
    p = grid_problem(7, 7, 7, L, 0.2, seed=48, cap=(0.3 * sc, 1.0 * sc), marginals=marg)
    per = (L + G - 1) // G
    bounds = [(min(g * per, L), min((g + 1) * per, L)) for g in range(G)]
    shards = [Solver(p, prec=prec, l_begin=a, l_count=b - a, options=dict(kernels=3)) for a, b in bounds]
    try:
        _lib.mmf_sweep_group([s.ctx for s in shards], 5)
        for s in shards:
            s.sync()
        F = sum(s.edge_flows() for s in shards)
        Ws = [s.cap_duals() for s in shards]
    finally:
        for s in shards:
            s.close()
    for W in Ws[1:]:
        assert np.array_equal(W, Ws[0])
    Fu, Wu, _ = run_gpu(p, 5, prec)
    tol = 1e-12 if prec == "fp64" else TOL[prec]
    assert max_rel_err(F, Fu, flow_floor(p)) < tol and max_rel_err(Ws[0], Wu, W_FLOOR) < tol
    Fo, Wo, _ = run_oracle(p, 5)
    assert max_rel_err(F, Fo, flow_floor(p)) < TOL[prec] and max_rel_err(Ws[0], Wo, W_FLOOR) < TOL[prec]
    assert np.min(Wo) < 0.99


# ---------------------------------------------------------------------------------------------
# NEXT-4: per-commodity entry / exit times

def _times(p, seed, T):
    """Horizon T with every commodity's window at least as long as the horizon its OD pair was drawn for (p.T)."""
    import dataclasses
    rng = np.random.default_rng(seed)
    t_in = rng.integers(0, T - p.T + 1, size=p.L)
    t_out = np.minimum(t_in + p.T + rng.integers(0, 2, size=p.L), T)
    return dataclasses.replace(p, T=T, t_in=t_in, t_out=t_out)


@pytest.mark.parametrize("prec,L,opts", [("fp64", 23, {}), ("fp32", 1019, {}), ("fp32", 150, dict(kernels=1)),
                                        ("fp32", 300, dict(kernels=3)), ("fp32", 1019, dict(schedule=1, theta_milli=500))])
def test_commodity_times_parity(prec, L, opts):
    """Commodities entering and leaving at their own layers (the library's holding-node construction, hidden from the
    readouts) against the oracle's native multi-tensor sweep (pinned by per-commodity window tensors), flows, duals and
    statistics; flows of a commodity vanish outside its window."""
    p = _times(grid_problem(8, 8, 8, L, 0.2, seed=49, cap=(0.3 * max(L, 100) / 100, 1.2 * max(L, 100) / 100)), seed=3,
               T=12)
    assert np.any(p.t_in > 0) and np.any(p.t_out < p.T)
    okw = dict(schedule="jacobi", theta=0.5) if opts.get("schedule") else None
    assert_parity(p, 4, prec, oracle_kw=okw, options=opts)
    if L == 23:
        from oracle import readout_commodity_flows
        from paper_2106_14485_b200 import Solver
        st = oracle_run(p, 4)
        with Solver(p, prec=prec) as s:
            s.sweep(4)
            for t in (0, 4, p.T - 1):
                Fl = s.commodity_flows(t)
                assert max_rel_err(Fl, readout_commodity_flows(st, t), 1e-30) < TOL[prec]
                absent = (t < p.t_in) | (t >= p.t_out)
                assert np.all(Fl[:, absent] == 0.0)


# ---------------------------------------------------------------------------------------------
# NEXT-1 remainder: symmetric Gauss-Seidel (option schedule = 2)

@pytest.mark.parametrize("prec,L,marg,opts", [("fp32", 1019, "point", {}), ("fp64", 37, "point", {}),
                                              ("fp64", 20, "dense", dict(kernels=1)), ("fp32", 300, "point", dict(kernels=3)),
                                              ("fp32", 60, "point", dict(kernels=4)), ("fp32", 300, "dense", dict(kernels=5))])
def test_symmetric_gs_parity(prec, L, marg, opts):
    """W updated in the forward and the backward pass (oracle_sweep_symmetric, pinned by the brute-force symmetric
    sweep) on every kernel family, flows, duals and statistics."""
    p = grid_problem(8, 8, 7, L, 0.2, seed=50, cap=(0.3 * max(L, 100) / 100, 1.2 * max(L, 100) / 100)
                     if marg == "point" else (0.05, 0.2), marginals=marg)
    assert_parity(p, 4, prec, oracle_kw=dict(schedule="sym"), options=dict(schedule=2, **opts))


def test_symmetric_gs_with_node_costs_and_times():
    import dataclasses
    p = grid_problem(8, 8, 8, 1019, 0.2, seed=51, cap=(3.0, 12.0))
    rng = np.random.default_rng(4)
    t_in = rng.integers(0, 3, size=p.L)
    p = dataclasses.replace(p, T=10, t_in=t_in, t_out=np.minimum(t_in + 8, 10),
                            node_cost=rng.uniform(0, 0.3, size=(p.L, p.N)))
    assert_parity(p, 3, "fp32", oracle_kw=dict(schedule="sym"), options=dict(schedule=2))


# ---------------------------------------------------------------------------------------------
# NEXT-3: node (state) capacities and the paper's state spaces on a synthetic street map

def _with_node_caps(p, seed, lo, hi, frac=0.5, tv=False):
    import dataclasses
    rng = np.random.default_rng(seed)
    shape = (p.T + 1, p.N) if tv else (p.N,)
    d = rng.uniform(lo, hi, size=shape)
    d[rng.random(shape) > frac] = np.inf
    return dataclasses.replace(p, node_cap=d)


def _node_parity(p, sweeps, prec, opts, oracle_kw=None):
    from paper_2106_14485_b200 import Solver
    assert_parity(p, sweeps, prec, oracle_kw=oracle_kw, options=opts)
    st = oracle_run(p, sweeps, **(oracle_kw or {}))
    with Solver(p, prec=prec, options=opts) as s:
        s.sweep(sweeps)
        U = s.node_duals()
    assert max_rel_err(U, np.exp(st.nu), W_FLOOR) < TOL[prec]
    assert np.min(np.exp(st.nu)) < 0.99


@pytest.mark.parametrize("prec,L,marg,opts,tv", [("fp32", 1019, "point", {}, False), ("fp64", 20, "point", dict(kernels=1), True),
                                                 ("fp32", 30, "dense", dict(kernels=1), False),
                                                 ("fp32", 1019, "point", dict(schedule=2), False)])
def test_node_caps_parity(prec, L, marg, opts, tv):
    """Node capacities (Algorithm 2's u_t on the states, k_node_cap after each forward step; pinned against brute-force
    tensors in tests/test_oracle_pins.py): flows, arc duals, node duals and statistics against the oracle."""
    sc = L / 64  # (mean node marginal)
    p = _with_node_caps(grid_problem(8, 8, 7, L, 0.2, seed=52, cap=(5 * sc, 20 * sc), marginals=marg), 3, 0.4 * sc,
                        1.5 * sc, tv=tv)
    okw = dict(schedule="sym") if opts.get("schedule") == 2 else None
    _node_parity(p, 4, prec, opts, okw)


def test_node_caps_unsupported_family_is_einval():
    from paper_2106_14485_b200 import MMFError, Solver
    p = _with_node_caps(grid_problem(5, 5, 5, 20, 0.2, seed=52), 3, 1.0, 2.0)
    with pytest.raises(MMFError) as e:
        Solver(p, prec="fp64")  # (fp64 default: the wide-lane kernels)
    assert e.value.name == "MMF_EINVAL"


@pytest.mark.parametrize("policy,prec,L,opts", [("edges+stay", "fp32", 257, {}), ("vertex_storage", "fp32", 300, {}),
                                                ("traffic", "fp32", 300, {}), ("traffic", "fp64", 12, dict(kernels=1)),
                                                ("vertex_storage", "fp64", 12, dict(kernels=1))])
def test_state_space_problems_parity(policy, prec, L, opts):
    """The arc-state (edges with staying), vertex-storage and traffic-routing state spaces of P:612, P:704-720 on a
    synthetic street map of the §5.3 size (57 junctions, 150 directed streets): state capacities (node capacities),
    commodity state costs C_L (node costs), against the oracle."""
    from workloads.statespace import state_problem
    p = state_problem(policy, T=12, eps=0.1, seed=2, L=L, edge_cap=(0.004 * L, 0.012 * L))
    _node_parity(p, 4, prec, opts)


# ---------------------------------------------------------------------------------------------
# the multi-GPU Gauss-Seidel exchange on the pipelined kernels (flows-only launch -> all-reduce -> dual update ->
# alpha-only launch; rem:multi_tensor_scheme P:1139-1147)

@pytest.mark.parametrize("opts", [dict(), dict(pexch=0), dict(pexch=1)])
def test_nccl_exchange_path_pipelined_one_rank(opts):
    """The per-step exchange of the commodity-sharded sweep with the pipelined forward split around the all-reduce
    (MODE 4 rank-partial flows of the capacitated arcs, k_dual on the sums, MODE 5 / 6 alpha with the updated W) on a
    one-rank NCCL communicator, fp32 and L >= 256, against the oracle; pexch=0 runs the wide-lane two-pass kernels."""
    import torch
    torch.cuda.nccl.version()
    from paper_2106_14485_b200 import _lib
    p = grid_problem(12, 12, 8, 1019, 0.1, seed=33, cap=(0.3, 1.5))
    assert_parity(p, 4, "fp32", nccl_uid=_lib.mmf_nccl_unique_id(), nranks=1, rank=0, options=opts)


@pytest.mark.parametrize("L,G,marg,opts", [(2040, 2, "point", {}), (1019, 3, "point", dict(pexch=1)), (600, 2, "dense", dict(pexch=1))])
def test_virtual_ranks_pipelined_exchange(L, G, marg, opts):
    """Virtual ranks (mmf_sweep_group) with the default kernels: every shard has L / G >= 256 commodities, so the
    sweep runs the pipelined exchange path (flows-only launches, device-side sum, dual update, alpha-only launches);
    the shards' duals agree, the summed flows equal the unsharded run and the oracle (fp32 tolerance)."""
    from paper_2106_14485_b200 import Solver, _lib
    sc = L / 100 if marg == "point" else 0.2
    p = grid_problem(9, 9, 7, L, 0.1, seed=52, cap=(0.3 * sc, 1.0 * sc), marginals=marg)
    per = (L + G - 1) // G
    bounds = [(min(g * per, L), min((g + 1) * per, L)) for g in range(G)]
    shards = [Solver(p, prec="fp32", l_begin=a, l_count=b - a, options=opts) for a, b in bounds]
    try:
        _lib.mmf_sweep_group([s.ctx for s in shards], 4)
        for s in shards:
            s.sync()
        F = sum(s.edge_flows() for s in shards)
        Ws = [s.cap_duals() for s in shards]
    finally:
        for s in shards:
            s.close()
    for W in Ws[1:]:
        assert np.array_equal(W, Ws[0])
    Fu, Wu, _ = run_gpu(p, 4, "fp32")
    assert max_rel_err(F, Fu, flow_floor(p)) < TOL["fp32"] and max_rel_err(Ws[0], Wu, W_FLOOR) < TOL["fp32"]
    Fo, Wo, _ = run_oracle(p, 4)
    assert max_rel_err(F, Fo, flow_floor(p)) < TOL["fp32"] and max_rel_err(Ws[0], Wo, W_FLOOR) < TOL["fp32"]
    assert np.min(Wo) < 0.99


# ---------------------------------------------------------------------------------------------
# node-tile backward with staged out-halos (option tbwd)

@pytest.mark.parametrize("L,opts", [(1019, dict(tbwd=1)), (1019, dict(tbwd=1, tile=64)), (300, dict(tbwd=1)),
                                    (2051, dict(tbwd=1, tile=16))])
def test_tile_backward_parity(L, opts):
    """The tile backward (BFS node tiles, out-halo rows staged per (tile, chunk) by TMA, consumers from shared
    memory) against the live oracle, with the hub / empty-item graph (high out-degree: arc batches of 32)."""
    assert_parity(_hub_problem(L, 22), 3, "fp32", options=opts)
    p = grid_problem(14, 14, 8, L, 0.1, seed=61, cap=(0.3 * L / 100, 1.2 * L / 100))
    assert_parity(p, 3, "fp32", options=opts)


@pytest.mark.parametrize("L,opts", [(2051, dict(tbwd=1, tfwd=1)), (1019, dict(tbwd=1, tfwd=1)),
                                    (600, dict(tbwd=1, tfwd=1, tile=16))])
def test_tile_forward_parity(L, opts):
    """The node-tile forward (alpha_t and the flow partials of step t per (tile, 128-commodity chunk) from staged in-
    and out-halo rows, fixed-order chunk sum and dual update per step) against the live oracle: a grid with a ragged
    commodity tail, the hub / empty-item graph, and commodity node costs (the layer factor applied before the flows)."""
    p = grid_problem(14, 14, 8, L, 0.1, seed=63, cap=(0.3 * L / 100, 1.2 * L / 100))
    assert_parity(p, 3, "fp32", options=opts)
    assert_parity(_hub_problem(L, 22), 3, "fp32", options=opts)
    assert_parity(_node_cost(p, 0.05, seed=7), 3, "fp32", options=opts)


@pytest.mark.parametrize("case", ["jacobi", "symmetric", "node_costs", "node_caps", "times", "time_varying"])
def test_tile_backward_with_next_rows(case):
    """The tile backward (forced: tbwd=1; the default on high-degree graphs, BJ [3] / [5]) under every NEXT-row feature:
    the Jacobi and symmetric schedules, commodity node costs and node capacities (factors applied after the launch),
    entry / exit times (holding nodes), time-varying costs and capacities — against the oracle."""
    L = 1019
    sc = L / 64
    p = grid_problem(8, 8, 7, L, 0.2, seed=71, cap=(0.3 * L / 100, 1.2 * L / 100))
    opts, okw = dict(tbwd=1), None
    if case == "jacobi":
        opts.update(schedule=1, theta_milli=500)
        okw = dict(schedule="jacobi", theta=0.5)
    elif case == "symmetric":
        opts.update(schedule=2)
        okw = dict(schedule="sym")
    elif case == "node_costs":
        p = _node_cost(p, 0.1, seed=5)
    elif case == "node_caps":
        p = _with_node_caps(grid_problem(8, 8, 7, L, 0.2, seed=52, cap=(5 * sc, 20 * sc)), 3, 0.4 * sc, 1.5 * sc)
        _node_parity(p, 4, "fp32", opts)
        return
    elif case == "times":
        p = _times(p, seed=3, T=10)
    else:
        p = grid_problem(8, 8, 7, L, 0.2, seed=71, cap=(0.3 * L / 100, 1.2 * L / 100), time_varying=True)
    assert_parity(p, 4, "fp32", oracle_kw=okw, options=opts)
