"""BASELINE.json configs [1]-[5] plus micro / lite variants, as seeded arrays.

Conventions fixed here (SURVEY.md §8(c) ambiguity table, also listed in DESIGN.md §3):

* Q1  node form: arcs ``A = E ∪ {(i→i)}``; user arc order is the moving arcs (both directions of
      each undirected edge, in generation order) followed by one self-loop ("stay" arc) per node.
* Q2  ``T`` transitions, layers ``0..T``.
* Q4  self-loops are uncapacitated (cap = +inf) in every config.
* Q12 [3],[5]: self-loop cost 0, arcs cost length / mean undirected length; [4]: grid edge 1.0,
      highway 0.3, stay 0.1.
* Q13 independent draw per *directed* arc for costs and capacities.
* Q14 [2]: per commodity and per end 3 Gaussian bumps, centres U[0,59]^2, sigma U[2,6], equal
      weights, normalised to mass 1.
* Q15/Q16 point-mass OD pairs: distinct s != g in the largest connected component with
      1 <= hop(s, g) <= T; unit mass ([1],[3],[4]) or 1/L ([5]).
* Q17 [4]: delete round(10%) of the 79,600 undirected grid edges, then add round(5% x remaining)
      undirected highways between distinct random nodes that are not already adjacent.
* Q18 [5]: cap = U[0.5, 2] * 100 / L on moving arcs.

Random streams: ``numpy.random.default_rng(SeedSequence(seed).spawn(4))`` for
``[graph, costs, caps, commodities]``; ``seed`` defaults to the config index.
Nothing here computes kernels, logs or any step of the Sinkhorn method.
"""
from __future__ import annotations

import dataclasses
from functools import lru_cache
from typing import Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csg
from scipy.spatial import cKDTree

CONFIG_NAMES = {1: "tiny-grid5x5", 2: "grid60x60", 3: "rgg20k-k6", 4: "road200x200", 5: "rgg5k-k8-many"}


@dataclasses.dataclass
class Problem:
    """One dynamic multi-commodity flow instance in node form.

    tail/head: int32 [A] arcs (user order), self-loops included.
    cost: float64 [A] (time-invariant) or [T, A] per-step arc cost C_t[a].
    cap:  float64 [A] or [T, A]; +inf = uncapacitated, 0 = closed.
    Marginals: either point masses (src, dst, mass: [L]) or dense mu0/muT [L, N].
    """
    name: str
    N: int
    tail: np.ndarray
    head: np.ndarray
    T: int
    eps: float
    cost: np.ndarray
    cap: np.ndarray
    L: int
    src: Optional[np.ndarray] = None
    dst: Optional[np.ndarray] = None
    mass: Optional[np.ndarray] = None
    mu0_dense: Optional[np.ndarray] = None
    muT_dense: Optional[np.ndarray] = None
    prec: str = "fp64"
    sweeps: int = 10
    coords: Optional[np.ndarray] = None
    meta: dict = dataclasses.field(default_factory=dict)
    # commodity-dependent node costs c[l, j] (finite), charged to commodity l for every
    # intermediate layer t = 1..T-1 it spends at node j (reading R-N); None = commodity-independent costs
    node_cost: Optional[np.ndarray] = None
    # per-commodity entry / exit layers 0 <= t_in[l] < t_out[l] <= T (rem:multi_tensor_scheme
    # P:1139-1149); None = 0 / T
    t_in: Optional[np.ndarray] = None
    t_out: Optional[np.ndarray] = None
    # node (state) capacities d_t[j] on the node marginal at the intermediate layers ([N] or
    # [T+1, N]; +inf free, 0 closed; layers 0 and T ignored): the paper's P_t(M) <= d_t of eq:multicommodity
    node_cap: Optional[np.ndarray] = None

    @property
    def A(self) -> int:
        return int(self.tail.shape[0])

    @property
    def is_point(self) -> bool:
        return self.src is not None

    @property
    def time_varying(self) -> bool:
        return self.cost.ndim == 2

    @property
    def n_loops(self) -> int:
        return int(np.count_nonzero(self.tail == self.head))

    @property
    def mu0(self) -> np.ndarray:
        """Dense source distribution [L, N] (built on demand from point masses)."""
        if self.mu0_dense is not None:
            return self.mu0_dense
        m = np.zeros((self.L, self.N))
        m[np.arange(self.L), self.src] = self.mass
        return m

    @property
    def muT(self) -> np.ndarray:
        if self.muT_dense is not None:
            return self.muT_dense
        m = np.zeros((self.L, self.N))
        m[np.arange(self.L), self.dst] = self.mass
        return m

    def cost_t(self, t: int) -> np.ndarray:
        return self.cost[t] if self.cost.ndim == 2 else self.cost

    def cap_t(self, t: int) -> np.ndarray:
        return self.cap[t] if self.cap.ndim == 2 else self.cap

    def updates_per_sweep(self) -> int:
        """Metric unit: L * |A| * T commodity-arc-timestep updates (loops included)."""
        return int(self.L) * self.A * int(self.T)

    def commodity_slice(self, l0: int, l1: int) -> "Problem":
        """Sub-problem with commodities [l0, l1) (same graph, costs, caps)."""
        kw = dataclasses.asdict(self)
        kw.update(L=l1 - l0, name=f"{self.name}[{l0}:{l1}]")
        for k in ("src", "dst", "mass", "mu0_dense", "muT_dense", "node_cost", "t_in", "t_out"):
            v = getattr(self, k)
            kw[k] = None if v is None else v[l0:l1].copy()
        return Problem(**kw)


# ----------------------------------------------------------------------------------------------
# graph helpers (pure combinatorics)

def _grid_undirected(rows: int, cols: int) -> np.ndarray:
    """4-neighbour grid, node id r*cols+c; undirected edges (u<v) in row-major order (right, down)."""
    edges = []
    for r in range(rows):
        for c in range(cols):
            u = r * cols + c
            if c + 1 < cols:
                edges.append((u, u + 1))
            if r + 1 < rows:
                edges.append((u, u + cols))
    return np.asarray(edges, dtype=np.int64).reshape(-1, 2)


def _directed_with_loops(N: int, und: np.ndarray):
    """Both directions of every undirected edge (u->v then v->u), then one self-loop per node."""
    tail = np.concatenate([np.stack([und[:, 0], und[:, 1]], 1).reshape(-1), np.arange(N)])
    head = np.concatenate([np.stack([und[:, 1], und[:, 0]], 1).reshape(-1), np.arange(N)])
    return tail.astype(np.int32), head.astype(np.int32)


def _knn_undirected(xy: np.ndarray, k: int) -> np.ndarray:
    """Symmetrised k-nearest-neighbour graph: {i,j} if j in kNN(i) or i in kNN(j)."""
    tree = cKDTree(xy)
    _, idx = tree.query(xy, k=k + 1)
    i = np.repeat(np.arange(xy.shape[0]), k)
    j = idx[:, 1:].reshape(-1)
    u = np.minimum(i, j)
    v = np.maximum(i, j)
    key = np.unique(u.astype(np.int64) * xy.shape[0] + v)
    return np.stack([key // xy.shape[0], key % xy.shape[0]], 1)


def _adjacency(N: int, und: np.ndarray):
    a = sp.coo_matrix((np.ones(len(und) * 2), (np.r_[und[:, 0], und[:, 1]], np.r_[und[:, 1], und[:, 0]])),
                      shape=(N, N)).tocsr()
    return a


def _largest_component(N: int, und: np.ndarray) -> np.ndarray:
    _, lab = csg.connected_components(_adjacency(N, und), directed=False)
    big = np.argmax(np.bincount(lab))
    return np.flatnonzero(lab == big)


def _sample_od(rng: np.random.Generator, N: int, und: np.ndarray, L: int, T: int) -> tuple:
    """Q16: L distinct-endpoint OD pairs in the largest component with 1 <= hop(s,g) <= T (rejection)."""
    comp = _largest_component(N, und)
    adj = _adjacency(N, und)
    src, dst = [], []
    while len(src) < L:
        batch = 256          # fixed draw size: the OD list of a smaller L is a prefix of a larger one
        s = comp[rng.integers(0, comp.size, size=batch)]
        g = comp[rng.integers(0, comp.size, size=batch)]
        uniq, inv = np.unique(s, return_inverse=True)
        dist = csg.shortest_path(adj, method="D", unweighted=True, indices=uniq)
        hop = dist[inv, g]
        for k in range(batch):
            if len(src) == L:
                break
            if s[k] != g[k] and 1 <= hop[k] <= T:
                src.append(int(s[k]))
                dst.append(int(g[k]))
    return np.asarray(src, np.int32), np.asarray(dst, np.int32)


def _streams(seed: int):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(4)]


# ----------------------------------------------------------------------------------------------
# configs

def _cfg1(seed, L=None, T=None):
    """[1] Tiny: 5x5 grid, T=10, L=3, move 1.0 / stay 0.1, eps 0.1, cap 0.5, unit point masses, fp64."""
    T = T or 10
    L = L or 3
    g_rng, c_rng, k_rng, m_rng = _streams(seed)
    und = _grid_undirected(5, 5)
    N = 25
    tail, head = _directed_with_loops(N, und)
    loop = tail == head
    cost = np.where(loop, 0.1, 1.0)
    cap = np.where(loop, np.inf, 0.5)
    src, dst = _sample_od(m_rng, N, und, L, T)
    return Problem("tiny-grid5x5", N, tail, head, T, 0.1, cost, cap, L, src=src, dst=dst,
                   mass=np.ones(L), prec="fp64", sweeps=200, meta={"readings": "Q2 Q4 Q15 Q16"})


def _bumps(rng, L, rows, cols):
    r, c = np.divmod(np.arange(rows * cols), cols)
    out = np.zeros((L, rows * cols))
    for l in range(L):
        for _ in range(3):
            cy, cx = rng.uniform(0, rows - 1), rng.uniform(0, cols - 1)
            sig = rng.uniform(2.0, 6.0)
            out[l] += np.exp(-((r - cy) ** 2 + (c - cx) ** 2) / (2 * sig * sig))
        out[l] /= out[l].sum()
    return out


def _cfg2(seed, L=None, T=None, prec="fp64"):
    """[2] 60x60 grid, T=60, L=32, move U[0.5,1.5], stay 0.05, eps 0.05, caps U[0.1,0.6], Gaussian bumps."""
    T = T or 60
    L = L or 32
    g_rng, c_rng, k_rng, m_rng = _streams(seed)
    und = _grid_undirected(60, 60)
    N = 3600
    tail, head = _directed_with_loops(N, und)
    loop = tail == head
    nm = int((~loop).sum())
    cost = np.full(tail.shape, 0.05)
    cost[~loop] = c_rng.uniform(0.5, 1.5, size=nm)
    cap = np.full(tail.shape, np.inf)
    cap[~loop] = k_rng.uniform(0.1, 0.6, size=nm)
    mu0 = _bumps(m_rng, L, 60, 60)
    muT = _bumps(m_rng, L, 60, 60)
    return Problem("grid60x60", N, tail, head, T, 0.05, cost, cap, L, mu0_dense=mu0, muT_dense=muT,
                   prec=prec, sweeps=100, meta={"readings": "Q2 Q4 Q13 Q14"})


def _rgg(seed, N, k, T, L, eps, cap_lo, cap_hi, cap_scale, mass_each, name, sweeps):
    g_rng, c_rng, k_rng, m_rng = _streams(seed)
    xy = g_rng.uniform(0.0, 1.0, size=(N, 2))
    und = _knn_undirected(xy, k)
    tail, head = _directed_with_loops(N, und)
    loop = tail == head
    length = np.linalg.norm(xy[und[:, 0]] - xy[und[:, 1]], axis=1)
    mean_len = length.mean()
    cost = np.zeros(tail.shape)
    cost[~loop] = np.repeat(length / mean_len, 2)
    nm = int((~loop).sum())
    cap = np.full(tail.shape, np.inf)
    cap[~loop] = k_rng.uniform(cap_lo, cap_hi, size=nm) * cap_scale
    src, dst = _sample_od(m_rng, N, und, L, T)
    return Problem(name, N, tail, head, T, eps, cost, cap, L, src=src, dst=dst,
                   mass=np.full(L, mass_each), prec="fp32", sweeps=sweeps, coords=xy,
                   meta={"readings": "Q2 Q4 Q12 Q13 Q15 Q16", "k": k})


def _cfg3(seed, L=None, T=None):
    """[3] RGG N=20000, kNN k=6 symmetric, cost len/mean, T=100, L=256 point OD, eps 0.02, caps U[0.05,0.3]."""
    return _rgg(seed, 20000, 6, T or 100, L or 256, 0.02, 0.05, 0.3, 1.0, 1.0, "rgg20k-k6", 10)


def _cfg4(seed, L=None, T=None):
    """[4] 200x200 grid -10% edges +5% highways (cost 0.3), grid 1.0, stay 0.1, T=200, L=1024, eps 0.01."""
    T = T or 200
    L = L or 1024
    g_rng, c_rng, k_rng, m_rng = _streams(seed)
    rows = cols = 200
    N = rows * cols
    und = _grid_undirected(rows, cols)
    n_del = int(round(0.10 * len(und)))
    keep = np.ones(len(und), bool)
    keep[g_rng.choice(len(und), size=n_del, replace=False)] = False
    und = und[keep]
    n_hw = int(round(0.05 * len(und)))
    existing = set((und[:, 0].astype(np.int64) * N + und[:, 1]).tolist())
    hw = []
    while len(hw) < n_hw:
        u, v = (int(x) for x in g_rng.integers(0, N, size=2))
        if u == v:
            continue
        a, b = min(u, v), max(u, v)
        key = a * N + b
        if key in existing:
            continue
        existing.add(key)
        hw.append((a, b))
    hw = np.asarray(hw, np.int64)
    und_all = np.concatenate([und, hw])
    tail, head = _directed_with_loops(N, und_all)
    loop = tail == head
    n_grid_dir = 2 * len(und)
    cost = np.full(tail.shape, 0.1)
    cost[:n_grid_dir] = 1.0
    cost[n_grid_dir:n_grid_dir + 2 * len(hw)] = 0.3
    nm = int((~loop).sum())
    cap = np.full(tail.shape, np.inf)
    cap[~loop] = k_rng.uniform(0.02, 0.2, size=nm)
    src, dst = _sample_od(m_rng, N, und_all, L, T)
    return Problem("road200x200", N, tail, head, T, 0.01, cost, cap, L, src=src, dst=dst,
                   mass=np.ones(L), prec="fp32", sweeps=3,
                   meta={"readings": "Q2 Q4 Q12 Q13 Q15 Q16 Q17", "highways": int(len(hw))})


def _cfg5(seed, L=None, T=None):
    """[5] RGG N=5000 k=8, T=100, L=8192 point OD of mass 1/L, caps U[0.5,2]*100/L, eps 0.01."""
    L = L or 8192
    return _rgg(seed, 5000, 8, T or 100, L, 0.01, 0.5, 2.0, 100.0 / L, 1.0 / L, "rgg5k-k8-many", 3)


_CFGS = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}


@lru_cache(maxsize=8)
def _gen_cached(config: int, seed: int, L, T, prec):
    kw = {"L": L, "T": T}
    if config == 2 and prec is not None:
        kw["prec"] = prec
    p = _CFGS[config](seed, **kw)
    if prec is not None:
        p.prec = prec
    return p


def gen(config: int, seed: Optional[int] = None, L: Optional[int] = None, T: Optional[int] = None,
        prec: Optional[str] = None) -> Problem:
    """Problem for BASELINE.json config ``config`` (1-based).  ``L``/``T`` override gives the
    "lite" variants (same graph and draws; the OD list is a prefix of the full one for fixed T)."""
    if config not in _CFGS:
        raise ValueError(f"unknown config {config}")
    p = _gen_cached(config, config if seed is None else seed, L, T, prec)
    return dataclasses.replace(p)


# ----------------------------------------------------------------------------------------------
# micro / special instances for pins

def grid_problem(rows: int, cols: int, T: int, L: int, eps: float, seed: int = 0, *,
                 move_cost=(0.5, 1.5), stay_cost=0.1, cap=(0.2, 0.8), loop_cap=np.inf,
                 marginals: str = "point", time_varying: bool = False, closed_arcs: int = 0,
                 mass=None, prec: str = "fp64") -> Problem:
    """Small grid with self-loops and random per-arc costs/caps (micro instances for brute force).

    move_cost / cap: (lo, hi) uniform ranges or scalars; cap=None -> uncapacitated moving arcs.
    marginals: "point" (random s != g, unit or given mass) or "dense" (random positive, mass 1 per
    commodity, some zero entries).  time_varying draws an independent [T, A] cost/cap per step.
    closed_arcs: number of moving arcs whose capacity is set to 0 (d = 0 closes the arc).
    """
    g_rng, c_rng, k_rng, m_rng = _streams(seed)
    und = _grid_undirected(rows, cols)
    N = rows * cols
    tail, head = _directed_with_loops(N, und)
    loop = tail == head
    A = tail.size
    shape = (T, A) if time_varying else (A,)

    def draw(rng, spec, n):
        if spec is None:
            return np.full(n, np.inf)
        if np.isscalar(spec):
            return np.full(n, float(spec))
        return rng.uniform(spec[0], spec[1], size=n)

    cost = np.empty(shape)
    capa = np.empty(shape)
    for idx in (range(T) if time_varying else [None]):
        c = np.empty(A)
        c[~loop] = draw(c_rng, move_cost, int((~loop).sum()))
        c[loop] = stay_cost
        k = np.empty(A)
        k[~loop] = draw(k_rng, cap, int((~loop).sum()))
        k[loop] = loop_cap
        if closed_arcs:
            k[g_rng.choice(np.flatnonzero(~loop), size=closed_arcs, replace=False)] = 0.0
        if idx is None:
            cost[:] = c
            capa[:] = k
        else:
            cost[idx] = c
            capa[idx] = k
    name = f"grid{rows}x{cols}-T{T}-L{L}-s{seed}"
    if marginals == "point":
        src, dst = _sample_od(m_rng, N, und, L, T)
        ms = np.ones(L) if mass is None else np.asarray(mass, float)
        return Problem(name, N, tail, head, T, eps, cost, capa, L, src=src, dst=dst, mass=ms, prec=prec,
                       sweeps=10)
    mu0 = m_rng.uniform(0.0, 1.0, size=(L, N))
    muT = m_rng.uniform(0.0, 1.0, size=(L, N))
    mu0[mu0 < 0.15] = 0.0
    muT[muT < 0.15] = 0.0
    ms = np.ones(L) if mass is None else np.asarray(mass, float)
    mu0 *= (ms / mu0.sum(1))[:, None]
    muT *= (ms / muT.sum(1))[:, None]
    return Problem(name, N, tail, head, T, eps, cost, capa, L, mu0_dense=mu0, muT_dense=muT, prec=prec,
                   sweeps=10)


def fig1_problem(T: int = 3) -> Problem:
    """The 3-node, 4-edge network of PAPER.md Fig. time_exp, edges read off the TikZ:
    1->2, 2->3, 3->1, 3->2 (0-based: 0->1, 1->2, 2->0, 2->1); no self-loops, unit costs, no caps."""
    tail = np.array([0, 1, 2, 2], np.int32)
    head = np.array([1, 2, 0, 1], np.int32)
    return Problem("fig1", 3, tail, head, T, 1.0, np.ones(4), np.full(4, np.inf), 1,
                   src=np.array([0], np.int32), dst=np.array([1], np.int32), mass=np.ones(1))
