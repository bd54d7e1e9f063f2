"""ORACLE (test infrastructure only): commodity sharding of the float64 oracle.

Given W, the L commodity chains are independent; the commodities couple only through the aggregate
flow sum in the capacity-dual update (rem:multi_tensor_scheme).  A shard runs
``oracle_sweep`` on its commodity slice with ``reduce_lse`` combining the per-arc log flow sums of all
shards (``combine_lse``); the end-of-sweep statistics are combined from per-shard pieces
(``combine_stats``).  Transport between shards (gloo, files) is the caller's.  Pinned against the
unsharded oracle by tests/test_sharding.py.
"""
from __future__ import annotations

import numpy as np

from .sweep import OracleState, readout_flows, dual_terms


def combine_lse(parts: np.ndarray) -> np.ndarray:
    """log sum_g exp(parts[g, a]) over shards g (max-shifted); an all -inf column stays -inf."""
    parts = np.asarray(parts, np.float64)
    mx = parts.max(axis=0)
    shift = np.where(np.isfinite(mx), mx, 0.0)
    with np.errstate(divide="ignore"):
        return shift + np.log(np.exp(parts - shift[None, :]).sum(axis=0))


def shard_pieces(st: OracleState) -> dict:
    """This shard's additive contributions to the end-of-sweep statistics:
    its edge flows, tensor mass, marginal L1 mismatches and the dual's commodity terms."""
    p = st.problem
    assert st.t_in is None and st.t_out is None, "sharded fixtures: no commodity times"
    F, _ = readout_flows(st)
    PT = np.exp(st.a[p.T] + st.lamT)          # (both stores hold a_T after a pass)
    P0 = np.exp(st.lam0 + st.b[0])
    s0, sT, sd = dual_terms(st)
    return {"F": F, "mass": float(PT.sum()), "src_mismatch": float(np.abs(P0 - p.mu0).sum()),
            "sink_mismatch": float(np.abs(PT - p.muT).sum()), "s0": float(s0), "sT": float(sT), "sd": float(sd)}


def combine_stats(problem, pieces: list, omega: np.ndarray, sweeps: int) -> dict:
    """stats() of the unsharded state from the shards' pieces (in shard order): F and the commodity
    sums add over shards; the capacity term sum d*omega is common (W is shared)."""
    p = problem
    F = pieces[0]["F"].copy()
    for q in pieces[1:]:
        F += q["F"]
    mass = sum(q["mass"] for q in pieces)
    cost = np.broadcast_to(p.cost, F.shape)
    cap = np.broadcast_to(p.cap, F.shape)
    s0 = sum(q["s0"] for q in pieces)
    sT = sum(q["sT"] for q in pieces)
    sd = pieces[0]["sd"]
    return {
        "F": F, "W": np.exp(omega),
        "mass": mass,
        "primal": float((cost * F).sum()),
        "dual": float(p.eps * (-mass + s0 + sT + sd)),
        "src_mismatch": sum(q["src_mismatch"] for q in pieces),
        "sink_mismatch": sum(q["sink_mismatch"] for q in pieces),
        "cap_violation": float(np.maximum(F - cap, 0.0)[np.isfinite(cap)].max(initial=0.0)),
        "cap_excess": float(np.maximum(F - cap, 0.0)[np.isfinite(cap)].sum()),
        "sweeps": sweeps,
        # magnitude of the dual's terms (the tolerance scale of a comparison of the dual: a sum of large terms of both
        # signs): eps (mass + sum over shards of |s0| + |sT| + |sd|)
        "dual_scale": float(p.eps * (mass + sum(abs(q["s0"]) + abs(q["sT"]) for q in pieces) + abs(sd))),
    }
