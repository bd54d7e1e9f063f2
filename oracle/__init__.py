"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct float64 CPU transcription of the paper's multi-commodity Sinkhorn
scheme (Haasler, Ringh, Chen, Karlsson, arXiv:2106.14485, Algorithm 2 ``alg:multi_commodity``,
PAPER.md P:1085-1107) in the node form of SURVEY.md §8.0, plus the independent pins that check it
(brute-force tensors, closed forms, an exact LP, extended-precision twins).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import or execute anything in this package.  It shares no code with the CUDA
library (``paper_2106_14485_b200``) and never imports it; the only thing both sides share is the
seeded input generator ``workloads`` (which holds none of the method's arithmetic).

Parity status per function is listed in DESIGN.md §4; every function here is pinned by at least
one ``-m "not gpu"`` test in ``tests/test_oracle_pins.py``.
"""
from .sweep import (OracleState, OracleInfeasible, oracle_init, oracle_sweep, oracle_run, readout_flows,  # noqa: F401
                    readout_commodity_flows, dual_objective, stats, oracle_sweep_jacobi, damped_update,
                    solve_error, oracle_solve, oracle_sweep_symmetric)
