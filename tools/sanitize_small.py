"""Small pipelined-path runs for compute-sanitizer (memcheck / synccheck): grid, L = 1019 and 251, 2 sweeps +
readouts, GS and Jacobi."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_14485_b200 import Solver
from workloads import grid_problem
for L, opts in [(1019, {}), (251, {}), (1019, dict(schedule=1)), (509, dict(bwd=2))]:
    p = grid_problem(6, 6, 4, L, 0.2, seed=44, cap=(0.3, 1.2))
    with Solver(p, prec="fp32", graph=False, options=opts) as s:
        s.sweep(2)
        F = s.edge_flows()
        W = s.cap_duals()
        Fl = s.commodity_flows(1)
        st = s.save_state()
    print(L, opts, "ok", float(F.sum()), flush=True)
