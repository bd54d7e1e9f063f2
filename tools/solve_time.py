"""Time to tolerance through the public API (Solver.solve: on-device error reductions every check_every sweeps)
for the Gauss-Seidel and the Jacobi schedules.  usage: python tools/solve_time.py [--config 4] [--tol 1e-3]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--tol", type=float, default=1e-3)
ap.add_argument("--max-sweeps", type=int, default=300)
ap.add_argument("--check-every", type=int, default=5)
a = ap.parse_args()

import torch  # noqa: E402,F401
from paper_2106_14485_b200 import Solver  # noqa: E402
from workloads import gen  # noqa: E402

p = gen(a.config)
out = {"config": a.config, "workload": p.name, "tol": a.tol, "check_every": a.check_every, "runs": {}}
for name, opts in [("gs", {}), ("jacobi_theta1", dict(schedule=1, theta_milli=1000))]:
    with Solver(p, prec=p.prec, options=opts) as s:
        s.sync()
        t0 = time.perf_counter()
        r = s.solve(a.tol, a.max_sweeps, a.check_every)
        dt = time.perf_counter() - t0
    out["runs"][name] = {"converged": r["converged"], "sweeps": r["sweeps"], "err": r["err"], "seconds": dt,
                         "history": [float(x) for x in r["history"]]}
    print(f"{name}: converged {r['converged']} sweeps {r['sweeps']} err {r['err']:.3e} in {dt:.2f} s",
          file=sys.stderr, flush=True)
print(json.dumps(out))
