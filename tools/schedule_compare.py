"""Convergence per sweep and per byte of the Gauss-Seidel schedule (Algorithm 2), the damped Jacobi schedule and the
symmetric Gauss-Seidel schedule on one config: after every sweep the end-of-sweep statistics
(mmf_read_stats: source-marginal L1 mismatch, worst capacity violation, dual objective), the measured sweep time and
the algorithmic bytes of the sweep (mmf_sweep_bytes; symmetric GS adds one flow pass per step: 3 N L B_e + 2 |A| B_w).

usage: python tools/schedule_compare.py [--config 4] [--sweeps 30] [--thetas 500,1000] > out.json"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--sweeps", type=int, default=30)
ap.add_argument("--thetas", default="500,1000")
a = ap.parse_args()

import torch  # noqa: E402,F401
from paper_2106_14485_b200 import Solver  # noqa: E402
from workloads import gen  # noqa: E402

p = gen(a.config)
mass = float(p.mass.sum()) if p.is_point else float(p.mu0.sum())
runs = [("gs", dict())] + [(f"jacobi_theta{int(th) / 1000:g}", dict(schedule=1, theta_milli=int(th)))
                          for th in a.thetas.split(",")] + [("symmetric_gs", dict(schedule=2))]
out = {"config": a.config, "workload": p.name, "sweeps": a.sweeps, "mass": mass, "runs": {}}
for name, opts in runs:
    rows = []
    with Solver(p, prec=p.prec, options=opts) as s:
        bsweep, _ = s.sweep_bytes()
        if opts.get("schedule") == 2:
            Be = 6.0 if p.prec == "fp32" else 12.0
            bsweep += p.T * (3 * p.N * p.L * Be + 2 * p.A * (Be - 2 + 4))
        for k in range(1, a.sweeps + 1):
            t0 = time.perf_counter()
            s.sweep(1)
            s.sync()
            dt = time.perf_counter() - t0
            st = s.stats()
            rows.append({"sweep": k, "src_mismatch_rel": st["src_mismatch"] / mass,
                         "cap_violation": st["cap_violation"], "dual": st["dual"], "sweep_s": dt,
                         "bytes": bsweep * k})
    out["runs"][name] = rows
    last = rows[-1]
    print(f"{name}: after {a.sweeps} sweeps src_mismatch/mass {last['src_mismatch_rel']:.3e} "
          f"cap_violation {last['cap_violation']:.3e} dual {last['dual']:.6e}", file=sys.stderr, flush=True)
print(json.dumps(out))
