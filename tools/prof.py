"""Profiling driver: build a Solver for a config and run a few sweeps with plain stream launches
(no CUDA graph) so that ncu / nsys see every kernel.  Usage:
    python tools/prof.py --config 4 --sweeps 2 [--L 64] [--opt tile=32 --opt cpt=2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--L", type=int, default=None)
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--graph", type=int, default=0)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--time", action="store_true")
a = ap.parse_args()

import torch  # noqa: E402
from paper_2106_14485_b200 import Solver  # noqa: E402
from workloads import gen  # noqa: E402

p = gen(a.config, L=a.L)
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
s = Solver(p, graph=bool(a.graph), options=opts, profile=a.time)
def sync():
    try:
        s.sync()
    except Exception as e:  # diagnostics runs (e.g. dry=1) leave meaningless messages behind
        print("sync:", str(e)[:80])


s.sweep(1)
sync()
t0 = time.perf_counter()
s.sweep(a.sweeps)
sync()
dt = time.perf_counter() - t0
print(f"{p.name} L={p.L} opts={opts}: {dt / a.sweeps * 1e3:.2f} ms/sweep (wall, incl. launch)")
if a.time:
    ks = s.kernel_stats()
    print({k: round(v["ms"] / (a.sweeps + 1), 3) for k, v in ks.items() if v["launches"]})
s.close()
