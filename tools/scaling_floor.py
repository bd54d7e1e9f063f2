"""Predicted strong-scaling floor of the commodity-sharded Gauss-Seidel sweep:
on ONE GPU, a rank's share L/G of [4] through the multi-GPU exchange path (one-rank NCCL communicator: partial flows ->
ncclAllReduce -> dual update per step, the same kernels and calls as G ranks make), for G = 1, 2, 4, 8, next to the
single-GPU path.  The G-GPU sweep cannot be faster than this per-rank time (+ the cross-GPU all-reduce latency, which a
one-rank communicator does not pay).   usage: python tools/scaling_floor.py [--config 4|5] > out.json"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

torch.cuda.nccl.version()
from paper_2106_14485_b200 import Solver, _lib  # noqa: E402
from workloads import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--sweeps", type=int, default=5)
ap.add_argument("--out", default=None, help="write the JSON here (NCCL prints its banner on stdout)")
a = ap.parse_args()
p = gen(a.config)
out = {"workload": p.name, "L": p.L, "rows": []}
for G in (1, 2, 4, 8):
    per = p.L // G
    for name, kw in [("single_path", {}), ("exchange_path", dict(nccl_uid=_lib.mmf_nccl_unique_id(), nranks=1, rank=0))]:
        with Solver(p, prec="fp32", l_begin=0, l_count=per, **kw) as s:
            s.sweep(2)
            s.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.sweep(a.sweeps)
            e1.record()
            s.sync()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.sweeps
        row = {"G": G, "L_rank": per, "path": name, "ms_per_sweep": ms}
        out["rows"].append(row)
        print(row, file=sys.stderr, flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f)
else:
    print(json.dumps(out))
