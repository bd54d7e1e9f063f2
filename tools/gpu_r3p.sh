#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "nccl or jacobi" 2>&1 | tail -3
cat > /tmp/ct.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2106_14485_b200 import Solver, _lib
from workloads import gen
p = gen(4)
for name, kw in [("jacobi single", {}), ("jacobi nccl1", dict(nccl_uid=_lib.mmf_nccl_unique_id(), nranks=1, rank=0))]:
    with Solver(p, prec="fp32", profile=True, options=dict(schedule=1, theta_milli=1000), **kw) as s:
        s.sweep(1); s.sync()
        t0 = time.perf_counter(); s.sweep(3); s.sync(); dt = (time.perf_counter() - t0) / 3
        print(name, f"{dt*1e3:.1f} ms/sweep", {k: round(v['ms'] / 4, 2) for k, v in s.kernel_stats().items() if v['launches']}, flush=True)
PY
timeout 600 python /tmp/ct.py
