"""Wall-clock breakdown of the end-to-end path bench.py times as `e2e` (upload, init, sweeps, readout), per
C-ABI call.  usage: python tools/e2e_breakdown.py [--config 4] [--sweeps 5]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--sweeps", type=int, default=5)
a = ap.parse_args()

import torch  # noqa: E402
from paper_2106_14485_b200 import _lib as L  # noqa: E402
from workloads import gen  # noqa: E402

p = gen(a.config)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
torch.cuda.synchronize()
T = {}


def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = time.perf_counter() - t0
    return time.perf_counter()


for rep in range(2):  # (the first repetition pays one-time costs: library load, CUDA context, module load)
    T.clear()
    t0 = t_all = time.perf_counter()
    ctx = L.mmf_create(0, L.MMF_FP32 if p.prec == "fp32" else L.MMF_FP64, stream.cuda_stream)
    t0 = tick("create", t0)
    L.mmf_set_graph(ctx, p.N, p.tail, p.head)
    t0 = tick("set_graph", t0)
    L.mmf_set_costs(ctx, p.T, p.eps, p.cost, p.cost.ndim == 2)
    t0 = tick("set_costs", t0)
    L.mmf_set_capacity(ctx, p.cap, p.cap.ndim == 2)
    t0 = tick("set_capacity", t0)
    if p.is_point:
        L.mmf_set_point_marginals(ctx, p.L, 0, p.src, p.dst, p.mass)
    else:
        L.mmf_set_marginals(ctx, p.L, 0, p.mu0, p.muT)
    t0 = tick("set_marginals", t0)
    nbytes = L.mmf_workspace_bytes(ctx)
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    L.mmf_set_workspace(ctx, ws.data_ptr(), nbytes)
    t0 = tick("workspace", t0)
    L.mmf_init(ctx)
    t0 = tick("init (enqueue)", t0)
    L.mmf_sync(ctx)
    t0 = tick("init (device)", t0)
    L.mmf_sweep(ctx, a.sweeps)
    L.mmf_sync(ctx)
    t0 = tick(f"{a.sweeps} sweeps", t0)
    F = L.mmf_read_edge_flows(ctx, p.T, p.A)
    t0 = tick("read_edge_flows", t0)
    W = L.mmf_read_cap_duals(ctx, p.T, p.A)
    t0 = tick("read_cap_duals", t0)
    L.mmf_destroy(ctx)
    del ws
    t0 = tick("destroy", t0)
    total = time.perf_counter() - t_all
    print(f"rep {rep}: total {total:.3f} s  " + "  ".join(f"{k} {v * 1e3:.1f}ms" for k, v in T.items()), flush=True)
