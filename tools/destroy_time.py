"""Time of mmf_destroy after a solve-like sequence (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_14485_b200 import Solver
from workloads import gen
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = gen(c)
for opts in [{}, dict(kernels=3), dict(graph=0)]:
    o = dict(opts)
    graph = bool(o.pop("graph", 1))
    s = Solver(p, prec="fp32", graph=graph, options=o)
    s.sweep(2); s.sync()
    F = s.edge_flows(); W = s.cap_duals()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s.close(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(opts, f"destroy {1e3 * (t1 - t0):.1f} ms", flush=True)
