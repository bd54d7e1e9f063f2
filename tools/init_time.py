"""Host-side setup time of a Solver (diagnostic): python tools/init_time.py CONFIG [key=value ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_14485_b200 import Solver
from workloads import gen
c = int(sys.argv[1])
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[2:]}
p = gen(c)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(p, prec="fp32", options=opts)
    s.sync()
    t1 = time.perf_counter()
    s.close()
    print(c, opts, f"init {1e3 * (t1 - t0):.1f} ms", flush=True)
