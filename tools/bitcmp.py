"""Bitwise fingerprint of a library build's results: edge flows, capacity duals and stats after a few sweeps.
usage: MMF_LIB=paper_2106_14485_b200/libmmf_X.so python tools/bitcmp.py --config 5 --sweeps 2"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--L", type=int, default=None)
ap.add_argument("--sweeps", type=int, default=2)
a = ap.parse_args()
import numpy as np  # noqa: E402
from paper_2106_14485_b200 import Solver  # noqa: E402
from workloads import gen  # noqa: E402

p = gen(a.config, L=a.L)
s = Solver(p)
s.sweep(a.sweeps)
s.sync()
F = np.ascontiguousarray(s.edge_flows())
W = np.ascontiguousarray(s.cap_duals())
h = lambda x: hashlib.sha1(x.tobytes()).hexdigest()[:12]
print(f"cfg{a.config} {os.environ.get('MMF_LIB', 'base')}: F {h(F)} W {h(W)} sumF {F.sum():.9e}")
s.close()
