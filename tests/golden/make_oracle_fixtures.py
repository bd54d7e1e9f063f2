"""Write sampled float64-oracle outputs for the configs too slow to run live in the GPU tests.

Calls only oracle/ (and the seeded generators in workloads/): every stored value is the oracle's.
Usage:  python tests/golden/make_oracle_fixtures.py <name> [...]   (names: see JOBS)
Each fixture holds, for each snapshot sweep count k: 20,000 uniformly sampled flat (t, a) indices of
the [T, A] outputs with the oracle's F_t[a] and W_t[a] there, and the end-of-sweep statistics.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle_init, oracle_sweep, readout_flows, stats  # noqa: E402
from workloads import gen  # noqa: E402

# name: (config, overrides, snapshot sweep counts)   -- SURVEY §8(c) Q21 sweep counts, "lite" L
JOBS = {
    "cfg3": (3, {}, [3, 10]),
    "cfg4lite": (4, {"L": 16}, [3, 20]),
    "cfg5lite": (5, {"L": 64}, [3, 20]),
    "cfg2": (2, {}, [100]),
    # the full [5] graph with L >= 256 (the pipelined kernels' slice widths), short horizon
    "cfg5pipe": (5, {"L": 512, "T": 6}, [3]),
}
NSAMPLE = 20000


def run(name):
    cfg, kw, snaps = JOBS[name]
    p = gen(cfg, **kw)
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(p.T * p.A, size=min(NSAMPLE, p.T * p.A), replace=False))
    out = {"config": cfg, "L": p.L, "T": p.T, "A": p.A, "N": p.N, "idx": idx, "snaps": np.array(snaps)}
    t0 = time.time()
    st = oracle_init(p)
    for k in range(1, max(snaps) + 1):
        oracle_sweep(st)
        print(f"{name}: sweep {k} at {time.time() - t0:.0f}s", flush=True)
        if k in snaps:
            F, W = readout_flows(st)
            s = stats(st)
            out[f"F_{k}"] = F.reshape(-1)[idx]
            out[f"W_{k}"] = W.reshape(-1)[idx]
            for key in ("mass", "primal", "dual", "src_mismatch", "sink_mismatch", "cap_violation"):
                out[f"{key}_{k}"] = s[key]
            np.savez_compressed(os.path.join(os.path.dirname(__file__), f"oracle_{name}.npz"), **out)
    print(f"{name}: done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    for n in sys.argv[1:]:
        run(n)
