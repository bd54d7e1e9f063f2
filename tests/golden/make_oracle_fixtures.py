"""Write sampled float64-oracle outputs for the configs too slow to run live in the GPU tests.

Calls only oracle/ (and the seeded generators in workloads/): every stored value is the oracle's.
Usage:  python tests/golden/make_oracle_fixtures.py [--shards G] <name> [...]   (names: see JOBS)

Each fixture holds, for each snapshot sweep count k: NSAMPLE uniformly sampled flat (t, a) indices of
the [T, A] outputs with the oracle's F_t[a] and W_t[a] there, full rows F_t, W_t at a few steps
(``rows``), and the end-of-sweep statistics.

--shards G (G > 1) runs the oracle commodity-sharded over G local processes (gloo on 127.0.0.1), each
with its slice of the commodities, the per-step flow sums combined by oracle.shard.combine_lse (the
coupling of rem:multi_tensor_scheme P:1139-1147; equal to the unsharded oracle to rounding,
tests/test_sharding.py).  Full-size [4] / [5] keep the backward messages in an np.memmap under
.scratch/ and only two forward layers in memory (oracle_init's storage options; bitwise equal to the
in-memory oracle, tests/test_oracle_pins.py::test_storage_options_bitwise_equal).
"""
import argparse
import os
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle_init, oracle_sweep, readout_flows, stats  # noqa: E402
from oracle.sweep import dual_terms  # noqa: E402
from workloads import gen  # noqa: E402

# name: (config, overrides, snapshot sweep counts)   -- SURVEY §8(c) Q21 sweep counts, "lite" L
JOBS = {
    "cfg3": (3, {}, [3, 10]),
    "cfg4": (4, {}, [3]),
    "cfg5": (5, {}, [3]),
    "cfg4lite": (4, {"L": 16}, [3, 20]),
    "cfg5lite": (5, {"L": 64}, [3, 20]),
    "cfg2": (2, {}, [100]),
    # the full [5] graph with L >= 256 (the pipelined kernels' slice widths), short horizon
    "cfg5pipe": (5, {"L": 512, "T": 6}, [3]),
}
NSAMPLE = 20000
NSAMPLE_FULL = 100000
STAT_KEYS = ("mass", "primal", "dual", "src_mismatch", "sink_mismatch", "cap_violation", "cap_excess", "dual_scale")
SCRATCH = os.path.join(ROOT, ".scratch")
BIG = ("cfg4", "cfg5")


def _sample(p, name):
    rng = np.random.default_rng(12345)
    n = NSAMPLE_FULL if name in BIG else NSAMPLE
    idx = np.sort(rng.choice(p.T * p.A, size=min(n, p.T * p.A), replace=False))
    rows = np.array(sorted({0, 1, p.T // 2, p.T - 1}))
    return idx, rows


def _record(out, k, F, W, s, idx, rows):
    out[f"F_{k}"] = F.reshape(-1)[idx]
    out[f"W_{k}"] = W.reshape(-1)[idx]
    out[f"Frows_{k}"] = F[out["rows"]]
    out[f"Wrows_{k}"] = W[out["rows"]]
    for key in STAT_KEYS:
        if key in s:
            out[f"{key}_{k}"] = s[key]


def run(name):
    cfg, kw, snaps = JOBS[name]
    p = gen(cfg, **kw)
    idx, rows = _sample(p, name)
    out = {"config": cfg, "L": p.L, "T": p.T, "A": p.A, "N": p.N, "idx": idx, "rows": rows,
           "snaps": np.array(snaps), "shards": 1}
    t0 = time.time()
    st = oracle_init(p)
    for k in range(1, max(snaps) + 1):
        oracle_sweep(st)
        print(f"{name}: sweep {k} at {time.time() - t0:.0f}s", flush=True)
        if k in snaps:
            F, W = readout_flows(st)
            s = stats(st)
            s["dual_scale"] = float(p.eps * (s["mass"] + sum(abs(x) for x in dual_terms(st))))
            _record(out, k, F, W, s, idx, rows)
            np.savez_compressed(os.path.join(os.path.dirname(__file__), f"oracle_{name}.npz"), **out)
    print(f"{name}: done in {time.time() - t0:.0f}s")


def _rank_main(rank, world, port, name):
    import torch
    import torch.distributed as dist
    from oracle.shard import combine_lse, shard_pieces, combine_stats

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, kw, snaps = JOBS[name]
    p = gen(cfg, **kw)
    per = (p.L + world - 1) // world
    l0, l1 = min(rank * per, p.L), min((rank + 1) * per, p.L)
    q = p.commodity_slice(l0, l1)
    big = name in BIG
    b_store = None
    if big:
        os.makedirs(SCRATCH, exist_ok=True)
        b_store = np.lib.format.open_memmap(os.path.join(SCRATCH, f"{name}_b_{rank}.npy"), mode="w+",
                                            dtype=np.float64, shape=(q.T + 1, q.L, q.N))

    def reduce_lse(v):
        parts = [torch.zeros(v.shape[0], dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(v, np.float64)))
        return combine_lse(np.stack([x.numpy() for x in parts]))

    t0 = time.time()
    st = oracle_init(q, b_store=b_store, keep_forward=not big)
    dist.barrier()
    if rank == 0:
        print(f"{name}: init at {time.time() - t0:.0f}s", flush=True)
    idx, rows = _sample(p, name)
    out = {"config": cfg, "L": p.L, "T": p.T, "A": p.A, "N": p.N, "idx": idx, "rows": rows,
           "snaps": np.array(snaps), "shards": world}
    for k in range(1, max(snaps) + 1):
        oracle_sweep(st, reduce_lse=reduce_lse)
        dist.barrier()
        if rank == 0:
            print(f"{name}: sweep {k} at {time.time() - t0:.0f}s", flush=True)
        if k in snaps:
            pieces = shard_pieces(st)
            np.savez(os.path.join(SCRATCH, f"{name}_piece_{rank}.npz"), **pieces)
            dist.barrier()
            if rank == 0:
                allp = []
                for r in range(world):
                    z = np.load(os.path.join(SCRATCH, f"{name}_piece_{r}.npz"))
                    allp.append({key: (z[key] if key == "F" else float(z[key])) for key in z.files})
                s = combine_stats(p, allp, st.omega, st.sweeps)
                _record(out, k, s["F"], s["W"], s, idx, rows)
                np.savez_compressed(os.path.join(os.path.dirname(__file__), f"oracle_{name}.npz"), **out)
                print(f"{name}: snapshot {k} written at {time.time() - t0:.0f}s "
                      f"(mass {s['mass']:.12g}, dual {s['dual']:.12g})", flush=True)
            dist.barrier()
    dist.destroy_process_group()
    if big:
        del st, b_store
        os.remove(os.path.join(SCRATCH, f"{name}_b_{rank}.npy"))


def run_sharded(name, world):
    import torch.multiprocessing as mp
    os.makedirs(SCRATCH, exist_ok=True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_rank_main, args=(world, port, name), nprocs=world, join=True)



def add_dual_scale(name):
    """Post hoc for fixtures written before dual_scale was recorded: the same quantity from the per-shard pieces the
    sharded run left in .scratch/ (oracle outputs of the fixture's last snapshot)."""
    path = os.path.join(os.path.dirname(__file__), f"oracle_{name}.npz")
    z = dict(np.load(path))
    k = int(max(z["snaps"]))
    world = int(z["shards"])
    pieces = [np.load(os.path.join(SCRATCH, f"{name}_piece_{r}.npz")) for r in range(world)]
    p = gen(*[JOBS[name][0]], **JOBS[name][1])
    mass = sum(float(q["mass"]) for q in pieces)
    assert abs(mass - float(z[f"mass_{k}"])) <= 1e-12 * mass, "pieces of another run"
    z[f"dual_scale_{k}"] = float(p.eps * (mass + sum(abs(float(q["s0"])) + abs(float(q["sT"])) for q in pieces)
                                          + abs(float(pieces[0]["sd"]))))
    np.savez_compressed(path, **z)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, default=1)
    ap.add_argument("--add-dual-scale", action="store_true")
    ap.add_argument("names", nargs="+")
    a = ap.parse_args()
    for n in a.names:
        if a.add_dual_scale:
            add_dual_scale(n)
        elif a.shards > 1:
            run_sharded(n, a.shards)
        else:
            run(n)

