"""Commodity sharding (rem:multi_tensor_scheme P:1139-1147): the commodities couple only
through the per-step aggregate edge flows in the capacity-dual update, so G ranks that each hold a slice of
the commodities and all-reduce the per-step flows before every W_t update reproduce the unsharded sweep.

CPU, world size 2, gloo: each rank runs the float64 oracle on its slice with the per-step flow sum
all-reduced (log domain: max-shifted sum) — the exchange the library performs with ncclAllReduce of F_t —
and the result must equal the unsharded oracle.  The library's own NCCL exchange path is exercised on
the GPU box with a one-rank communicator (tests/test_gpu_parity.py::test_nccl_exchange_path_one_rank).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from workloads import grid_problem

SWEEPS = 6


def _problem():
    return grid_problem(4, 5, 6, 6, 0.2, seed=41, cap=(0.2, 0.6))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from oracle import oracle_init, oracle_sweep
    from oracle.sweep import readout_commodity_flows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = _problem()
    per = (p.L + world - 1) // world
    l0, l1 = rank * per, min((rank + 1) * per, p.L)
    q = p.commodity_slice(l0, l1)

    def reduce_lse(v):
        v = torch.from_numpy(np.asarray(v, np.float64).copy())
        finite = torch.isfinite(v)
        m = torch.where(finite, v, torch.full_like(v, -1e300))
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        e = torch.where(finite, torch.exp(v - m), torch.zeros_like(v))
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        with np.errstate(divide="ignore"):
            return np.where(e.numpy() > 0, m.numpy() + np.log(e.numpy()), -np.inf)

    st = oracle_init(q)
    for _ in range(SWEEPS):
        oracle_sweep(st, reduce_lse=reduce_lse)
    F = torch.from_numpy(np.stack([readout_commodity_flows(st, t).sum(axis=1) for t in range(p.T)]))
    dist.all_reduce(F, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.savez(os.path.join(out_dir, "sharded.npz"), F=F.numpy(), W=np.exp(st.omega))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_commodity_sharding_equals_unsharded(tmp_path):
    from oracle import oracle_run, readout_flows
    from tests._metrics import max_rel_err, flow_floor

    port = _free_port()
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    z = np.load(tmp_path / "sharded.npz")
    p = _problem()
    Fo, Wo = readout_flows(oracle_run(p, SWEEPS))
    assert max_rel_err(z["F"], Fo, flow_floor(p)) < 1e-12
    assert max_rel_err(z["W"], Wo, 1e-30) < 1e-12
    assert np.min(Wo) < 0.999  # capacities bind: the exchange matters


def test_shard_bounds_cover_all_commodities():
    """bench.py's slicing: rank r owns [r*ceil(L/G), min((r+1)*ceil(L/G), L)); the slices partition [0, L)."""
    for L in (1, 3, 32, 1024, 8192):
        for G in (1, 2, 4, 8):
            per = (L + G - 1) // G
            sl = [(min(r * per, L), min((r + 1) * per, L)) for r in range(G)]
            covered = np.zeros(L, int)
            for a, b in sl:
                covered[a:b] += 1
            assert np.all(covered == 1)
