"""Convenience wrapper: one ``Solver`` = one mmf context (include/mmf.h), marshalling only.

PyTorch supplies the device workspace (a uint8 tensor) and the CUDA stream; every computation of the
sweep happens in libmmf.so.  Commodity sharding: pass ``l_begin``/``l_count`` and an NCCL unique id.
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np

from . import _lib as L


class Solver:
    def __init__(self, problem, prec: Optional[str] = None, device: int = 0, stream=None, graph: bool = True,
                 reorder: bool = True, profile: bool = False, l_begin: int = 0, l_count: Optional[int] = None,
                 nccl_uid: Optional[bytes] = None, nranks: int = 1, rank: int = 0, options: Optional[dict] = None):
        import torch  # device memory + streams only

        self.p = problem
        prec = prec or getattr(problem, "prec", "fp64")
        self.prec = prec
        self.device = device
        self.torch_device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.torch_device)
        self.stream = stream
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self.ctx = L.mmf_create(device, L.MMF_FP32 if prec == "fp32" else L.MMF_FP64, handle)
        self._ws = None
        try:
            L.mmf_set_option(self.ctx, "graph", int(graph))
            L.mmf_set_option(self.ctx, "reorder", int(reorder))
            L.mmf_set_option(self.ctx, "profile", int(profile))
            opts = dict(options or {})
            if "kernels" not in opts and os.environ.get("MMF_KERNELS"):  # test / profiling override
                opts["kernels"] = int(os.environ["MMF_KERNELS"])
            for k, v in opts.items():
                L.mmf_set_option(self.ctx, k, int(v))
            self.upload(problem, l_begin, l_count)
            if nccl_uid is not None:
                L.mmf_attach_nccl(self.ctx, nccl_uid, nranks, rank)
            nbytes = L.mmf_workspace_bytes(self.ctx)
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.torch_device)
            L.mmf_set_workspace(self.ctx, self._ws.data_ptr(), nbytes)
            L.mmf_init(self.ctx)
        except Exception:
            self.close()
            raise

    def upload(self, p, l_begin: int = 0, l_count: Optional[int] = None):
        l_count = p.L - l_begin if l_count is None else l_count
        self.l_begin, self.l_count = l_begin, l_count
        L.mmf_set_graph(self.ctx, p.N, p.tail, p.head)
        L.mmf_set_costs(self.ctx, p.T, p.eps, p.cost, p.cost.ndim == 2)
        L.mmf_set_capacity(self.ctx, p.cap, p.cap.ndim == 2)
        if getattr(p, "node_cap", None) is not None:  # SURVEY 8(f) NEXT-3 (state capacities)
            L.mmf_set_node_capacity(self.ctx, p.node_cap, np.ndim(p.node_cap) == 2)
        sl = slice(l_begin, l_begin + l_count)
        if p.is_point:
            L.mmf_set_point_marginals(self.ctx, p.L, l_begin, p.src[sl], p.dst[sl], p.mass[sl])
        else:
            L.mmf_set_marginals(self.ctx, p.L, l_begin, p.mu0[sl], p.muT[sl])
        if getattr(p, "node_cost", None) is not None:
            L.mmf_set_node_costs(self.ctx, p.node_cost[sl])
        if getattr(p, "t_in", None) is not None or getattr(p, "t_out", None) is not None:
            t_in = np.zeros(p.L, np.int32) if p.t_in is None else np.asarray(p.t_in, np.int32)
            t_out = np.full(p.L, p.T, np.int32) if p.t_out is None else np.asarray(p.t_out, np.int32)
            L.mmf_set_commodity_times(self.ctx, t_in[sl], t_out[sl])

    def sweep(self, n: int = 1):
        L.mmf_sweep(self.ctx, n)

    def sync(self):
        L.mmf_sync(self.ctx)

    def commodity_flows(self, t: int) -> np.ndarray:
        """Per-commodity arc flows of step t, [A, l_count] fp64 in user arc order (this solver's commodities)."""
        return L.mmf_read_commodity_flows(self.ctx, t, self.p.A, self.l_count)

    def save_state(self) -> bytes:
        """Checkpoint (W and UT of the end-of-sweep state; include/mmf.h mmf_save_state)."""
        return L.mmf_save_state(self.ctx)

    def load_state(self, state: bytes):
        """Resume from a checkpoint of the same problem (any kernel options)."""
        L.mmf_load_state(self.ctx, state)

    def solve(self, tol: float, max_sweeps: int, check_every: int = 1) -> dict:
        """Sweeps until the end-of-sweep error (marginal mismatches + capacity excess, relative to the mass)
        is below tol; returns {converged, sweeps, err, history}."""
        return L.mmf_solve(self.ctx, tol, max_sweeps, check_every)

    def edge_flows(self) -> np.ndarray:
        return L.mmf_read_edge_flows(self.ctx, self.p.T, self.p.A)

    def cap_duals(self) -> np.ndarray:
        return L.mmf_read_cap_duals(self.ctx, self.p.T, self.p.A)

    def node_duals(self) -> np.ndarray:
        """Node-capacity duals u_t[j], [T+1, N] (NEXT-3)."""
        return L.mmf_read_node_duals(self.ctx, self.p.T, self.p.N)

    def stats(self) -> dict:
        return L.mmf_read_stats(self.ctx)

    def kernel_stats(self) -> dict:
        return L.mmf_read_kernel_stats(self.ctx)

    def sweep_bytes(self):
        return L.mmf_sweep_bytes(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            L.mmf_destroy(self.ctx)
            self.ctx = None
        self._ws = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
