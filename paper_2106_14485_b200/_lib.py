"""Thin ctypes binding of include/mmf.h: same names, argument marshalling only.

Every step of the sweep runs in libmmf.so's CUDA kernels.  There is no CPU fallback: if the library
(or a CUDA device) is missing, the calls raise ``MMFError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmmf.so")

STATUS = {0: "MMF_OK", 1: "MMF_EVERIFY", 2: "MMF_EINVAL", 3: "MMF_ENOTCONV", 4: "MMF_EINFEASIBLE",
          5: "MMF_ENOMEM", 6: "MMF_ECUDA", 7: "MMF_ENCCL", 8: "MMF_ESTATE", 9: "MMF_ERANGE"}
MMF_FP64, MMF_FP32 = 0, 1

# functions declared in include/mmf.h (checked by tests/test_abi.py against the header)
EXPORTS = ["mmf_create", "mmf_set_graph", "mmf_set_costs", "mmf_set_capacity", "mmf_set_marginals",
           "mmf_set_point_marginals", "mmf_workspace_bytes", "mmf_set_workspace", "mmf_attach_nccl", "mmf_nccl_unique_id",
           "mmf_set_option", "mmf_init", "mmf_sweep", "mmf_sync", "mmf_read_edge_flows", "mmf_read_cap_duals",
           "mmf_read_stats", "mmf_read_kernel_stats", "mmf_sweep_bytes", "mmf_destroy", "mmf_last_error",
           "mmf_version", "mmf_solve", "mmf_state_bytes", "mmf_save_state", "mmf_load_state",
           "mmf_read_commodity_flows", "mmf_set_node_costs", "mmf_sweep_group",
           "mmf_set_commodity_times", "mmf_set_node_capacity", "mmf_read_node_duals"]


class MMFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class mmf_stats(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("mass", C.c_double), ("src_mismatch", C.c_double),
                ("sink_mismatch", C.c_double), ("cap_violation", C.c_double), ("dual", C.c_double),
                ("primal", C.c_double)]


_lib = None


def load(path: str = None):
    """Load libmmf.so (raises if it was not built: there is no fallback path).  MMF_LIB overrides the
    path (profiling builds of the same sources)."""
    path = path or os.environ.get("MMF_LIB", LIB_PATH)
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise MMFError(6, f"{path} not built (run __graft_entry__.build() or python paper_2106_14485_b200/build.py)")
    lib = C.CDLL(path)
    vp, i32, i64, dp, ip = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int32)
    sig = {
        "mmf_create": ([C.POINTER(vp), C.c_int, C.c_int, vp], C.c_int),
        "mmf_set_graph": ([vp, i32, i64, ip, ip], C.c_int),
        "mmf_set_costs": ([vp, i32, C.c_double, dp, C.c_int], C.c_int),
        "mmf_set_capacity": ([vp, dp, C.c_int], C.c_int),
        "mmf_set_marginals": ([vp, i32, i32, i32, dp, dp], C.c_int),
        "mmf_set_point_marginals": ([vp, i32, i32, i32, ip, ip, dp], C.c_int),
        "mmf_workspace_bytes": ([vp, C.POINTER(C.c_size_t)], C.c_int),
        "mmf_set_workspace": ([vp, vp, C.c_size_t], C.c_int),
        "mmf_attach_nccl": ([vp, C.c_char_p, C.c_int, C.c_int], C.c_int),
        "mmf_nccl_unique_id": ([C.c_char_p], C.c_int),
        "mmf_set_option": ([vp, C.c_char_p, i64], C.c_int),
        "mmf_init": ([vp], C.c_int),
        "mmf_sweep": ([vp, i32], C.c_int),
        "mmf_sync": ([vp], C.c_int),
        "mmf_read_edge_flows": ([vp, dp], C.c_int),
        "mmf_read_cap_duals": ([vp, dp], C.c_int),
        "mmf_read_stats": ([vp, C.POINTER(mmf_stats)], C.c_int),
        "mmf_solve": ([vp, C.c_double, i32, i32, C.POINTER(C.c_int32), dp, dp], C.c_int),
        "mmf_state_bytes": ([vp, C.POINTER(C.c_size_t)], C.c_int),
        "mmf_read_commodity_flows": ([vp, i32, dp], C.c_int),
        "mmf_save_state": ([vp, vp, C.c_size_t], C.c_int),
        "mmf_load_state": ([vp, vp, C.c_size_t], C.c_int),
        "mmf_read_kernel_stats": ([vp, C.POINTER(C.c_int64), dp, C.c_int], C.c_int),
        "mmf_sweep_bytes": ([vp, dp, dp, C.c_int], C.c_int),
        "mmf_set_node_costs": ([vp, dp], C.c_int),
        "mmf_sweep_group": ([C.POINTER(vp), i32, i32], C.c_int),
        "mmf_set_commodity_times": ([vp, ip, ip], C.c_int),
        "mmf_set_node_capacity": ([vp, dp, C.c_int], C.c_int),
        "mmf_read_node_duals": ([vp, dp], C.c_int),
        "mmf_destroy": ([vp], C.c_int),
        "mmf_last_error": ([vp], C.c_char_p),
        "mmf_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name, None)
        if f is None and "MMF_LIB" in os.environ:  # (an older build for comparisons: only the calls it has)
            continue
        f.argtypes, f.restype = args, res
    _lib = lib
    return lib


def _check(ctx, status: int):
    if status != 0:
        msg = load().mmf_last_error(ctx).decode(errors="replace")
        raise MMFError(status, msg)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ----------------------------------------------------------------------------- the C calls

def mmf_version() -> str:
    return load().mmf_version().decode()


def mmf_create(device: int, prec: int, stream: int = 0):
    lib = load()
    ctx = C.c_void_p()
    st = lib.mmf_create(C.byref(ctx), int(device), int(prec), C.c_void_p(stream or None))
    if st != 0:
        raise MMFError(st, lib.mmf_last_error(None).decode())
    return ctx


def mmf_set_graph(ctx, N: int, tail, head):
    tail, head = _i32(tail), _i32(head)
    _check(ctx, load().mmf_set_graph(ctx, int(N), int(tail.size), _p(tail, C.c_int32), _p(head, C.c_int32)))


def mmf_set_costs(ctx, T: int, eps: float, cost, time_varying: bool):
    cost = _f64(cost)
    _check(ctx, load().mmf_set_costs(ctx, int(T), float(eps), _p(cost, C.c_double), int(bool(time_varying))))


def mmf_set_capacity(ctx, cap, time_varying: bool):
    cap = _f64(cap)
    _check(ctx, load().mmf_set_capacity(ctx, _p(cap, C.c_double), int(bool(time_varying))))


def mmf_set_marginals(ctx, L_global: int, l_begin: int, mu0, muT):
    mu0, muT = _f64(mu0), _f64(muT)
    _check(ctx, load().mmf_set_marginals(ctx, int(L_global), int(l_begin), int(mu0.shape[0]),
                                         _p(mu0, C.c_double), _p(muT, C.c_double)))


def mmf_set_point_marginals(ctx, L_global: int, l_begin: int, src, dst, mass):
    src, dst, mass = _i32(src), _i32(dst), _f64(mass)
    _check(ctx, load().mmf_set_point_marginals(ctx, int(L_global), int(l_begin), int(src.size), _p(src, C.c_int32),
                                               _p(dst, C.c_int32), _p(mass, C.c_double)))


def mmf_set_node_costs(ctx, c):
    """c: [l_count, N] commodity node costs (None clears)."""
    if c is None:
        _check(ctx, load().mmf_set_node_costs(ctx, None))
        return
    c = _f64(c)
    _check(ctx, load().mmf_set_node_costs(ctx, _p(c, C.c_double)))


def mmf_set_commodity_times(ctx, t_in, t_out):
    """Per-commodity entry / exit layers of this context's commodities (None clears)."""
    if t_in is None:
        _check(ctx, load().mmf_set_commodity_times(ctx, None, None))
        return
    t_in, t_out = _i32(t_in), _i32(t_out)
    _check(ctx, load().mmf_set_commodity_times(ctx, _p(t_in, C.c_int32), _p(t_out, C.c_int32)))


def mmf_set_node_capacity(ctx, cap, time_varying: bool):
    if cap is None:
        _check(ctx, load().mmf_set_node_capacity(ctx, None, 0))
        return
    cap = _f64(cap)
    _check(ctx, load().mmf_set_node_capacity(ctx, _p(cap, C.c_double), int(bool(time_varying))))


def mmf_read_node_duals(ctx, T: int, N: int) -> np.ndarray:
    out = np.empty((T + 1, N), np.float64)
    _check(ctx, load().mmf_read_node_duals(ctx, _p(out, C.c_double)))
    return out


def mmf_workspace_bytes(ctx) -> int:
    n = C.c_size_t()
    _check(ctx, load().mmf_workspace_bytes(ctx, C.byref(n)))
    return int(n.value)


def mmf_set_workspace(ctx, dptr: int, nbytes: int):
    _check(ctx, load().mmf_set_workspace(ctx, C.c_void_p(dptr), C.c_size_t(nbytes)))


def mmf_attach_nccl(ctx, unique_id: bytes, nranks: int, rank: int):
    assert len(unique_id) == 128
    _check(ctx, load().mmf_attach_nccl(ctx, C.c_char_p(bytes(unique_id)), int(nranks), int(rank)))


def mmf_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load().mmf_nccl_unique_id(buf)
    if st != 0:
        raise MMFError(st, load().mmf_last_error(None).decode())
    return buf.raw


def mmf_set_option(ctx, key: str, value: int):
    _check(ctx, load().mmf_set_option(ctx, key.encode(), int(value)))


def mmf_init(ctx):
    _check(ctx, load().mmf_init(ctx))


def mmf_sweep(ctx, n: int):
    _check(ctx, load().mmf_sweep(ctx, int(n)))


def mmf_sweep_group(ctxs, n: int):
    """Virtual ranks: sweep the contexts (commodity shards of one problem on one device) together."""
    arr = (C.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    _check(ctxs[0], load().mmf_sweep_group(arr, len(ctxs), int(n)))


def mmf_sync(ctx):
    _check(ctx, load().mmf_sync(ctx))


def mmf_read_edge_flows(ctx, T: int, A: int, out=None) -> np.ndarray:
    out = np.empty((T, A), np.float64) if out is None else out
    _check(ctx, load().mmf_read_edge_flows(ctx, _p(out, C.c_double)))
    return out


def mmf_read_cap_duals(ctx, T: int, A: int, out=None) -> np.ndarray:
    out = np.empty((T, A), np.float64) if out is None else out
    _check(ctx, load().mmf_read_cap_duals(ctx, _p(out, C.c_double)))
    return out


def mmf_solve(ctx, tol: float, max_sweeps: int, check_every: int = 1) -> dict:
    """Sweeps until the end-of-sweep error is below tol (MMF_ENOTCONV is reported as converged=False)."""
    done = C.c_int32(0)
    err = C.c_double(0.0)
    hist = np.zeros(max(1, -(-max_sweeps // max(check_every, 1))), np.float64)
    st = load().mmf_solve(ctx, float(tol), int(max_sweeps), int(check_every), C.byref(done), C.byref(err),
                          hist.ctypes.data_as(C.POINTER(C.c_double)))
    if st not in (0, 3):
        _check(ctx, st)
    n = -(-done.value // max(check_every, 1))
    return {"converged": st == 0, "sweeps": done.value, "err": err.value, "history": hist[:n].copy()}


def mmf_read_commodity_flows(ctx, t: int, A: int, L: int) -> np.ndarray:
    out = np.empty((A, L), np.float64)
    _check(ctx, load().mmf_read_commodity_flows(ctx, int(t), _p(out, C.c_double)))
    return out


def mmf_save_state(ctx) -> bytes:
    n = C.c_size_t(0)
    _check(ctx, load().mmf_state_bytes(ctx, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(ctx, load().mmf_save_state(ctx, buf, n))
    return buf.raw


def mmf_load_state(ctx, state: bytes):
    _check(ctx, load().mmf_load_state(ctx, C.c_char_p(state), len(state)))


def mmf_read_stats(ctx) -> dict:
    s = mmf_stats()
    _check(ctx, load().mmf_read_stats(ctx, C.byref(s)))
    return {k: getattr(s, k) for k, _ in mmf_stats._fields_}


KERNEL_KINDS = ["bwd_step", "fwd_flow", "fwd_reduce", "fwd_update", "boundary", "other", "fwd_fused", "spare"]


def mmf_read_kernel_stats(ctx) -> dict:
    n = len(KERNEL_KINDS)
    launches = (C.c_int64 * n)()
    ms = (C.c_double * n)()
    _check(ctx, load().mmf_read_kernel_stats(ctx, launches, ms, n))
    return {k: {"launches": int(launches[i]), "ms": float(ms[i])} for i, k in enumerate(KERNEL_KINDS)}


def mmf_sweep_bytes(ctx) -> tuple:
    n = len(KERNEL_KINDS)
    tot = C.c_double()
    per = (C.c_double * n)()
    _check(ctx, load().mmf_sweep_bytes(ctx, C.byref(tot), per, n))
    return float(tot.value), {k: float(per[i]) for i, k in enumerate(KERNEL_KINDS)}


def mmf_destroy(ctx):
    load().mmf_destroy(ctx)
