"""bench.py — one Gauss-Seidel Sinkhorn sweep per step, B200, JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl mmf|reference]

Default workload: BASELINE.json config [4] (road-like 200x200 grid, T=200, L=1024, eps=0.01, fp32
mode) — the config the north star's >=60 % HBM and 8-GPU scaling targets are quoted on.
Under torchrun (N > 1) the L commodities are sharded over ranks (strong scaling) and the per-step
edge flows are all-reduced with NCCL inside the library.

value   = L_global * |A| * T updates per sweep / device time per sweep (max over ranks), inputs resident
e2e     = same metric through the public API with host buffers: problem upload, init, K sweeps,
          edge-flow + dual readout to host, all inside the timed region
roofline: dominant kernel's algorithmic bytes per launch / its average CUDA-event duration (an
          attribution pass of the same K sweeps with per-kernel events on the launch stream)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "commodity·edge·timestep updates/s per Sinkhorn sweep; % of HBM peak"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--L", type=int, default=None, help="override L (lite variants)")
    ap.add_argument("--prec", default=None)
    ap.add_argument("--impl", default="mmf", choices=["mmf", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def workload_name(p, cfg):
    from workloads import CONFIG_NAMES
    return f"cfg{cfg}-{CONFIG_NAMES.get(cfg, p.name)}" + ("" if p.L == {1: 3, 2: 32, 3: 256, 4: 1024, 5: 8192}[cfg] else f"-L{p.L}")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9 for k in range(4) if r[5 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(p, budget_L=4):
    """The oracle as it stands on a bounded sample: the same graph, T, eps and capacities with the
    first ``budget_L`` commodities, one sweep timed (init excluded), single process."""
    from oracle import oracle_init, oracle_sweep
    q = p.commodity_slice(0, min(budget_L, p.L))
    st = oracle_init(q)
    t0 = time.perf_counter()
    oracle_sweep(st)
    dt = time.perf_counter() - t0
    return {"value": q.updates_per_sweep() / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 sweep, first {q.L} of {p.L} commodities, full graph (|A|={p.A}) and T={p.T}; "
                      f"{dt:.1f} s; host os.cpu_count()={os.cpu_count()}",
            "seconds_per_sweep_sample": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads import gen
    from oracle import oracle_init, oracle_sweep
    p = gen(args.config, L=args.L, prec=args.prec)
    q = p.commodity_slice(0, min(2, p.L))
    st = oracle_init(q)
    for _ in range(args.warmup):
        oracle_sweep(st)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_sweep(st)
    dt = (time.perf_counter() - t0) / args.steps
    value = q.updates_per_sweep() / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(p, args.config), "N": p.N, "A": p.A, "T": p.T, "L": p.L, "eps": p.eps},
        "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", "cores": 1,
                         "sample": f"each step = 1 oracle sweep of the first {q.L} commodities (full graph, T)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def l2_note(p, prec, nl):
    """Working set a sweep streams (alpha and beta stores, extended range) against the 126 MB L2."""
    be = 6 if prec == "fp32" else 12
    store = 2 * (p.T + 1) * p.N * nl * be
    if store > 4 * 126e6:
        return f"inputs larger than L2 (message stores {store / 1e9:.1f} GB per sweep, no flush)"
    return (f"message stores {store / 1e6:.0f} MB per sweep: partly L2-resident, no flush "
            "(small parity config, not the bench workload)")


def self_launch(args):
    """--gpus N without a torchrun environment: launch N ranks here (one per GPU, 127.0.0.1 rendezvous) with the same
    arguments; rank 0's JSON line passes through."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(self_launch(args))
    if world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2106_14485_b200 import Solver, _lib
    from workloads import gen

    p = gen(args.config, L=args.L, prec=args.prec)
    prec = args.prec or p.prec
    per = (p.L + world - 1) // world
    l0, l1 = min(rank * per, p.L), min((rank + 1) * per, p.L)
    uid = None
    if world > 1:
        obj = [_lib.mmf_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.Stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    solver = Solver(p, prec=prec, device=local, stream=stream, l_begin=l0, l_count=l1 - l0, nccl_uid=uid,
                    nranks=world, rank=rank)
    with torch.cuda.stream(stream):
        solver.sweep(args.warmup)
        solver.sync()
        k0 = solver.kernel_stats()
        barrier()
        torch.cuda.synchronize(dev)
        clocks = Clocks(local)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solver.sweep(args.steps)
        e1.record(stream)
        solver.sync()
        torch.cuda.synchronize(dev)
        clk = clocks.stop()
        barrier()
        ms_total = max_over_ranks(e0.elapsed_time(e1))
        k1 = solver.kernel_stats()
        launches = sum(k1[k]["launches"] - k0[k]["launches"] for k in k1)
        ms_step = ms_total / args.steps
        U = p.updates_per_sweep()
        value = U / (ms_step / 1e3)
        bytes_total, bytes_kind = solver.sweep_bytes()
        # attribution pass: same K sweeps, per-kernel CUDA events on the launch stream
        _lib.mmf_set_option(solver.ctx, "profile", 1)
        kp0 = solver.kernel_stats()
        solver.sweep(args.steps)
        solver.sync()
        kp1 = solver.kernel_stats()
        _lib.mmf_set_option(solver.ctx, "profile", 0)
    kinds = {k: {"launches": kp1[k]["launches"] - kp0[k]["launches"], "ms": kp1[k]["ms"] - kp0[k]["ms"]} for k in kp1}
    tot_ms = sum(v["ms"] for v in kinds.values()) or 1.0
    dom = max(kinds, key=lambda k: kinds[k]["ms"])
    dom_launch_ms = kinds[dom]["ms"] / max(kinds[dom]["launches"], 1)
    dom_bytes_per_launch = bytes_kind[dom] / max(kinds[dom]["launches"] / args.steps, 1)
    peak, peak_kind = measured_peaks()
    achieved = dom_bytes_per_launch / (dom_launch_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_final", "traffic.json")
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    if os.path.exists(tpath):  # ncu dram bytes per launch of the same kernel and workload (committed capture)
        with open(tpath) as f:
            tj = json.load(f).get(workload_name(p, args.config), {}).get(dom)
        if tj:
            traffic = tj["dram_read"] + tj["dram_write"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_kind, "traffic": traffic,
            "share_of_step": kinds[dom]["ms"] / tot_ms,
            "bytes_per_launch": dom_bytes_per_launch, "avg_launch_ms": dom_launch_ms}
    sweep_gbs = bytes_total / (ms_step / 1e3) / 1e9  # (per GPU: mmf_sweep_bytes counts this rank's commodities)

    e2e = None
    if not args.no_e2e:
        uid2 = None
        if world > 1:
            obj = [_lib.mmf_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid2 = obj[0]
        solver.close()
        dts = []
        for rep in range(2 if world == 1 else 1):  # (one GPU: two repetitions, the faster one reported; both listed)
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                s2 = Solver(p, prec=prec, device=local, stream=stream, l_begin=l0, l_count=l1 - l0, nccl_uid=uid2,
                            nranks=world, rank=rank)
                s2.sweep(args.steps)
                F = s2.edge_flows()
                W = s2.cap_duals()
                s2.close()
            dts.append(max_over_ranks(time.perf_counter() - t0))
        dt = min(dts)
        nl = l1 - l0
        h2d = (2 * p.A * 4 + p.cost.nbytes + p.cap.nbytes + (nl * 16 if p.is_point else 2 * nl * p.N * 8)) / args.steps
        d2h = (F.nbytes + W.nbytes) / args.steps
        e2e = {"value": U * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "seconds": dt, "seconds_all_repetitions": dts, "includes": "set_graph/costs/capacity/marginals (host->device), init, K sweeps, "
                                          "edge flows + duals (device->host), per rank"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(p)
    solver.close()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": workload_name(p, args.config), "N": p.N, "A": p.A, "E": p.A - p.n_loops,
                       "T": p.T, "L": p.L, "eps": p.eps, "prec": prec,
                       "message_format": "significand f32 + exponent i16" if prec == "fp32" else "f64 + i32",
                       "parallelism": f"commodity-shard x{world}",
                       "l2": l2_note(p, prec, l1 - l0)},
            "sweeps_per_s": 1e3 / ms_step,
            "updates_per_s_E_only": (p.A - p.n_loops) * p.L * p.T / (ms_step / 1e3),
            "bytes_per_sweep_model": bytes_total * world,
            "hbm_frac_sweep_model": sweep_gbs / peak,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": launches,
            "kernel_breakdown_ms_per_step": {k: v["ms"] / args.steps for k, v in kinds.items() if v["launches"]},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
