#!/usr/bin/env python
"""Benchmark of the colour-coding hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sg2v|reference]
                    [--template u15-1] [--precision f32] [--scale 20]

One STEP = one colouring: the whole hot path of SURVEY §8(a) (colouring kernel,
histogram, every fused SpMM+eMA step, top step, reduction) over the
RMAT-1M-like graph (SURVEY §8(d) D4 recipe) for the named template.
N > 1 (torchrun, one rank per GPU, NCCL): replica sharding of colourings
 — rank r runs colourings j ≡ r (mod N), an NCCL all-reduce
of the per-colouring counts ends the job; scaling "weak" (K colourings per rank).

Printed value = seconds per colouring for the whole job (max-over-ranks device
time ÷ colourings processed), lower is better.  `e2e` is the same metric through
the public API from HOST buffers (CSR upload + degree order + count + result
read-back inside the timed region).  `cpu_baseline` / `--impl reference` time the
CPU oracle (oracle/, as it stands) on the box's host cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seconds per coloring (u12–u17, RMAT-1M-like) at 1/2/4/8 B200; SpMM+eMA HBM GB/s"
UNIT = "s/coloring"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sg2v", choices=["sg2v", "reference"])
    p.add_argument("--template", default="u15-1")
    p.add_argument("--precision", default="f32", choices=["f32", "f64", "u64"])
    p.add_argument("--layout", default="anchored", choices=["anchored", "anchored_plain", "dense"])
    p.add_argument("--scale", type=int, default=20)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--mode", default="replicas", choices=["replicas", "vertex"],
                   help="replicas: colourings sharded over ranks (weak); vertex: every colouring's tables "
                        "row-partitioned over ranks with NCCL column-tile all-gathers (strong, SURVEY 8(e) V)")
    p.add_argument("--col-tile", type=int, default=0)
    return p.parse_args()


def _template(name):
    from sg2v_inputs import TEMPLATES
    e = TEMPLATES[name]
    return 1 + max(max(x) for x in e), e


def _workload_name(args, g):
    return (f"{args.template} on RMAT-1M-like (scale {args.scale}, RMAT(0.45,0.22,0.22,0.11), "
            f"n={g.n}, nnz={g.nnz})")


# --------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU oracle sample
def oracle_work(O, k, edges, n, nnz):
    """Loop count of the oracle's two-stage DP (SPEC-rule chain, root 0):
    Σ_steps nnz·C(k,p) + n·C(k,s)·C(s,a)  (gathers + eMA terms)."""
    nodes = O.partition(k, edges, 0)
    w = 0
    for size, _, a, p in nodes:
        if a < 0:
            continue
        sa, sp = nodes[a][0], nodes[p][0]
        w += nnz * math.comb(k, sp) + n * math.comb(k, size) * math.comb(size, sa)
    return w


def cpu_sample(args, k, edges, full_n, full_nnz, steps=1, target_s=12.0):
    """Time the CPU oracle (unchanged, two-stage, U64, OpenMP on all host cores)
    on a bounded sample: one colouring of the same template on the same RMAT
    recipe at a reduced scale, extrapolated to the full graph by the oracle's
    own work formula.  Returns (seconds per colouring list, description)."""
    from oracle import oracle as O
    from sg2v_inputs import rmat_1m_like
    O.build()
    cores = O.get_threads()
    full_w = oracle_work(O, k, edges, full_n, full_nnz)
    # pick the scale so one sample costs ~target_s (~4.5e8 u64 loop iterations/s/core, measured)
    rate = 4.5e8 * cores
    scale = 10
    while scale < args.scale:
        n_s = 1 << (scale + 1)
        if full_w * n_s / full_n / rate > target_s:
            break
        scale += 1
    g = rmat_1m_like(scale=scale, seed=args.seed)
    w = oracle_work(O, k, edges, g.n, g.nnz)
    out = []
    for t in range(steps):
        cols = O.colors(args.seed, t, g.n, k)
        t0 = time.perf_counter()
        O.count(g, k, edges, cols)
        out.append((time.perf_counter() - t0) * full_w / w)
    desc = (f"oracle two-stage DP (U64, OpenMP {cores} threads), 1 colouring per step of {args.template} on "
            f"RMAT-1M-like scale {scale} (n={g.n}, nnz={g.nnz}), extrapolated x{full_w / w:.1f} to the full "
            f"workload by the oracle's loop count sum_s nnz*C(k,p)+n*C(k,s)*C(s,a)")
    return out, desc, cores


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from sg2v_inputs import rmat_1m_like
    k, edges = _template(args.template)
    # full-size graph shape only (n, nnz) is needed for the extrapolation
    g = rmat_1m_like(scale=args.scale, seed=args.seed)
    n, nnz = g.n, g.nnz
    del g
    per, desc, cores = cpu_sample(args, k, edges, n, nnz, steps=args.warmup + args.steps, target_s=6.0)
    timed = per[args.warmup:]
    v = statistics.mean(timed)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.template} on RMAT-1M-like (scale {args.scale}, n={n}, nnz={nnz})",
                       "template": args.template, "precision": "u64"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def _setup_dist(world, local):
    """One rank per GPU over NCCL.  SG2V_BENCH_SHARED_GPU=1 (tests only) lets several
    ranks share the visible GPUs, with gloo for the (CPU) collectives."""
    import torch
    import torch.distributed as dist
    shared = os.environ.get("SG2V_BENCH_SHARED_GPU") == "1"
    dev = local % max(torch.cuda.device_count(), 1) if shared else local
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return dev


def _dist_device():
    import torch
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return "cuda"


def run_sg2v(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    dev = _setup_dist(world, local)

    import paper_2009_11665_b200 as sg
    from paper_2009_11665_b200.build import build
    from sg2v_inputs import degree_stats, rmat_1m_like

    build()
    k, edges = _template(args.template)
    g = rmat_1m_like(scale=args.scale, seed=args.seed)
    stats = degree_stats(g)
    # pinned host copies for the e2e leg
    ro_h = torch.from_numpy(g.row_offsets).pin_memory()
    ci_h = torch.from_numpy(g.col_indices).pin_memory()
    stream = torch.cuda.current_stream()

    G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
    T = sg.template_build(k, edges)
    plan = sg.plan_describe(G, T, args.precision, args.layout)
    ws = sg.Workspace(plan["workspace_bytes"])

    def colouring(t):  # colouring index of this rank's t-th colouring
        return rank + world * t

    # warm-up (untimed)
    for t in range(args.warmup):
        sg.count(G, T, n_iter=1, seed=args.seed, iter_offset=colouring(t), precision=args.precision,
                 workspace=ws, allow_overflow=True, layout=args.layout)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: K colourings per rank, device time (CUDA events) ----
    counts = torch.zeros(world * args.steps, dtype=torch.float64, device=_dist_device())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sg.profile_enable(True)
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        est, c = sg.count(G, T, n_iter=args.steps, seed=args.seed, iter_offset=colouring(args.warmup),
                          iter_stride=world, precision=args.precision, workspace=ws, allow_overflow=True, layout=args.layout)
        for t in range(args.steps):
            counts[rank + world * t] = float(c[t])
        if world > 1:
            dist.all_reduce(counts)  # NCCL: per-colouring counts of every rank
        ev1.record(stream)
        torch.cuda.synchronize()
    prof = sg.profile_read()
    sg.profile_enable(False)
    dev_s = ev0.elapsed_time(ev1) / 1e3
    t_max = torch.tensor([dev_s], dtype=torch.float64, device=_dist_device())
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total = world * args.steps
    value = float(t_max.item()) / total

    # ---- e2e: the public API from pinned HOST buffers, copies inside the timed region ----
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    del G
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(e2e_steps):
        Ge = sg.graph_load_csr(g.n, ro_h.numpy(), ci_h.numpy())
        sg.count(Ge, T, n_iter=1, seed=args.seed, iter_offset=colouring(args.warmup + args.steps + t),
                 precision=args.precision, workspace=ws, allow_overflow=True, layout=args.layout)  # includes D2H of the count
        Ge.free()
    e1.record(stream)
    torch.cuda.synchronize()
    e_max = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=_dist_device())
    if world > 1:
        dist.all_reduce(e_max, op=dist.ReduceOp.MAX)
    e2e_value = float(e_max.item()) / (world * max(e2e_steps, 1))

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel class (live CUDA events on the launching stream) ----
    dom = max(("step", "top", "hist"), key=lambda c: prof[c]["ms"])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = prof[dom]["bytes"] / (prof[dom]["ms"] / 1e3) / 1e9 if prof[dom]["ms"] > 0 else 0.0
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            key = f"{args.template}/{args.precision}/{args.layout}/scale{args.scale}"
            if key in tr:
                traffic = tr[key]
        except Exception:
            traffic = None
    launches = prof["color"]["launches"] + prof["hist"]["launches"] + prof["step"]["launches"] + \
        prof["top"]["launches"] + 2 * prof["reduce"]["launches"]
    clocks = clk.summary()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": _workload_name(args, g), "template": args.template, "k": k,
                   "precision": args.precision, "layout": args.layout, "graph": stats,
                   "parallelism": f"replicas{world}",
                   "colourings": total, "root": plan["root"], "workspace_GB": plan["workspace_bytes"] / 1e9,
                   "l2": "inputs larger than L2 (CSR %.2f GB + count tables %.1f GB >> 126 MB); no flush"
                         % (g.nbytes() / 1e9, plan["tables_bytes"] / 1e9)},
        "estimate": est, "colorful_first": float(c[0]),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(g.nbytes()),
                "d2h_bytes_per_step": 8},
        "gpu_launches": int(launches),
        "kernel_ms_per_step": {kk: v["ms"] / args.steps for kk, v in prof.items()},
        "roofline": {"bound": "hbm", "kernel": f"{dom} (fused SpMM+eMA, all launches)" if dom == "step" else dom,
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                     "bytes_per_step": prof[dom]["bytes"] / args.steps},
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        per, desc, cores = cpu_sample(args, k, edges, g.n, g.nnz, steps=1)
        line["cpu_baseline"] = {"value": per[0], "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_vertex(args):
    """--mode vertex: 1D vertex partition of every table across the ranks (capacity mode)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = world
    dev = _setup_dist(world, local)
    import paper_2009_11665_b200 as sg
    from paper_2009_11665_b200.build import build
    from sg2v_inputs import degree_stats, rmat_1m_like

    build()
    k, edges = _template(args.template)
    g = rmat_1m_like(scale=args.scale, seed=args.seed)
    stats = degree_stats(g)
    b, nl = sg.partition_rows(g.n, rank, world)
    ro = np.ascontiguousarray(g.row_offsets[b:b + nl + 1] - g.row_offsets[b])
    ci = np.ascontiguousarray(g.col_indices[g.row_offsets[b]:g.row_offsets[b + nl]])
    uid = [sg.Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = sg.Comm.nccl(uid[0], rank, world)
    Gp = sg.graph_load_partition(g.n, b, nl, ro, ci)
    T = sg.template_build(k, edges)
    kw = dict(seed=args.seed, precision=args.precision, comm=comm, col_tile=args.col_tile, allow_overflow=True)
    for t in range(args.warmup):
        sg.count(Gp, T, n_iter=1, iter_offset=t, **kw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sg.profile_enable(True)
    with Clocks(dev) as clk:
        ev0.record(stream)
        est, c = sg.count(Gp, T, n_iter=args.steps, iter_offset=args.warmup, **kw)
        ev1.record(stream)
        torch.cuda.synchronize()
    prof = sg.profile_read()
    sg.profile_enable(False)
    t_max = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device=_dist_device())
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    value = float(t_max.item()) / args.steps
    # e2e: partition upload from host + count + read-back, per step
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(e2e_steps):
        Ge = sg.graph_load_partition(g.n, b, nl, ro, ci)
        sg.count(Ge, T, n_iter=1, iter_offset=args.warmup + args.steps + t, **kw)
        Ge.free()
    e1.record(stream)
    torch.cuda.synchronize()
    e_max = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=_dist_device())
    if world > 1:
        dist.all_reduce(e_max, op=dist.ReduceOp.MAX)
    e2e_value = float(e_max.item()) / max(e2e_steps, 1)
    comm.free()
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        dom = "step"
        achieved = prof[dom]["bytes"] / (prof[dom]["ms"] / 1e3) / 1e9 if prof[dom]["ms"] > 0 else 0.0
        launches = sum(v["launches"] for v in prof.values()) + prof["reduce"]["launches"]
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
                "config": {"workload": _workload_name(args, g), "template": args.template, "k": k,
                           "precision": args.precision, "layout": "anchored", "graph": stats,
                           "parallelism": f"vertex{world}", "rows_per_rank": nl, "col_tile": args.col_tile,
                           "l2": "inputs larger than L2; no flush"},
                "estimate": est, "colorful_first": float(c[0]),
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(ro.nbytes + ci.nbytes),
                        "d2h_bytes_per_step": 8},
                "gpu_launches": int(launches),
                "kernel_ms_per_step": {kk: v["ms"] / args.steps for kk, v in prof.items()},
                "roofline": {"bound": "hbm", "kernel": "step (tile gathers of rank 0)", "achieved": achieved,
                             "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "vertex":
        return run_vertex(args)
    return run_sg2v(args)


if __name__ == "__main__":
    sys.exit(main())
