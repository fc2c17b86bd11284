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
    p.add_argument("--graph", default="rmat1m", choices=["rmat1m", "gs22", "miami", "orkut"],
                   help="rmat1m: RMAT-1M-like at --scale (D4); gs22: Graph500-like scale 22 (D5a); miami (D2); orkut (D3)")
    p.add_argument("--no-balance", action="store_true",
                   help="vertex mode: uniform row blocks of the input ids instead of the degree-dealt relabelling")
    return p.parse_args()


def _template(name):
    from sg2v_inputs import TEMPLATES
    e = TEMPLATES[name]
    return 1 + max(max(x) for x in e), e


def _workload_name(args, g):
    if args.graph != "rmat1m":
        return f"{args.template} on {g.name} (n={g.n}, nnz={g.nnz})"
    return (f"{args.template} on RMAT-1M-like (scale {args.scale}, RMAT(0.45,0.22,0.22,0.11), "
            f"n={g.n}, nnz={g.nnz})")


def _load_graph(args):
    from sg2v_inputs import BIG_GRAPHS, rmat_1m_like
    if args.graph == "rmat1m":
        return rmat_1m_like(scale=args.scale, seed=args.seed)
    return BIG_GRAPHS[args.graph]()


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
    # pick the scale so one sample costs ~target_s (~4.5e8 u64 loop iterations/s/core, measured),
    # but never below the scale whose widest oracle table is ~1 GB: small samples are cache- and
    # overhead-dominated and extrapolate badly (scale 11: 2x the full-graph time, scale 14: 0.75x)
    rate = 4.5e8 * cores
    scale = 10
    while scale < args.scale and _widest_table_gb(O, k, edges, 1 << scale) < 0.8:
        scale += 1
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
            f"RMAT-1M-like scale {scale} (n={g.n}, nnz={g.nnz}; its widest table "
            f"{_widest_table_gb(O, k, edges, g.n):.2f} GB >> the host's L3), extrapolated x{full_w / w:.1f} to the "
            f"full workload by the oracle's loop count sum_s nnz*C(k,p)+n*C(k,s)*C(s,a)")
    return out, desc, cores


def _widest_table_gb(O, k, edges, n):
    return max(math.comb(k, size) for size, _, _, _ in O.partition(k, edges, 0)) * n * 8 / 1e9


def full_graph_oracle_record(template, scale):
    """The oracle timed on the FULL bench graph (tools/make_golden_big.py on the GPU box's
    host; tests/golden/big_configs.json), for cross-checking the bounded sample."""
    if scale != 20:
        return None
    try:
        cases = json.load(open(os.path.join(ROOT, "tests", "golden", "big_configs.json")))["cases"]
    except Exception:
        return None
    for c in cases:
        if c["graph"] == "rmat1m" and c["template"] == template and c.get("oracle_seconds_u64"):
            h = c.get("host", {})
            return {"full_graph_u64_s": c["oracle_seconds_u64"], "threads": c.get("threads"),
                    "cpu_model": h.get("cpu_model"), "mem_total_GB": h.get("mem_total_GB"),
                    "j": c["j"], "source": "tests/golden/big_configs.json (tools/make_golden_big.py)"}
    return None


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
    cb = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    full = full_graph_oracle_record(args.template, args.scale)
    if full:
        cb["full_graph_measured"] = full
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.template} on RMAT-1M-like (scale {args.scale}, n={n}, nnz={nnz})",
                       "template": args.template, "precision": "u64"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- roofline
SMEM_B_PER_CLK_SM = 128      # shared-memory bandwidth per SM (B200_PROFILING.md / B300_MICROARCH.md)
# each split term reads M_a(i,I_a) and B(i,I_p) from shared memory: 2 x element bytes
FMA_PER_CLK_SM = 128         # fp32 FMA lanes per SM


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return {"hbm_gbs": 6650.0}, "of fallback (B200_PROFILING.md: 6.65 TB/s)"


def _traffic(args):
    """ncu DRAM bytes per launch of THIS source tree (profiles/ncu_traffic.json, stamped with
    build.source_hash()); None when the committed capture belongs to other sources."""
    from paper_2009_11665_b200.build import source_hash
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return None, "no profiles/ncu_traffic.json"
    rec = tr.get(f"{args.template}/{args.precision}/{args.layout}/scale{args.scale}")
    if not isinstance(rec, dict):
        return None, "no capture for this configuration"
    if rec.get("src_hash") != source_hash():
        return None, f"capture {rec.get('src_hash')} is for other sources than {source_hash()} (re-run tools/traffic.sh)"
    return rec, rec.get("source")


def roofline(args, prof, recs, plan):
    """Dominant kernel class: SURVEY §8(d) algorithmic bytes per launch (the plan's per-step
    alg_bytes: useful gather + CSR + M_a + plain-width output) / the class's mean CUDA-event
    launch time on the launching stream, against MEASURED_PEAKS hbm_gbs.  Also: the
    implemented layout's bytes (impl), ncu DRAM traffic of this source tree, a per-step
    table of one colouring (mean over the timed colourings), and the eMA terms/s of the
    GENERAL steps against the shared-memory roof."""
    peaks, psrc = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    dom = max(("step", "top", "hist"), key=lambda c: prof[c]["ms"])
    mine = [r for r in recs if r["cls"] == dom]
    ms = sum(r["ms"] for r in mine)
    alg = sum(r["alg_bytes"] for r in mine)
    impl = sum(r["impl_bytes"] for r in mine)
    nl = max(len(mine), 1)
    achieved = alg / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    tr, tsrc = _traffic(args)
    traffic = tr["per_class_dram_bytes_per_launch"].get(dom) if tr else None
    rf = {"bound": "hbm", "kernel": {"step": "astep_kernel (fused SpMM + eMA, non-top steps)",
                                     "top": "top step (fused gather + dot product)", "hist": "bucket/hist"}[dom],
          "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
          "traffic": traffic, "traffic_source": tsrc,
          "alg_bytes_per_launch": alg / nl, "launches": len(mine), "ms_per_launch": ms / nl,
          "impl_bytes_per_launch": impl / nl, "impl_over_alg": impl / alg if alg else None,
          "frac_impl": (impl / (ms / 1e3) / 1e9) / peak if ms > 0 else None,
          "frac_dram": (traffic / (ms / nl / 1e3) / 1e9) / peak if (traffic and ms > 0) else None,
          "peak_source": psrc,
          "definition": "achieved = SURVEY 8(d) algorithmic bytes (plan alg_bytes: anchored useful gather "
                        "nnz*(k-1)/k*C(k-2,p-1)*E + CSR 4*nnz + row metadata + M_a + output at plain width "
                        "C(k-1,s-1)*E) / mean launch time (CUDA events); frac_impl uses the implemented "
                        "layout's bytes; frac_dram uses ncu DRAM bytes of this source tree"}
    # per-step table: records in launch order; a colouring starts at each "color" record
    cols, cur = [], None
    for r in recs:
        if r["cls"] == "color":
            cur = []
            cols.append(cur)
        if cur is not None:
            cur.append(r)
    steps_tab = []
    if cols:
        L = len(cols[0])
        same = [c for c in cols if len(c) == L]
        names = ["color", "bucket" if args.layout != "dense" else "hist"]
        nch = -(-plan.get("n_rows", 0) // plan["split_rows"]) if plan.get("split_rows") else 0
        for st in plan["steps"]:
            nm = (f"s={st['s']}={st['a']}+{st['p']}{' top' if st['top'] else ''}"
                  f"{' self' if st.get('self') else ''}")
            if st.get("split_ema") and nch:  # split pipeline: a gather and an eMA launch per chunk
                names += [nm + " (split: gather)", nm + " (split: eMA)"] * nch
            else:
                names.append(nm)
        names.append("reduce")
        agg = {}
        for q in range(L):
            nm = names[q] if len(names) == L else same[0][q]["cls"] + f"#{q}"
            a = agg.setdefault(nm, {"launch": nm, "ms": 0.0, "alg_GB": 0.0, "impl_GB": 0.0, "ema_terms": 0.0,
                                    "launches": 0})
            a["ms"] += statistics.mean(c[q]["ms"] for c in same)
            a["alg_GB"] += same[0][q]["alg_bytes"] / 1e9
            a["impl_GB"] += same[0][q]["impl_bytes"] / 1e9
            a["ema_terms"] += same[0][q]["ema_terms"]
            a["launches"] += 1
        for a in agg.values():
            a["alg_frac"] = a["alg_GB"] / (a["ms"] / 1e3) / peak if a["ms"] > 0 and a["alg_GB"] > 0 else None
            if a["ema_terms"] > 0 and a["ms"] > 0:
                a["ema_terms_per_s"] = a["ema_terms"] / (a["ms"] / 1e3)
            steps_tab.append(a)
    ema = None
    gen = [a for a in steps_tab if a.get("ema_terms_per_s")]
    if gen:
        smem_roof = 148 * SMEM_B_PER_CLK_SM * sm_mhz * 1e6 / (2 * plan["elem"])
        fma_roof = 148 * FMA_PER_CLK_SM * sm_mhz * 1e6
        top = max(gen, key=lambda a: a["ema_terms"])
        rate = top["ema_terms_per_s"]
        ema = {"step": top["launch"], "terms_per_colouring": top["ema_terms"], "ms_per_colouring": top["ms"],
               "terms_per_s": rate, "smem_roof_terms_per_s": smem_roof, "frac_smem": rate / smem_roof,
               "fma_roof_per_s": fma_roof, "frac_fma": rate / fma_roof,
               "note": "the GENERAL step with the most split terms; its eMA launches' CUDA-event time (split "
                       "pipeline: the eMA launches alone; fused: gather included, a lower bound on the eMA rate). "
                       "smem roof = 148 SMs x 128 B/clk x SM clock / (2 operands x element bytes)"}
    return rf, steps_tab, ema


def _spawn_ranks(args):
    """--gpus N without torchrun: relaunch this command under torch.distributed.run
    (one rank per GPU, rendezvous on 127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    dev = _setup_dist(world, local)

    import paper_2009_11665_b200 as sg
    from paper_2009_11665_b200.build import build
    from sg2v_inputs import degree_stats, rmat_1m_like

    build()
    k, edges = _template(args.template)
    g = _load_graph(args)
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

    overflow = []  # colourings whose F32 count overflowed (EOVERFLOW), reported in the line

    def count(GG, n_iter, off, stride=1, wsp=None):
        # one DP run per colouring: EOVERFLOW (an F32 table entry overflowed) is recorded, not retried
        wsp = ws if wsp is None else wsp
        r = sg.count(GG, T, n_iter=n_iter, seed=args.seed, iter_offset=off, iter_stride=stride,
                     precision=args.precision, workspace=wsp, layout=args.layout, allow_overflow=True)
        if sg.sg2v.LAST_STATUS == sg.sg2v.EOVERFLOW:
            overflow.append(off)
        return r

    # warm-up (untimed)
    for t in range(args.warmup):
        count(G, 1, colouring(t))
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
        est, c = count(G, args.steps, colouring(args.warmup), world)
        for t in range(args.steps):
            counts[rank + world * t] = float(c[t])
        if world > 1:
            dist.all_reduce(counts)  # NCCL: per-colouring counts of every rank
        ev1.record(stream)
        torch.cuda.synchronize()
    prof = sg.profile_read()
    launches_rec = sg.profile_read_launches()
    n_kernels = sg.profile_kernel_count()  # every kernel of libsg2v launched in the timed region
    sg.profile_enable(False)
    dev_s = ev0.elapsed_time(ev1) / 1e3
    t_max = torch.tensor([dev_s], dtype=torch.float64, device=_dist_device())
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total = world * args.steps
    value = float(t_max.item()) / total

    # ---- e2e: the public API from pinned HOST buffers, copies inside the timed region ----
    # (the workspace is requested inside the timed region too, as a user's call does;
    # torch's caching allocator hands back the same block after the first step)
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    del G
    ws_bytes = ws.nbytes
    ws = None  # (count() looks `ws` up at call time: the timed e2e steps allocate their own)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(e2e_steps):
        Ge = sg.graph_load_csr(g.n, ro_h.numpy(), ci_h.numpy())
        wse = sg.Workspace(ws_bytes)
        count(Ge, 1, colouring(args.warmup + args.steps + t), wsp=wse)  # includes D2H of the count
        Ge.free()
        del wse
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
    rf, steps_tab, ema = roofline(args, prof, launches_rec, plan)
    launches = n_kernels
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
        "status": "EOVERFLOW" if overflow else "OK", "overflowed_calls": len(overflow),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(g.nbytes()),
                "d2h_bytes_per_step": 8},
        "gpu_launches": int(launches),
        "kernel_ms_per_step": {kk: v["ms"] / args.steps for kk, v in prof.items()},
        "roofline": rf,
        "steps_per_colouring": steps_tab,
        "clocks": clocks,
    }
    if ema:
        line["ema"] = ema
    if world == 1 and not args.no_cpu_baseline:
        per, desc, cores = cpu_sample(args, k, edges, g.n, g.nnz, steps=1, target_s=20.0)
        line["cpu_baseline"] = {"value": per[0], "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        full = full_graph_oracle_record(args.template, args.scale)
        if full:
            line["cpu_baseline"]["full_graph_measured"] = full
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_vertex(args):
    """--mode vertex: 1D vertex partition of every table across the ranks (capacity mode,
    SURVEY §8(e) V).  Rows are dealt to the rank blocks by degree (sg2v_partition_relabel,
    colours keyed by the input ids) unless --no-balance."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = _setup_dist(world, local)
    import paper_2009_11665_b200 as sg
    from paper_2009_11665_b200.build import build
    from sg2v_inputs import degree_stats

    build()
    k, edges = _template(args.template)
    g = _load_graph(args)
    stats = degree_stats(g)
    b, nl = sg.partition_rows(g.n, rank, world)
    if args.no_balance:
        ro_all, ci_all, oon = g.row_offsets, g.col_indices, None
    else:
        oon, ro_all, ci_all = sg.partition_relabel(g.row_offsets, g.col_indices, world)
    ro = np.ascontiguousarray(ro_all[b:b + nl + 1] - ro_all[b])
    ci = np.ascontiguousarray(ci_all[ro_all[b]:ro_all[b + nl]])
    uid = [sg.Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    comm = sg.Comm.nccl(uid[0], rank, world)

    def load():
        G = sg.graph_load_partition(g.n, b, nl, ro, ci)
        if oon is not None:
            sg.graph_set_vertex_ids(G, oon)
        return G

    Gp = load()
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
    n_kernels = sg.profile_kernel_count()  # every kernel of libsg2v launched in the timed region
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
        Ge = load()
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
        peaks, psrc = _peaks()
        peak = float(peaks.get("hbm_gbs", 6650.0))
        dom = "step"
        achieved = prof[dom]["bytes"] / (prof[dom]["ms"] / 1e3) / 1e9 if prof[dom]["ms"] > 0 else 0.0
        launches = n_kernels
        # NVLink: bytes each rank receives per colouring in the whole-row exchange (the
        # plain anchored plan on nl rows: (W-1)·nl·ldp·E per gather step), over the
        # colouring's time — a lower bound on the link rate while exchanging
        plain = sg.plan_describe_n(-(-g.n // world), max(g.nnz // world, 1), T, args.precision, "anchored_plain")
        E = plain["elem"]
        nlr = -(-g.n // world)
        recv = sum((world - 1) * nlr * st["ldp"] * E for st in plain["steps"] if st["src"] == "gather")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
                "config": {"workload": _workload_name(args, g), "template": args.template, "k": k,
                           "precision": args.precision, "layout": "anchored (plain tables)", "graph": stats,
                           "parallelism": f"vertex{world}", "rows_per_rank": nl, "col_tile": args.col_tile,
                           "balanced_relabel": oon is not None,
                           "l2": "inputs larger than L2; no flush"},
                "estimate": est, "colorful_first": float(c[0]),
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(ro.nbytes + ci.nbytes),
                        "d2h_bytes_per_step": 8},
                "gpu_launches": int(launches),
                "kernel_ms_per_step": {kk: v["ms"] / args.steps for kk, v in prof.items()},
                "roofline": {"bound": "hbm", "kernel": "step (rank 0)", "achieved": achieved,
                             "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                             "peak_source": psrc},
                "nvlink": {"recv_bytes_per_colouring_per_rank": recv,
                           "achieved_GBps_lower_bound": recv / value / 1e9 if value > 0 else 0.0,
                           "peak_GBps": 900.0, "frac_lower_bound": recv / value / 1e9 / 900.0 if value > 0 else 0.0},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = _args()
    world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world is None:
        return _spawn_ranks(args)
    if world is not None and int(world) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "vertex":
        return run_vertex(args)
    return run_sg2v(args)


if __name__ == "__main__":
    sys.exit(main())
