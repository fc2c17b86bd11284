"""Writes oracle goldens for the BASELINE.json full-size configs: colorful counts (U64
residue, fp64 value, fp64 max intermediate), wall time per arithmetic, and optionally
per-vertex values on a seeded sample of rows.

Calls ONLY oracle/ and sg2v_inputs/ (no CUDA path).  Colouring: COLOR(seed=1, j).

    python tools/make_golden_big.py                      # the default CASES -> tests/golden/big_configs.json
    python tools/make_golden_big.py --case rmat1m:u15-1:0:u64,f64 --case rmat1m:u15-1:5:u64 \
        --rows 4096 --out gpurun_out/golden_u15.json     # the bench workload (run on the GPU box's host:
                                                          # 196 GB RAM, the oracle's peak is ~109 GB)

Row sample (--rows R): the 64 highest-degree vertices plus R-64 uniform picks
(numpy default_rng(20091166)), sorted.  Per-vertex values count embeddings with the
template ROOT mapped to the vertex, so they are recorded with the oracle's root
(--root, default 0) and the GPU side must be rooted there too.
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from sg2v_inputs import BIG_GRAPHS, TEMPLATES, degree_stats  # noqa: E402

CASES = ["rmat1m:u5-2:0:u64,f64", "rmat1m:u7-2:0:u64,f64", "rmat1m:u12-1:0:u64,f64",
         "miami:u5-2:0:u64,f64", "miami:u7-2:0:u64,f64", "orkut:u10-2:0:u64,f64"]


def host_info():
    info = {"nproc": os.cpu_count(), "threads": O.get_threads(), "machine": platform.machine()}
    try:
        info["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
        info["mem_total_GB"] = int([l.split()[1] for l in open("/proc/meminfo") if l.startswith("MemTotal")][0]) / 1e6
    except Exception:
        pass
    return info


def sample_rows(g, r):
    deg = np.diff(g.row_offsets)
    hubs = np.argsort(-deg, kind="stable")[:64]
    rng = np.random.default_rng(20091166)
    rest = rng.choice(g.n, size=max(r - 64, 0), replace=False)
    return np.unique(np.concatenate([hubs, rest])).astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", help="graph:template:j:arith[,arith]")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--root", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "big_configs.json"))
    a = ap.parse_args()
    cases = a.case or CASES
    res = {"source": "tools/make_golden_big.py: oracle/sg2v_oracle.c two-stage DP (SPEC-rule chain, root "
                     f"{a.root}), colouring COLOR(seed=1, j) of SURVEY §8(c) step 1; graphs from sg2v_inputs "
                     "(SURVEY §8(d) D2-D4)",
           "host": host_info(), "cases": []}
    if os.path.exists(a.out):
        try:
            old = json.load(open(a.out))
            res["cases"] = old.get("cases", [])
        except Exception:
            pass
    graphs = {}
    for spec in cases:
        gname, tname, j, ariths = spec.split(":")
        j = int(j)
        if gname not in graphs:
            graphs = {gname: BIG_GRAPHS[gname]()}
        g = graphs[gname]
        e = TEMPLATES[tname]
        k = 1 + max(max(x) for x in e)
        rows = sample_rows(g, a.rows) if a.rows else None
        cols = O.colors(1, j, g.n, k)
        rec = {"graph": gname, "graph_stats": degree_stats(g), "template": tname, "k": k, "seed": 1, "j": j,
               "root": a.root, "threads": O.get_threads(), "host": res["host"]}
        for ar in ariths.split(","):
            t0 = time.time()
            if ar == "u64":
                out = O.count(g, k, e, cols, root=a.root, rows=rows is not None)
                u, ru = out if rows is not None else (out, None)
                rec["colorful_u64"] = str(u)
                rec["oracle_seconds_u64"] = time.time() - t0
                if ru is not None:
                    rec["rows"] = rows.tolist()
                    rec["rows_u64"] = [str(int(x)) for x in ru[rows]]
            else:
                out = O.count(g, k, e, cols, root=a.root, arith=O.ARITH_F64, rows=rows is not None)
                f, vmax = out[0], out[1]
                rec["colorful_f64"] = f
                rec["max_intermediate"] = vmax
                rec["oracle_seconds_f64"] = time.time() - t0
                if rows is not None:
                    rec["rows"] = rows.tolist()
                    rec["rows_f64"] = [float(x) for x in out[2][rows]]
            print(json.dumps({kk: v for kk, v in rec.items() if not kk.startswith("rows")}), flush=True)
        rec["oracle_seconds"] = rec.get("oracle_seconds_u64", 0.0) + rec.get("oracle_seconds_f64", 0.0)
        res["cases"] = [c for c in res["cases"] if not (c["graph"] == gname and c["template"] == tname and
                                                        c["j"] == j and c.get("root", 0) == a.root)]
        res["cases"].append(rec)
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
