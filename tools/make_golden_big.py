"""Writes tests/golden/big_configs.json: oracle colorful counts (U64 residue, fp64 value,
fp64 max intermediate) for the BASELINE.json configs the CPU oracle can finish.

Calls ONLY oracle/ and sg2v_inputs/ (no CUDA path).  Colouring: COLOR(seed=1, j=0).
    python tools/make_golden_big.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from sg2v_inputs import BIG_GRAPHS, TEMPLATES, degree_stats  # noqa: E402

CASES = [("rmat1m", "u5-2"), ("rmat1m", "u7-2"), ("rmat1m", "u12-1"),
         ("miami", "u5-2"), ("miami", "u7-2"), ("orkut", "u10-2")]


def main():
    out_path = os.path.join(ROOT, "tests", "golden", "big_configs.json")
    res = {"source": "tools/make_golden_big.py: oracle/sg2v_oracle.c two-stage DP (SPEC-rule chain, root 0), "
                     "colouring COLOR(seed=1, j) of SURVEY §8(c) step 1; graphs from sg2v_inputs (SURVEY §8(d) D2-D4)",
           "cases": []}
    graphs = {}
    for gname, tname in CASES:
        if gname not in graphs:
            graphs = {gname: BIG_GRAPHS[gname]()}
        g = graphs[gname]
        e = TEMPLATES[tname]
        k = 1 + max(max(x) for x in e)
        for j in (0,):
            cols = O.colors(1, j, g.n, k)
            t0 = time.time()
            u = O.count(g, k, e, cols)
            f, vmax = O.count(g, k, e, cols, arith=O.ARITH_F64)
            dt = time.time() - t0
            rec = {"graph": gname, "graph_stats": degree_stats(g), "template": tname, "k": k, "seed": 1, "j": j,
                   "colorful_u64": str(u), "colorful_f64": f, "max_intermediate": vmax,
                   "oracle_seconds": dt, "threads": O.get_threads()}
            print(json.dumps(rec), flush=True)
            res["cases"].append(rec)
            with open(out_path, "w") as fh:
                json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
