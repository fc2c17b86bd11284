"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
register, warp-row and bulk-staged gathers (SG2V_BULK_MIN=1 forces the bulk kernel onto narrow rows too,
SG2V_RING=1 the bulk-copy warp rings), 512-thread V-row eMA (u17 in U64),
CTA-per-heavy-row, V-row eMA, the split eMA pipeline, dense layout, vertex mode (tiles and
whole rows, world 1).  Checks U64 counts against the oracle so a silent corruption fails too."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_11665_b200 as sg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from sg2v_inputs import TEMPLATES, csr_from_edges, erdos_renyi  # noqa: E402

torch.cuda.set_device(0)
n = 2600
rng = np.random.default_rng(0)
u = np.concatenate([np.zeros(n - 100, np.int64), rng.integers(1, n, 6000)])   # one hub of degree ~2500
v = np.concatenate([np.arange(1, n - 99), rng.integers(1, n, 6000)])
graphs = {"hub": csr_from_edges(n, u, v), "er": erdos_renyi(1500, 7000, seed=3)}
bad = 0
for gname, g in graphs.items():
    G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices, validate=True)
    for name in ("u5-2", "u7-2", "u12-1", "u13-2", "u15-1", "u17"):
        e = TEMPLATES[name]
        k = 1 + max(max(x) for x in e)
        want = O.count(g, k, e, O.colors(2, 0, g.n, k))
        T = sg.template_build(k, e)
        for layout in ("anchored", "anchored_plain", "dense") if k <= 7 else ("anchored", "anchored_plain"):
            _, c = sg.count(G, T, n_iter=1, seed=2, precision="u64", layout=layout)
            ok = int(c[0]) == want
            bad += not ok
            print(gname, name, layout, "ok" if ok else f"MISMATCH {int(c[0])} != {want}", flush=True)
        if gname == "er":  # vertex mode, world 1: whole rows and column tiles
            comm = sg.Comm.nccl(sg.Comm.unique_id(), 0, 1)
            Gp = sg.graph_load_partition(g.n, 0, g.n, g.row_offsets, g.col_indices)
            for tile in (0, 8):
                _, c = sg.count(Gp, T, n_iter=1, seed=2, precision="u64", comm=comm, col_tile=tile)
                ok = int(c[0]) == want
                bad += not ok
                print(gname, name, f"vertex tile={tile}", "ok" if ok else "MISMATCH", flush=True)
            comm.free()
torch.cuda.synchronize()
print("sanitize_run:", "PASS" if bad == 0 else f"{bad} MISMATCHES")
sys.exit(1 if bad else 0)
