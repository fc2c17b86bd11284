"""Skew sweep: the paper claims comparable SubGraph2Vec time
regardless of the degree skew (RMAT K=3/5/8 rows of Table III).
RMAT scale 20 with ~1.05e8 drawn edges, a in {0.40, 0.45, 0.50, 0.57}
(b = c = 0.4(1-a), d = 0.2(1-a)); seconds per colouring (CUDA events, 3 timed
after 2 warm-up) for u12-1 F32, anchored.  Prints one JSON line per a."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_11665_b200 as sg  # noqa: E402
from sg2v_inputs import TEMPLATES, degree_stats, rmat  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "u12-1"
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
e = TEMPLATES[name]
k = 1 + max(max(x) for x in e)
torch.cuda.set_device(0)
for a in (0.40, 0.45, 0.50, 0.57):
    g = rmat(20, 105_000_000, a, 0.4 * (1 - a), 0.4 * (1 - a), seed=1, perm_seed=7)
    G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
    T = sg.template_build(k, e)
    ws = sg.Workspace(sg.workspace_bytes(G, T, prec))
    sg.count(G, T, n_iter=2, seed=1, precision=prec, workspace=ws, allow_overflow=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    sg.count(G, T, n_iter=3, seed=1, iter_offset=2, precision=prec, workspace=ws, allow_overflow=True)
    s1.record()
    torch.cuda.synchronize()
    st = degree_stats(g)
    print(json.dumps({"template": name, "precision": prec, "a": a, "graph": st,
                      "s_per_colouring": s0.elapsed_time(s1) / 3e3,
                      "ns_per_edge": s0.elapsed_time(s1) / 3e3 / st["nnz"] * 1e9}), flush=True)
    del ws, G
    torch.cuda.empty_cache()
