"""Exact cross-check of kernel configurations on RMAT-1M-like (U64 residues must agree)."""
import json, os, sys
import torch
sys.path.insert(0, ".")
import paper_2009_11665_b200 as sg
from sg2v_inputs import TEMPLATES, rmat_1m_like
g = rmat_1m_like()
torch.cuda.set_device(0)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
for name in sys.argv[2].split(","):
    e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    out = {"tag": sys.argv[1], "template": name}
    for prec in sys.argv[3].split(","):
        d = sg.plan_describe(G, T, prec)
        ws = sg.Workspace(d["workspace_bytes"])
        _, c = sg.count(G, T, n_iter=1, seed=1, precision=prec, workspace=ws, allow_overflow=True)
        out[prec] = int(c[0]) if prec == "u64" else float(c[0])
        del ws; torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
