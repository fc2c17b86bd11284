"""One template/precision on RMAT-1M-like, for ncu captures (not a bench)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2009_11665_b200 as sg
from sg2v_inputs import rmat_1m_like, TEMPLATES
name, prec = sys.argv[1], sys.argv[2]
layout = sys.argv[3] if len(sys.argv) > 3 else "anchored"
n_iter = int(sys.argv[4]) if len(sys.argv) > 4 else 1
scale = int(sys.argv[5]) if len(sys.argv) > 5 else 20
g = rmat_1m_like(scale=scale)
torch.cuda.set_device(0)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
T = sg.template_build(k, e)
d = sg.plan_describe(G, T, prec, layout)
print([(s['s'], s['a'], s['p'], s['gt'], s['comb'][0]) for s in d['steps']], flush=True)
ws = sg.Workspace(d['workspace_bytes'])
est, c = sg.count(G, T, n_iter=n_iter, seed=1, precision=prec, workspace=ws, allow_overflow=True, layout=layout)
torch.cuda.synchronize()
print(name, prec, layout, list(c))
