"""Where does the e2e overhead go? (graph upload / order / count / free)"""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_2009_11665_b200 as sg
from sg2v_inputs import rmat_1m_like, TEMPLATES
g = rmat_1m_like()
torch.cuda.set_device(0)
ro = torch.from_numpy(g.row_offsets).pin_memory(); ci = torch.from_numpy(g.col_indices).pin_memory()
e = TEMPLATES['u15-1']; T = sg.template_build(15, e)
G0 = sg.graph_load_csr(g.n, ro.numpy(), ci.numpy())
ws = sg.Workspace(sg.workspace_bytes(G0, T, 'f32'))
sg.count(G0, T, n_iter=1, seed=1, precision='f32', workspace=ws)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    G = sg.graph_load_csr(g.n, ro.numpy(), ci.numpy()); torch.cuda.synchronize(); t1 = time.perf_counter()
    sg.count(G, T, n_iter=1, seed=1, iter_offset=it, precision='f32', workspace=ws); torch.cuda.synchronize(); t2 = time.perf_counter()
    G.free(); torch.cuda.synchronize(); t3 = time.perf_counter()
    sg.count(G0, T, n_iter=1, seed=1, iter_offset=it, precision='f32', workspace=ws); torch.cuda.synchronize(); t4 = time.perf_counter()
    print('load %.1f ms  count(new G) %.1f ms  free %.1f ms  count(resident G) %.1f ms' % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3), flush=True)
