"""Treelet distribution timing: all trees of size k on RMAT-1M-like, batch vs one by one."""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_2009_11665_b200 as sg
from sg2v_inputs import rmat_1m_like, all_trees
k = int(sys.argv[1]) if len(sys.argv) > 1 else 7
prec = sys.argv[2] if len(sys.argv) > 2 else 'f64'
g = rmat_1m_like()
torch.cuda.set_device(0)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
Ts = [sg.template_build(k, e) for e in all_trees(k)]
sg.count_batch(G, Ts, n_iter=1, seed=1, precision=prec)
torch.cuda.synchronize(); t = time.perf_counter()
est, col = sg.count_batch(G, Ts, n_iter=2, seed=1, iter_offset=1, precision=prec)
torch.cuda.synchronize(); tb = (time.perf_counter() - t) / 2
t = time.perf_counter()
for T in Ts:
    sg.count(G, T, n_iter=2, seed=1, iter_offset=1, precision=prec)
torch.cuda.synchronize(); ts = (time.perf_counter() - t) / 2
print(f'k={k} trees={len(Ts)} batch {tb:.3f} s/colouring  separate {ts:.3f} s/colouring  speedup {ts/tb:.2f}')
