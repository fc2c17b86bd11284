"""Quick timing exploration on the GPU box (not part of the bench contract)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_11665_b200 as sg
from sg2v_inputs import rmat_1m_like, TEMPLATES, degree_stats
t = time.time(); g = rmat_1m_like(); print('gen', time.time() - t, degree_stats(g), flush=True)
torch.cuda.set_device(0)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
for name in sys.argv[1].split(','):
    e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    for prec in sys.argv[2].split(','):
        d = sg.plan_describe(G, T, prec)
        try:
            ws = sg.Workspace(d['workspace_bytes'])
            sg.count(G, T, n_iter=1, seed=1, precision=prec, workspace=ws, allow_overflow=True)
            torch.cuda.synchronize()
            sg.profile_enable(True)
            s = torch.cuda.Event(enable_timing=True); f = torch.cuda.Event(enable_timing=True)
            s.record(); est, c = sg.count(G, T, n_iter=2, seed=1, iter_offset=1, precision=prec, workspace=ws, allow_overflow=True); f.record(); torch.cuda.synchronize()
            p = sg.profile_read(); sg.profile_enable(False)
            ms = s.elapsed_time(f) / 2
            print(json.dumps({'t': name, 'prec': prec, 'root': d['root'], 'ws_GB': d['workspace_bytes'] / 1e9, 's_per_col': ms / 1e3,
                              'colorful': [float(x) for x in c], 'model_s': d['model_seconds'],
                              'prof': {kk: (v['launches'], round(v['ms'], 2), round(v['bytes'] / max(v['ms'], 1e-9) / 1e6, 1)) for kk, v in p.items()}}), flush=True)
            del ws
        except Exception as ex:
            print(name, prec, 'ERR', ex, flush=True)
        torch.cuda.empty_cache()
