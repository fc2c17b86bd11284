"""Seconds per colouring for the u12–u17 family on RMAT-1M-like (BASELINE metric),
1xB200, CUDA events, 2 warm-up + 3 timed colourings; F32 (paper precision) and, where
F32 overflows, F64.  One JSON line per (template, precision)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_11665_b200 as sg  # noqa: E402
from sg2v_inputs import TEMPLATES, rmat_1m_like  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else \
    ["u12-1", "u13-1", "u14-1", "u15-1", "u15-2", "u16-1", "u17-1", "u13-2", "u14-2", "u16-2", "u17"]
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6535.4)
g = rmat_1m_like()
torch.cuda.set_device(0)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices)
for name in names:
    e = TEMPLATES[name]
    k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    for prec in ("f32", "f64"):
        try:
            d = sg.plan_describe(G, T, prec)
            ws = sg.Workspace(d["workspace_bytes"])
            sg.count(G, T, n_iter=2, seed=1, precision=prec, workspace=ws, allow_overflow=True)
            torch.cuda.synchronize()
            sg.profile_enable(True)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            est, c = sg.count(G, T, n_iter=3, seed=1, iter_offset=2, precision=prec, workspace=ws,
                              allow_overflow=True)
            s1.record()
            torch.cuda.synchronize()
            p = sg.profile_read()
            recs = sg.profile_read_launches()
            sg.profile_enable(False)
            gen = [r for r in recs if r["ema_terms"] > 0]
            gms = sum(r["ms"] for r in gen)
            terms = sum(r["ema_terms"] for r in gen)
            # shared-memory roof of the eMA: 148 SMs x 128 B/clk / 8 B per term (two fp32 operands)
            ema_roof = 148 * 128 * 1965e6 / 8
            dt = s0.elapsed_time(s1) / 3e3
            b = p["step"]["bytes"] + p["top"]["bytes"]
            ms = p["step"]["ms"] + p["top"]["ms"]
            finite = all(x == x and abs(x) != float("inf") for x in c)
            print(json.dumps({"template": name, "k": k, "precision": prec, "s_per_colouring": dt,
                              "steps": len(d["steps"]), "root": d["root"], "workspace_GB": d["workspace_bytes"] / 1e9,
                              "alg_GBps": b / ms / 1e6 if ms else 0, "frac": b / ms / 1e6 / peak if ms else 0,
                              "impl_frac": sum(r["impl_bytes"] for r in recs if r["cls"] in ("step", "top")) / ms / 1e6 / peak if ms else 0,
                              "ema_terms_per_s": terms / gms * 1e3 if gms else None,
                              "ema_frac_smem": terms / gms * 1e3 / ema_roof if gms else None,
                              "ema_ms": gms / 3,
                              "finite": finite, "colorful0": float(c[0])}), flush=True)
            del ws
            torch.cuda.empty_cache()
            if finite:
                break
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"template": name, "precision": prec, "error": str(ex)}), flush=True)
