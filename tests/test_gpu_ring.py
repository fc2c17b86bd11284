"""GPU parity of the warp-per-row gathers (astep_wrow_kernel: registers across colour
buckets; astep_ring_kernel: self-fed rings of bulk copies) vs the oracle.

They run the narrow and medium gather steps (SpMM stage 1, fused with the eMA /
projected stores of stage 2).  Rows with >= 2048 neighbours are split over the W
warps of a CTA (every W-th neighbour, W private B copies added in a fixed order) — a graph
with several such hubs exercises that path, the rest of the rows the warp-per-row path
(the ring's issue cursor running across rows; the bucket kernel's CTA-per-row path).  Each
configuration runs in its own subprocess (the knobs are read once per process):
per-vertex values in U64 bit-exact against the oracle rooted where the planner rooted,
F32 totals within rel 1e-4 (BASELINE.json north_star).
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from sg2v_inputs import TEMPLATES, csr_from_edges  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ("u5-2", "u7-2", "u12-1", "u14-2", "u15-1")
SEED, J = 9, 2


def hub_graph():
    """n = 9000: hubs of degree ~2100 / 2600 / 4100 / 6000 (>= 2^11: the CTA-team path) on
    a sparse random background (the warp-per-row path, many rows of degree 0-20)."""
    n = 9000
    rng = np.random.default_rng(23)
    us, vs = [], []
    for h, d in ((0, 2100), (1, 2600), (2, 4100), (3, 6000)):
        nb = rng.choice(np.arange(4, n), size=d, replace=False)
        us.append(np.full(d, h))
        vs.append(nb)
    us.append(rng.integers(0, n, 30000))
    vs.append(rng.integers(0, n, 30000))
    return csr_from_edges(n, np.concatenate(us), np.concatenate(vs))


_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2009_11665_b200 as sg
from sg2v_inputs import TEMPLATES
from tests.test_gpu_ring import hub_graph, SEED, J
torch.cuda.set_device(0)
g = hub_graph()
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices, validate=True)
out = {}
for name in sys.argv[1].split(","):
    e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    for layout in ("anchored", "anchored_plain"):
        rv = torch.zeros(g.n, dtype=torch.int64, device="cuda")
        _, c = sg.count(G, T, n_iter=1, seed=SEED, iter_offset=J, precision="u64", row_values=rv, layout=layout)
        out[f"{name}/{layout}/rows"] = rv.cpu().numpy().view(np.uint64)
        out[f"{name}/{layout}/root"] = np.array([sg.plan_describe(G, T, "u64", layout)["root"]])
        _, c = sg.count(G, T, n_iter=1, seed=SEED, iter_offset=J, precision="f32", allow_overflow=True, layout=layout)
        out[f"{name}/{layout}/f32"] = np.array([float(c[0])])
np.savez(sys.argv[2], **{k.replace("/", "__"): v for k, v in out.items()})
""" % ROOT

CONFIGS = [{}, {"SG2V_WROW_MIN": "1"}, {"SG2V_WROW_U": "2"}, {"SG2V_WROW_U": "4"}, {"SG2V_WROW_U": "3"},
           {"SG2V_WROW": "0", "SG2V_RING": "1"}, {"SG2V_WROW": "0", "SG2V_RING": "1", "SG2V_RING_KB": "1"},
           {"SG2V_WROW": "0", "SG2V_RING": "1", "SG2V_RING_MAX": "256", "SG2V_RING_KB": "2"},
           {"SG2V_WROW": "0"}, {"SG2V_WROW": "0", "SG2V_HEAVY": "0"}, {"SG2V_NARROW": "0"}]


@pytest.fixture(scope="module")
def want(oracle):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return {}


def _run(oracle, want, tmp_path, cfg, names):
    g = hub_graph()
    assert (np.diff(g.row_offsets) >= 2048).sum() >= 4
    f = tmp_path / "rows.npz"
    env = dict(os.environ, **cfg)
    p = subprocess.run([sys.executable, "-c", _SCRIPT, ",".join(names), str(f)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    got = np.load(f)
    for name in names:
        e = TEMPLATES[name]
        k = 1 + max(max(x) for x in e)
        cols = oracle.colors(SEED, J, g.n, k)
        for layout in ("anchored", "anchored_plain"):
            rho = int(got[f"{name}__{layout}__root"][0])
            key = (name, rho)
            if key not in want:
                want[key] = (oracle.count(g, k, e, cols, root=rho, rows=True),
                             oracle.count(g, k, e, cols, arith=oracle.ARITH_F64)[0])
            (tot, rows), f64 = want[key]
            r = got[f"{name}__{layout}__rows"]
            assert np.array_equal(r, rows), (cfg, name, layout, np.flatnonzero(r != rows)[:10])
            f32 = float(got[f"{name}__{layout}__f32"][0])
            assert math.isclose(f32, f64, rel_tol=1e-4), (cfg, name, layout, f32, f64)


@pytest.mark.parametrize("cfg", CONFIGS, ids=[",".join(f"{a}={b}" for a, b in d.items()) or "default" for d in CONFIGS])
def test_ring_gather_vs_oracle(oracle, want, tmp_path, cfg):
    _run(oracle, want, tmp_path, cfg, NAMES)


# eMA-heavy GENERAL steps whose V = 4 interleaved rows fill the SM's shared memory (U64 /
# F64 rows of u17's 10 = 5 + 5: 198 KB) run as one 512-thread CTA; SG2V_EMA512=0 keeps the
# 256-thread CTA.  SG2V_SPLIT=0: the same steps fused (gather + V-row eMA in one kernel).
@pytest.mark.parametrize("cfg", [{}, {"SG2V_EMA512": "0"}, {"SG2V_EMA512": "2"}, {"SG2V_EMA512": "3"}, {"SG2V_SPLIT": "0"}],
                         ids=["default", "ema256", "ema1024", "emaV8", "fused"])
def test_vrow_ema_512_vs_oracle(oracle, want, tmp_path, cfg):
    _run(oracle, want, tmp_path, cfg, ("u17", "u16-2"))
