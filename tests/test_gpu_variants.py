"""GPU parity of every kernel configuration the experiment knobs select, vs the oracle.

The launch heuristics (row-group width, U neighbours in flight, V rows per split-table
load, M_a staging, the L2 hub-row policy) pick among template instantiations of the same
fused SpMM+eMA step.  The defaults are covered by
test_gpu_parity.py; here each knob (read once per process) is set in a
fresh subprocess so every instantiation it reaches is checked against the oracle:
U64 bit-exact, F32 rel 1e-4 (BASELINE.json north_star).
"""
import json
import math
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from sg2v_inputs import TEMPLATES, rmat  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ("u15-1", "u14-2", "u12-1", "u7-2")
LAYOUTS = ("anchored", "anchored_plain")
SEED, J = 11, 3

# each entry: the environment of one subprocess (SG2V_TUNE values as in akernels.cu)
KNOBS = [
    {"SG2V_TUNE": "1"}, {"SG2V_TUNE": "2"}, {"SG2V_TUNE": "4"}, {"SG2V_TUNE": "5"},
    {"SG2V_TUNE": "6"}, {"SG2V_TUNE": "9"}, {"SG2V_TUNE": "16"},
    {"SG2V_VTPB": "0"}, {"SG2V_STAGE_KB": "0"}, {"SG2V_STAGE_KB": "4096"},
    {"SG2V_HINT": "0"}, {"SG2V_HOTFRAC": "0.00001"}, {"SG2V_HOTFRAC": "50"},
    {"SG2V_BULK": "0"}, {"SG2V_BULK_MIN": "1"}, {"SG2V_BULK_KB": "8"}, {"SG2V_HEAVY": "0"},
    {"SG2V_EMA_SCHED": "1"}, {"SG2V_SPLIT": "0"},
    {"SG2V_GTDIV": "4"}, {"SG2V_GTDIV": "16"}, {"SG2V_EMA512": "0"}, {"SG2V_WROW": "0"}, {"SG2V_WROW_MIN": "1"},
    {"SG2V_UNSTAGE": "1"}, {"SG2V_NARROW": "0"}, {"SG2V_BULK1": "1"}, {"SG2V_CORDER": "0"},
]

_SCRIPT = r"""
import json, sys, torch
import paper_2009_11665_b200 as sg
from sg2v_inputs import TEMPLATES, rmat
torch.cuda.set_device(0)
g = rmat(11, 24000, 0.57, 0.19, 0.19, seed=5)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices, validate=True)
out = {}
for name in sys.argv[1].split(","):
    e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    for layout in sys.argv[2].split(","):
        for prec in ("u64", "f32"):
            _, c = sg.count(G, T, n_iter=1, seed=%d, iter_offset=%d, precision=prec,
                            allow_overflow=True, layout=layout)
            out[f"{name}/{layout}/{prec}"] = int(c[0]) if prec == "u64" else float(c[0])
print(json.dumps(out))
""" % (SEED, J)


def _graph():
    return rmat(11, 24000, 0.57, 0.19, 0.19, seed=5)


@pytest.fixture(scope="module")
def want(oracle):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    g = _graph()
    res = {}
    for name in NAMES:
        e = TEMPLATES[name]
        k = 1 + max(max(x) for x in e)
        cols = oracle.colors(SEED, J, g.n, k)
        res[name] = (oracle.count(g, k, e, cols),
                     oracle.count(g, k, e, cols, arith=oracle.ARITH_F64)[0])
    return res


@pytest.mark.parametrize("knob", KNOBS, ids=[",".join(f"{a}={b}" for a, b in d.items()) for d in KNOBS])
def test_knob_configuration_vs_oracle(want, knob):
    env = dict(os.environ, **knob)
    p = subprocess.run([sys.executable, "-c", _SCRIPT, ",".join(NAMES), ",".join(LAYOUTS)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    for name in NAMES:
        wu, wf = want[name]
        for layout in LAYOUTS:
            assert got[f"{name}/{layout}/u64"] == wu, (knob, name, layout)
            f32 = got[f"{name}/{layout}/f32"]
            assert math.isclose(f32, wf, rel_tol=1e-4), (knob, name, layout, f32, wf)


# n % (row-group rows) != 0 with M_a not staged (SG2V_STAGE_KB=0) and the V-row eMA variants
# (V = 2/4 rows per group, GENERAL steps with many split terms): the inactive tail rows of
# the last slot must stay inside the block's shared memory (the zero-fill of
# an inactive row once ran past it).  Per-vertex values in U64 against the oracle.
_TAIL_SCRIPT = r"""
import sys, numpy as np, torch
import paper_2009_11665_b200 as sg
from sg2v_inputs import TEMPLATES, erdos_renyi
torch.cuda.set_device(0)
g = erdos_renyi(1001, 6000, seed=17)
G = sg.graph_load_csr(g.n, g.row_offsets, g.col_indices, validate=True)
out = {}
for name in sys.argv[1].split(","):
    e = TEMPLATES[name]; k = 1 + max(max(x) for x in e)
    T = sg.template_build(k, e)
    for layout in ("anchored", "anchored_plain"):
        rv = torch.zeros(g.n, dtype=torch.int64, device="cuda")
        _, c = sg.count(G, T, n_iter=1, seed=3, precision="u64", row_values=rv, layout=layout)
        out[f"{name}/{layout}"] = rv.cpu().numpy().view(np.uint64)
        out[f"{name}/{layout}/root"] = np.array([sg.plan_describe(G, T, "u64", layout)["root"]])
np.savez(sys.argv[2], **{k.replace("/", "__"): v for k, v in out.items()})
"""


@pytest.mark.parametrize("stage_kb", ["0", "100"])
def test_ragged_tail_rows_vrow_variants(oracle, tmp_path, stage_kb):
    import numpy as np
    from sg2v_inputs import erdos_renyi
    names = ("star17", "u17-s22", "u14-2", "star12")
    f = tmp_path / "rows.npz"
    env = dict(os.environ, SG2V_STAGE_KB=stage_kb)
    p = subprocess.run([sys.executable, "-c", _TAIL_SCRIPT, ",".join(names), str(f)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    got = np.load(f)
    g = erdos_renyi(1001, 6000, seed=17)
    for name in names:
        e = TEMPLATES[name]
        k = 1 + max(max(x) for x in e)
        cols = oracle.colors(3, 0, g.n, k)
        for layout in ("anchored", "anchored_plain"):
            rho = int(got[f"{name}__{layout}__root"][0])
            want_tot, want_rows = oracle.count(g, k, e, cols, root=rho, rows=True)
            r = got[f"{name}__{layout}"]
            assert np.array_equal(r, want_rows), (name, layout, stage_kb)
            assert int(r.sum(dtype=np.uint64)) == want_tot
