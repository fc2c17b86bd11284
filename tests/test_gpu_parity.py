"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bars (BASELINE.json north_star):
  * U64: bit-exact residues mod 2^64, every colouring, every config;
  * F64: bit-exact while the oracle's max intermediate < 2^53, else rel 1e-12;
  * F32: rel 1e-4 (bit-exact when the oracle's max intermediate < 2^24).
Per-vertex values Σ_C M_0(i,·) are compared element by element.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2009_11665_b200 as sg  # noqa: E402
from sg2v_inputs import (TEMPLATES, complete_graph, csr_from_edges, erdos_renyi,  # noqa: E402
                         path_template, random_tree, rmat, star_template)


def _k(e):
    return 1 + max((max(x) for x in e), default=0)


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.set_device(0)


def _load(g):
    return sg.graph_load_csr(g.n, g.row_offsets, g.col_indices, validate=True)


# anchored without / with every eligible exclusion-projected table (the default
# "anchored" picks between the two per class), dense
LAYOUTS = ("anchored_plain", "anchored_proj", "dense")


FLT_MAX = 3.4028234663852886e38


def _rows(G, T, seed, j, prec, layout="anchored"):
    """(status, total, per-vertex values) of one colouring; status 0 or EOVERFLOW."""
    dt = torch.int64 if prec == "u64" else torch.float64
    rv = torch.zeros(max(G.n, 1), dtype=dt, device="cuda")
    status = 0
    try:
        _, tot = sg.count(G, T, n_iter=1, seed=seed, iter_offset=j, precision=prec, row_values=rv, layout=layout)
    except sg.Sg2vError as ex:
        assert ex.code == sg.sg2v.EOVERFLOW, ex
        status = ex.code
        _, tot = sg.count(G, T, n_iter=1, seed=seed, iter_offset=j, precision=prec, row_values=rv,
                          allow_overflow=True, layout=layout)
    r = rv.cpu().numpy()[:G.n]
    return status, tot[0], (r.view(np.uint64) if prec == "u64" else r)


def assert_f32_rows(r, want):
    """F32 per-vertex values: exact zeros where the oracle's value is 0 (sums of
    non-negative terms), relative error <= 1e-4 element by element elsewhere."""
    zero = want == 0
    assert np.all(r[zero] == 0), np.flatnonzero(r[zero] != 0)[:5]
    nz = ~zero
    rel = np.abs(r[nz] - want[nz]) / want[nz]
    assert rel.size == 0 or float(rel.max()) <= 1e-4, float(rel.max())


def _check_all(oracle, g, e, seeds_js, roots=(-1,), precs=("u64", "f64", "f32"), rows=True, layouts=LAYOUTS):
    k = _k(e)
    G = _load(g)
    for root in roots:
        T = sg.template_build(k, e, root_hint=root)
        for seed, j in seeds_js:
            cols = oracle.colors(seed, j, g.n, k)
            for prec, layout in [(p, l) for p in precs for l in layouts]:
                # per-vertex values count embeddings with the ROOT mapped to i, so the
                # oracle is rooted where the planner rooted (the total is root-free)
                rho = sg.plan_describe(G, T, prec, layout).get("root", 0) if k > 1 else 0
                want_u, want_ru = oracle.count(g, k, e, cols, root=rho, rows=True)
                want_f, vmax, vlive, want_rf = oracle.count(g, k, e, cols, root=rho, arith=oracle.ARITH_F64,
                                                            rows=True, live=True)
                status, tot, r = _rows(G, T, seed, j, prec, layout)
                if not rows:
                    r = None
                if prec == "u64":
                    assert status == 0
                    assert int(tot) == want_u, (root, seed, j, layout)
                    if r is not None:
                        assert np.array_equal(r, want_ru)
                elif prec == "f64":
                    assert status == 0
                    if vmax < 2 ** 53:
                        assert tot == want_f
                        if r is not None:
                            assert np.array_equal(r, want_rf)
                    else:
                        assert math.isclose(tot, want_f, rel_tol=1e-12)
                        if r is not None:
                            assert np.allclose(r, want_rf, rtol=1e-12, atol=0)
                else:
                    # EOVERFLOW contract: every F32-held entry below FLT_MAX -> finite;
                    # some held entry above it -> EOVERFLOW (the dense layout also holds
                    # dead B entries, gated by the all-entries max)
                    if vlive > FLT_MAX * 1.001:
                        assert status == sg.sg2v.EOVERFLOW, (layout, vlive)
                        continue
                    if vmax < FLT_MAX * 0.999 or (layout != "dense" and vlive < FLT_MAX * 0.999):
                        assert status == 0 and math.isfinite(tot), (layout, vmax, vlive)
                    if status:
                        continue
                    if vmax < 2 ** 24:
                        assert tot == want_f
                        if r is not None:
                            assert np.array_equal(r, want_rf)
                    else:
                        assert math.isclose(tot, want_f, rel_tol=1e-4)
                        if r is not None:
                            assert_f32_rows(r, want_rf)


# --------------------------------------------------------------------------- a1
def test_colorize_matches_oracle(oracle):
    n = 100_003
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    for seed, j, k in ((1, 0, 3), (42, 7, 17), (2**63 + 5, 123456, 31), (9, 2, 1)):
        sg.colorize(seed, j, n, k, out)
        assert np.array_equal(out.cpu().numpy(), oracle.colors(seed, j, n, k))


# --------------------------------------------------------------------------- D1 (configs[0])
def test_d1_u3_er1000_100_colourings(oracle):
    g = erdos_renyi(1000, 4000, seed=1)
    e = TEMPLATES["u3-1"]
    G = _load(g)
    T = sg.template_build(3, e)
    want = [oracle.count(g, 3, e, oracle.colors(1, j, g.n, 3)) for j in range(100)]
    for prec, layout in [(p, l) for p in ("u64", "f64", "f32") for l in LAYOUTS]:
        est, got = sg.count(G, T, n_iter=100, seed=1, precision=prec, layout=layout)
        assert [int(x) for x in got] == want  # all values < 2^24: bit-exact in every mode
        if prec != "u64":
            P = math.factorial(3) / 27
            assert math.isclose(est, sum(want) / 100 / (P * 2), rel_tol=1e-12)
        else:
            assert math.isnan(est)


# --------------------------------------------------------------------------- template zoo
ZOO = ["u2", "u3-1", "star4", "path4", "u5-2", "star5", "path6", "star6", "u7-2", "u10-2"]


@pytest.mark.parametrize("name", ZOO)
def test_zoo_small_rmat(oracle, name):
    g = rmat(11, 30_000, 0.45, 0.22, 0.22, seed=3)
    e = TEMPLATES[name]
    roots = (-1, 0, _k(e) - 1)
    _check_all(oracle, g, e, [(1, 0), (7, 3)], roots=roots)


@pytest.mark.parametrize("k", [4, 6, 8, 9])
def test_random_trees_all_roots(oracle, k):
    g = erdos_renyi(300, 1500, seed=k)
    e = random_tree(k, 31 * k)
    _check_all(oracle, g, e, [(5, 1)], roots=tuple(range(-1, k)), precs=("u64",))


def test_wide_rows_multiple_passes(oracle):
    # u15-1: c_p up to C(15,7)=6435 -> several 1024-vector passes per row (fp32) and
    # odd widths (ragged tails of the 16-B vectors); also u12-1
    g = erdos_renyi(1500, 9000, seed=4)
    # "anchored_proj" plans use exclusion-projected tables (written by leaf-active
    # copies; read by projected gathers)
    G = _load(g)
    for name in ("u15-1", "u12-1"):
        d = sg.plan_describe(G, sg.template_build(_k(TEMPLATES[name]), TEMPLATES[name]), "u64", "anchored_proj")
        assert any(s["proj_p"] for s in d["steps"]) and any(s["proj_out"] for s in d["steps"]), name
    _check_all(oracle, g, TEMPLATES["u15-1"], [(1, 0)], precs=("u64", "f64", "f32"))
    _check_all(oracle, g, TEMPLATES["u12-1"], [(2, 5)], roots=(-1, 0, 5))


def test_heavy_hub_and_isolated(oracle):
    # one hub adjacent to every vertex + a sparse remainder + isolated vertices
    n = 3000
    rng = np.random.default_rng(0)
    u = np.concatenate([np.zeros(n - 100, np.int64), rng.integers(1, n, 4000)])
    v = np.concatenate([np.arange(1, n - 99), rng.integers(1, n, 4000)])
    g = csr_from_edges(n + 50, u, v)
    assert int(np.diff(g.row_offsets).max()) >= 2048  # the CTA-per-heavy-row kernel runs
    for name in ("u5-2", "path6", "star5", "u10-2", "u12-1"):
        _check_all(oracle, g, TEMPLATES[name], [(3, 2)])


# --------------------------------------------------------------------------- edge cases
def test_k1_k2_and_tiny(oracle):
    g = erdos_renyi(50, 200, seed=2)
    G = _load(g)
    T1 = sg.template_build(1, [])
    _, c = sg.count(G, T1, n_iter=3, seed=1, precision="u64")
    assert [int(x) for x in c] == [50] * 3
    T2 = sg.template_build(2, [(0, 1)])
    for j in range(3):
        cols = oracle.colors(1, j, g.n, 2)
        ed = g.edges()
        want = 2 * int(np.sum(cols[ed[:, 0]] != cols[ed[:, 1]]))
        _, c = sg.count(G, T2, n_iter=1, seed=1, iter_offset=j, precision="u64")
        assert int(c[0]) == want
    # n < k: no colourful embedding possible
    gk = complete_graph(3)
    _, c = sg.count(_load(gk), sg.template_build(5, TEMPLATES["u5-2"]), n_iter=2, seed=1, precision="u64")
    assert list(c) == [0, 0]
    # graph without edges
    ge = csr_from_edges(10, [], [])
    _, c = sg.count(_load(ge), sg.template_build(3, path_template(3)), n_iter=1, seed=1, precision="f32")
    assert list(c) == [0.0]


def test_empty_graph():
    G = sg.graph_load_csr(0, np.zeros(1, np.int64), np.zeros(0, np.int32))
    _, c = sg.count(G, sg.template_build(3, path_template(3)), n_iter=2, seed=1, precision="u64")
    assert list(c) == [0, 0]


def test_errors():
    g = erdos_renyi(20, 40, seed=1)
    G = _load(g)
    T = sg.template_build(3, path_template(3))
    with pytest.raises(sg.Sg2vError) as e:
        sg.count(G, T, n_iter=0, seed=1)
    assert e.value.code == sg.sg2v.EINVAL
    # unsorted / asymmetric / self-loop CSR rejected by VALIDATE
    bad = [
        (np.array([0, 2, 3, 4]), np.array([2, 1, 0, 0], np.int32)),  # row 0 unsorted
        (np.array([0, 1, 1, 1]), np.array([1], np.int32)),           # asymmetric
        (np.array([0, 1, 1, 1]), np.array([0], np.int32)),           # self-loop
    ]
    for ro, ci in bad:
        with pytest.raises(sg.Sg2vError) as e:
            sg.graph_load_csr(3, ro, ci, validate=True)
        assert e.value.code == sg.sg2v.EINVAL
    # memory budget / workspace too small: ENOMEM before allocating
    big = sg.template_build(12, path_template(12))
    with pytest.raises(sg.Sg2vError) as e:
        sg.count(G, big, n_iter=1, seed=1, workspace=sg.Workspace(16))
    assert e.value.code == sg.sg2v.ENOMEM
    o = sg.Options()
    sg.lib().sg2v_options_default(o)
    o.precision = sg.U64
    o.mem_budget_bytes = 1024
    rc = sg.lib().sg2v_count_ex(G.handle, big.handle, 12, 1, 1, o, None, None, None)
    assert rc == sg.sg2v.ENOMEM and b"needs" in sg.lib().sg2v_last_error()


def test_determinism_and_sharding():
    # bitwise determinism (fixed summation order, no atomics); promised for U64 and F64
    # below 2^53; F32 is also run-to-run identical in this build
    g = rmat(12, 60_000, 0.45, 0.22, 0.22, seed=5)
    G = _load(g)
    T = sg.template_build(7, TEMPLATES["u7-2"])
    for layout in LAYOUTS:
        _, a = sg.count(G, T, n_iter=8, seed=11, precision="u64", layout=layout)
        _, b = sg.count(G, T, n_iter=8, seed=11, precision="u64", layout=layout)
        assert np.array_equal(a, b)                                   # run-to-run bitwise
        _, s0 = sg.count(G, T, n_iter=4, seed=11, iter_offset=0, iter_stride=2, precision="u64", layout=layout)
        _, s1 = sg.count(G, T, n_iter=4, seed=11, iter_offset=1, iter_stride=2, precision="u64", layout=layout)
        assert np.array_equal(a[0::2], s0) and np.array_equal(a[1::2], s1)  # replica shards
        _, f = sg.count(G, T, n_iter=8, seed=11, precision="f32", layout=layout)
        _, f2 = sg.count(G, T, n_iter=8, seed=11, precision="f32", layout=layout)
        assert np.array_equal(f, f2)


def test_closed_form_tree_on_complete_graph(oracle):
    # colorful = k!·Π_c n_c for any tree on K_n (SURVEY §8(c) pin 2), independent of the oracle
    g = complete_graph(120)
    G = _load(g)
    for k, e in ((5, TEMPLATES["u5-2"]), (7, TEMPLATES["u7-2"]), (9, star_template(9))):
        T = sg.template_build(k, e)
        _, got = sg.count(G, T, n_iter=3, seed=4, precision="u64")
        for j in range(3):
            nc = np.bincount(oracle.colors(4, j, g.n, k), minlength=k)
            want = math.factorial(k) * math.prod(int(x) for x in nc)
            assert int(got[j]) == want % (1 << 64)


def test_f32_close_to_f64_on_dense_graph():
    g = complete_graph(200)
    G = _load(g)
    T = sg.template_build(8, path_template(8))
    _, f = sg.count(G, T, n_iter=1, seed=1, precision="f32")
    _, d = sg.count(G, T, n_iter=1, seed=1, precision="f64")
    assert math.isclose(f[0], d[0], rel_tol=1e-4)


# --------------------------------------------------------------------------- multi-template batch
def test_count_batch_equals_single_counts(oracle):
    from sg2v_inputs import all_trees
    g = rmat(11, 30_000, 0.45, 0.22, 0.22, seed=8)
    G = _load(g)
    trees = all_trees(6)
    Ts = [sg.template_build(6, e) for e in trees]
    for layout in LAYOUTS:
        est, col = sg.count_batch(G, Ts, n_iter=3, seed=4, precision="u64", layout=layout)
        for t, e in enumerate(trees):
            _, one = sg.count(G, Ts[t], n_iter=3, seed=4, precision="u64", layout=layout)
            assert np.array_equal(col[t], one)
            assert int(col[t][1]) == oracle.count(g, 6, e, oracle.colors(4, 1, g.n, 6))
        estf, colf = sg.count_batch(G, Ts, n_iter=3, seed=4, precision="f64", layout=layout)
        for t in range(len(trees)):
            _, onef = sg.count(G, Ts[t], n_iter=3, seed=4, precision="f64", layout=layout)
            assert np.array_equal(colf[t], onef)
    with pytest.raises(sg.Sg2vError):
        sg.count_batch(G, [Ts[0], sg.template_build(5, TEMPLATES["u5-2"])], n_iter=1, seed=1)


def test_fig1_analogue_treelet_distributions():
    # SPEC S:540 / P:107-117: distributions over the 11 size-7 trees separate two
    # structurally different random-graph models more than two samples of one model
    from paper_2009_11665_b200.estimator import compare_distributions, estimate_distribution
    from sg2v_inputs import all_trees, csr_from_edges
    trees = all_trees(7)
    Ts = [sg.template_build(7, e) for e in trees]

    def regular(seed, n=500, d=6):
        rng = np.random.default_rng(seed)
        stubs = np.repeat(np.arange(n), d)
        rng.shuffle(stubs)
        return csr_from_edges(n, stubs[0::2], stubs[1::2])

    def pref_attach(seed, n=500, m=3):
        rng = np.random.default_rng(seed)
        us, vs, targets = [], [], list(range(m))
        for v in range(m, n):
            pick = rng.choice(targets, size=m, replace=True)
            for u in pick:
                us.append(v)
                vs.append(int(u))
            targets += list(pick) + [v] * m
        return csr_from_edges(n, us, vs)

    dists = []
    for g in (regular(1), regular(2), pref_attach(1), pref_attach(2)):
        d, _, _ = estimate_distribution(_load(g), Ts, n_iter=200, seed=3, precision="f64")
        dists.append(d)
    D = compare_distributions(dists)
    within = max(D[0, 1], D[2, 3])
    between = min(D[0, 2], D[0, 3], D[1, 2], D[1, 3])
    assert between > within


# --------------------------------------------------------------------------- table sharing / self steps
SYMMETRIC = {
    "spider3x2": [(0, 1), (1, 2), (0, 3), (3, 4), (0, 5), (5, 6)],          # 3 identical legs
    "spider4x2": [(0, 1), (1, 2), (0, 3), (3, 4), (0, 5), (5, 6), (0, 7), (7, 8)],
    "double_star": [(0, 1), (0, 2), (0, 3), (1, 4), (1, 5), (1, 6)],        # two isomorphic halves
    "path9": [(i, i + 1) for i in range(8)],                                 # middle root: self top
    "caterpillar": [(0, 1), (1, 2), (2, 3), (3, 4), (1, 5), (3, 6)],
}


@pytest.mark.parametrize("name", sorted(SYMMETRIC))
def test_shared_and_self_steps_vs_oracle(oracle, name):
    e = SYMMETRIC[name]
    k = _k(e)
    g = erdos_renyi(400, 2400, seed=k)
    T = sg.template_build(k, e)
    d = sg.plan_describe(G := _load(g), T, "u64")
    assert len(d["steps"]) < k - 1 or any(s.get("self") for s in d["steps"]) or name == "caterpillar"
    _check_all(oracle, g, e, [(3, 0), (3, 1)], roots=tuple(range(-1, k)), precs=("u64",))


def test_split_ema_pipeline(oracle):
    """eMA-heavy GENERAL steps run as the two-stream split pipeline (gather of row chunk c
    beside the eMA of chunk c-1, B rows handed over in HBM): per-vertex values equal the
    oracle's with several chunks (n = 5000 -> 1024-row chunks), U64 exact and F32 1e-4."""
    g = erdos_renyi(5000, 25_000, seed=21)
    G = _load(g)
    for name in ("u13-2", "u14-2"):
        e = TEMPLATES[name]
        d = sg.plan_describe(G, sg.template_build(_k(e), e), "u64")
        assert any(s["split_ema"] for s in d["steps"]), name
        _check_all(oracle, g, e, [(4, 1)], precs=("u64", "f32"), layouts=("anchored",))
