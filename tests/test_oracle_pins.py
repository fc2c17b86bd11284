"""Pins for the CPU oracle (runs with -m "not gpu").

Every check compares the oracle with something OTHER than itself
(SURVEY.md §8(c) "What pins each part"): brute-force enumeration of the
definition (tests/brute.py), closed forms, exhaustive unbiasedness over all
k^n colourings, and worked examples printed in SPEC.md / SURVEY.md
(tests/golden/*.json, each with its citation).
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from sg2v_inputs import (complete_graph, cycle_graph, csr_from_edges, disjoint_union,
                         erdos_renyi, house_tail_graph, path_graph, path_template,
                         random_tree, star_template)
from tests.brute import injective_homs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _graph(n, edges):
    if not edges:
        return csr_from_edges(n, [], [])
    u, v = zip(*edges)
    return csr_from_edges(n, u, v)


# --------------------------------------------------------------------------- colouring
def test_colour_vectors(oracle):
    for c in _gold("colour_vectors.json")["cases"]:
        got = oracle.colors(c["seed"], c["j"], 16, c["k"]).tolist()
        assert got == c["colors"]


def test_colour_balance(oracle):
    # SURVEY §8(c) step 1 balance check; S:325 (each class within 5σ of n/k)
    n, k = 1 << 20, 17
    cnt = np.bincount(oracle.colors(1, 0, n, k), minlength=k)
    mu = n / k
    sd = math.sqrt(n * (1 / k) * (1 - 1 / k))
    assert np.all(np.abs(cnt - mu) <= 5 * sd)
    assert oracle.colors(5, 3, 100, 1).tolist() == [0] * 100  # k=1 -> all zeros


# --------------------------------------------------------------------------- combinatorics
def test_rank_examples(oracle):
    g = _gold("spec_examples.json")["rank"]
    for s, r in g["cases"]:
        assert oracle.rank(g["k"], s) == r


def test_rank_is_lexicographic_bijection(oracle):
    for k in (4, 6, 7):
        for s in range(k + 1):
            combos = list(itertools.combinations(range(k), s))  # lexicographic (library)
            assert [oracle.rank(k, c) for c in combos] == list(range(len(combos)))


def test_partition_examples(oracle):
    g = _gold("spec_examples.json")
    assert len(oracle.partition(3, [(0, 1), (1, 2)], 1)) == g["partition_P3_root1"]["n_nodes"]
    assert len(oracle.partition(2, [(0, 1)], 0)) == g["partition_edge"]["n_nodes"]
    assert oracle.partition(1, [], 0) == [(1, 0, -1, -1)]


def test_partition_invariants(oracle):
    # leaves sum to k; internal sizes = sum of children; 2k-1 nodes
    for k in range(2, 12):
        for seed in range(5):
            e = random_tree(k, seed)
            for root in range(k):
                nodes = oracle.partition(k, e, root)
                assert len(nodes) == 2 * k - 1
                assert nodes[-1][0] == k
                for i, (size, r, a, p) in enumerate(nodes):
                    if a < 0:
                        assert size == 1
                    else:
                        assert a < i and p < i
                        assert size == nodes[a][0] + nodes[p][0]
                        assert nodes[a][1] == r  # active child keeps the root


def test_not_a_tree(oracle):
    with pytest.raises(ValueError):
        oracle.partition(3, [(0, 1), (1, 2), (0, 2)], 0)  # cycle
    with pytest.raises(ValueError):
        oracle.partition(4, [(0, 1), (1, 2), (0, 2)], 0)  # disconnected
    g = _graph(3, [(0, 1)])
    with pytest.raises(ValueError):
        oracle.count(g, 3, [(0, 1), (0, 1)], np.zeros(3, np.uint8))


def test_alpha_examples(oracle):
    for k, e, a in _gold("spec_examples.json")["alpha"]["cases"]:
        assert oracle.alpha_bruteforce(k, e) == a
        assert oracle.alpha_ahu(k, e) == a


def test_alpha_ahu_matches_bruteforce(oracle):
    for k in range(1, 9):
        for seed in range(12):
            e = random_tree(k, 1000 + seed)
            assert oracle.alpha_ahu(k, e) == oracle.alpha_bruteforce(k, e), (k, e)
        assert oracle.alpha_ahu(k, path_template(k)) == (1 if k == 1 else 2)
        assert oracle.alpha_ahu(k, star_template(k)) == (math.factorial(k - 1) if k > 2 else (1 if k == 1 else 2))


def test_colorful_probability(oracle):
    for k, p in _gold("spec_examples.json")["P"]["cases"]:
        assert oracle.colorful_probability(k) == Fraction(p)
    for k in range(1, 6):  # exhaustive over k^k colourings
        good = sum(len(set(c)) == k for c in itertools.product(range(k), repeat=k))
        assert Fraction(good, k ** k) == oracle.colorful_probability(k)


# --------------------------------------------------------------------------- kernels
def test_spmm_and_ema_examples(oracle):
    g = _gold("spec_examples.json")
    for key in ("spmv_path", "spmv_triangle_ones"):
        c = g[key]
        out = oracle.spmm(_graph(c["n"], c["edges"]), np.array(c["x"], float))
        assert out.ravel().tolist() == c["out"]
    c = g["spmm_batch"]
    out = oracle.spmm(_graph(c["n"], c["edges"]), np.array(c["x"], float))
    assert out.tolist() == c["out"]
    c = g["ema"]
    assert oracle.ema(np.array(c["dst"], float), np.array(c["a"], float), np.array(c["b"], float)).tolist() == c["out"]


def test_spmm_matches_dense_matmul(oracle):
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 60))
        g = erdos_renyi(n, int(rng.integers(0, n * (n - 1) // 2 + 1)), seed=int(rng.integers(1 << 30))) if n > 1 else _graph(1, [])
        A = np.zeros((n, n))
        for i in range(n):
            A[i, g.col_indices[g.row_offsets[i]:g.row_offsets[i + 1]]] = 1
        X = rng.integers(0, 100, size=(n, 7)).astype(float)
        assert np.array_equal(oracle.spmm(g, X), A @ X)


# --------------------------------------------------------------------------- DP vs brute force
SMALL_TREES = {
    1: [[]],
    2: [[(0, 1)]],
    3: [[(0, 1), (1, 2)]],
    4: [path_template(4), star_template(4)],
    5: [path_template(5), star_template(5), [(0, 1), (1, 2), (0, 3), (0, 4)], [(0, 1), (1, 2), (2, 3), (1, 4)]],
}


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_dp_equals_bruteforce_all_roots(oracle, k):
    rng = random.Random(k)
    for gi in range(6):
        n = rng.randint(k, 9)
        m = rng.randint(n - 1, min(n * (n - 1) // 2, 3 * n))
        g = erdos_renyi(n, m, seed=100 * k + gi)
        for e in SMALL_TREES[k]:
            for j in range(3):
                cols = oracle.colors(rng.randint(0, 1 << 40), j, n, k)
                want = injective_homs(g, k, e, cols)
                for root in range(k):
                    assert oracle.count(g, k, e, cols, root=root) == want
                    tot, vmax = oracle.count(g, k, e, cols, root=root, arith=oracle.ARITH_F64)
                    assert tot == float(want) and vmax >= want
                assert oracle.count(g, k, e, cols, form=oracle.FORM_ALG2) == want


def test_spec_dp_example(oracle):
    c = _gold("spec_examples.json")["dp_edge_triangle"]
    g = _graph(c["n"], c["edges"])
    col = np.array(c["colors"], np.uint8)
    got = oracle.count(g, c["k"], [(0, 1)], col)
    assert got == c["colorful"]
    assert oracle.final_count(got, 2, [(0, 1)]) == c["final"]
    assert oracle.count(g, 1, [], np.zeros(3, np.uint8)) == 3  # single vertex -> n


def test_spec_exact_counts(oracle):
    graphs = {"K3": complete_graph(3), "K4": complete_graph(4)}
    temps = {"edge": (2, [(0, 1)]), "P3": (3, [(0, 1), (1, 2)])}
    for gname, tname, want in _gold("spec_examples.json")["exact_counts"]["cases"]:
        k, e = temps[tname]
        assert injective_homs(graphs[gname], k, e) // oracle.alpha(k, e) == want


def test_house_tail_golden(oracle):
    gd = _gold("house_tail.json")
    g = _graph(gd["n"], gd["graph_edges"])
    assert oracle.colors(gd["seed"], 0, gd["n"], 3).tolist() == gd["colors_k3_j0"]
    for t in gd["templates"]:
        e = [tuple(x) for x in t["edges"]]
        k = 1 + max(max(x) for x in e)
        assert oracle.alpha(k, e) == t["alpha"]
        assert injective_homs(g, k, e) == t["emb"] * t["alpha"]
        got = [oracle.count(g, k, e, oracle.colors(gd["seed"], j, gd["n"], k)) for j in range(4)]
        assert got == t["colorful"]
        est = sum(Fraction(x) for x in got) / 4 / (oracle.colorful_probability(k) * t["alpha"])
        assert est == Fraction(t["estimate"])


# --------------------------------------------------------------------------- closed forms
def test_closed_form_tree_on_complete_graph(oracle):
    # colorful = k!·Π_c n_c for any tree on K_n (SURVEY §8(c) pin 2)
    for n in (6, 9, 13):
        g = complete_graph(n)
        for k in (3, 4, 5):
            for e in (path_template(k), star_template(k), random_tree(k, n)):
                for j in range(4):
                    cols = oracle.colors(7, j, n, k)
                    nc = np.bincount(cols, minlength=k)
                    want = math.factorial(k) * int(np.prod(nc[:k].astype(object)))
                    assert oracle.count(g, k, e, cols) == want


def test_closed_form_star(oracle):
    # colorful(S_k) = (k-1)!·Σ_i Π_{c≠c(i)} H(i,c), H = neighbour colour histogram
    g = erdos_renyi(60, 400, seed=5)
    for k in (3, 4, 5, 6):
        for j in range(3):
            cols = oracle.colors(11, j, g.n, k)
            want = 0
            for i in range(g.n):
                nb = g.col_indices[g.row_offsets[i]:g.row_offsets[i + 1]]
                H = np.bincount(cols[nb], minlength=k).astype(object)
                p = 1
                for c in range(k):
                    if c != cols[i]:
                        p *= H[c]
                want += p
            want *= math.factorial(k - 1)
            for root in (0, 1):
                assert oracle.count(g, k, star_template(k), cols, root=root) == want


def test_closed_form_path_on_cycle_and_path(oracle):
    for n in (9, 14):
        for k in (3, 4, 5, 6):
            for j in range(3):
                cols = oracle.colors(3, j, n, k)
                win = sum(len({int(cols[(s + t) % n]) for t in range(k)}) == k for s in range(n))
                assert oracle.count(cycle_graph(n), k, path_template(k), cols) == 2 * win
                win2 = sum(len({int(cols[s + t]) for t in range(k)}) == k for s in range(n - k + 1))
                assert oracle.count(path_graph(n), k, path_template(k), cols) == 2 * win2


def test_closed_form_edge(oracle):
    g = erdos_renyi(50, 200, seed=9)
    cols = oracle.colors(1, 0, 50, 2)
    e = g.edges()
    want = 2 * int(np.sum(cols[e[:, 0]] != cols[e[:, 1]]))
    assert oracle.count(g, 2, [(0, 1)], cols) == want


# --------------------------------------------------------------------------- unbiasedness
def test_exhaustive_unbiasedness(oracle):
    # mean over all k^n colourings of colorful/(P·α) == emb exactly
    cases = [
        (path_graph(4), 3, [(0, 1), (1, 2)]),
        (complete_graph(4), 3, [(0, 1), (1, 2)]),
        (cycle_graph(4), 2, [(0, 1)]),
        (_graph(5, [(0, 1), (1, 2), (2, 3), (1, 4), (0, 2)]), 4, star_template(4)),
        (_graph(5, [(0, 1), (1, 2), (2, 3), (1, 4), (0, 2)]), 4, path_template(4)),
    ]
    for g, k, e in cases:
        tot = 0
        for cols in itertools.product(range(k), repeat=g.n):
            tot += oracle.count(g, k, e, np.array(cols, np.uint8))
        alpha = oracle.alpha(k, e)
        emb = Fraction(injective_homs(g, k, e), alpha)
        assert Fraction(tot, k ** g.n) / (oracle.colorful_probability(k) * alpha) == emb
    # SURVEY §8(c) pin 3 integer: P3 in P_4, summed over 81 colourings = 72
    tot = sum(oracle.count(path_graph(4), 3, [(0, 1), (1, 2)], np.array(c, np.uint8))
              for c in itertools.product(range(3), repeat=4))
    assert tot == 72


# --------------------------------------------------------------------------- invariants
def test_colour_permutation_and_union(oracle):
    g1 = erdos_renyi(40, 160, seed=2)
    g2 = erdos_renyi(30, 90, seed=3)
    gu = disjoint_union(g1, g2)
    k, e = 5, [(0, 1), (1, 2), (0, 3), (0, 4)]
    for j in range(3):
        c1 = oracle.colors(4, j, g1.n, k)
        c2 = oracle.colors(5, j, g2.n, k)
        cu = np.concatenate([c1, c2])
        a = oracle.count(g1, k, e, c1)
        b = oracle.count(g2, k, e, c2)
        assert oracle.count(gu, k, e, cu) == a + b
        perm = np.array([3, 0, 4, 1, 2], np.uint8)
        assert oracle.count(g1, k, e, perm[c1]) == a


def test_u64_matches_f64_below_2_53(oracle):
    g = erdos_renyi(1000, 4000, seed=1)  # D1
    for k, e in ((3, path_template(3)), (5, [(0, 1), (1, 2), (0, 3), (0, 4)]), (6, random_tree(6, 4))):
        cols = oracle.colors(1, 0, g.n, k)
        u = oracle.count(g, k, e, cols)
        f, vmax = oracle.count(g, k, e, cols, arith=oracle.ARITH_F64)
        assert vmax < 2 ** 53 and f == float(u)


# --------------------------------------------------------------------------- α beyond brute-force k! (k = 9, 10, repo templates)
def test_alpha_ahu_vs_enumeration(oracle):
    """The oracle's α for k >= 9 comes from the AHU product formula; pin it against
    explicit enumeration of the automorphisms (tests/brute.py, backtracking, no AHU)
    for random trees with k = 9, 10 and every repo template whose group is listable,
    and against the closed form |Aut(S_k)| = (k-1)! for stars (k >= 3)."""
    from sg2v_inputs import TEMPLATES
    from tests.brute import automorphisms_backtrack
    cases = [(k, random_tree(k, 1000 * k + s)) for k in (9, 10) for s in range(8)]
    cases += [(1 + max(max(x) for x in e), e) for name, e in TEMPLATES.items()
              if e and not name.startswith("star")]
    checked = 0
    for k, e in cases:
        a = automorphisms_backtrack(k, e, cap=50_000)
        if a is None:
            continue
        assert oracle.alpha_ahu(k, e) == a, (k, e)
        assert oracle.alpha(k, e) == a
        checked += 1
    assert checked >= len(cases) - 2
    for k in range(3, 21):
        assert oracle.alpha_ahu(k, star_template(k)) == math.factorial(k - 1)


# --------------------------------------------------------------------------- max-intermediate gates
def test_max_intermediate_includes_B_and_live_max_excludes_dead(oracle):
    """vmax (the "exact below 2^53 / 2^24" gate, SURVEY §8(c) pin 6) must include the
    B = A·M_p entries, and max_live (the F32-overflow gate) must leave out the B entries
    that only meet zeros (I_p ∋ c(i)) and a leaf-active top's B.  Crafted on the star
    K_{1,m} (centre 0) with closed-form values."""
    m = 7
    g = _graph(m + 1, [(0, x) for x in range(1, m + 1)])
    # monochromatic: colorful = 0, every table entry <= 1, but B(centre,{0}) = m
    tot, vmax, live = oracle.count(g, 2, [(0, 1)], np.zeros(m + 1, np.uint8), arith=oracle.ARITH_F64, live=True)
    assert (tot, vmax, live) == (0.0, float(m), 1.0)
    # centre colour 0, leaves colour 1: colorful = 2m (both orientations), leaf tables = 1,
    # the top's B(i,[k]\{c(i)}) = per-vertex totals (m at the centre) are not F32-held
    c = np.ones(m + 1, np.uint8)
    c[0] = 0
    tot, vmax, live = oracle.count(g, 2, [(0, 1)], c, arith=oracle.ARITH_F64, live=True)
    assert (tot, vmax, live) == (2.0 * m, 2.0 * m, 1.0)
    # P3 rooted at its centre on the star, leaves alternating colours 1, 2 (4 and 3 of
    # them): colorful = 2·4·3; the largest held entry is M_{edge}(centre,{0,1}) = 4
    c = np.array([0] + [1, 2] * 3 + [1], np.uint8)
    tot, vmax, live = oracle.count(g, 3, [(0, 1), (1, 2)], c, root=1, arith=oracle.ARITH_F64, live=True)
    assert tot == 24.0 and live == 4.0 and vmax == 24.0
