"""Template trees as data (edge lists over vertex ids 0..k-1).

The paper's template shapes are lost (Fig. 4 is an image, PAPER.md:502-509;
"templates with more than 12 nodes are randomly selected"), so
the shapes are repo data, as SURVEY.md §8(d) "Template files" proposes:

* ``uK-1`` = path P_K (Fascia-style "-1" naming; the shape is a guess).
* ``u5-2``, ``u7-2``, ``u10-2``, ``u17``, ``u17-s22``, ``u20``: the concrete
  trees listed in SURVEY §8(d) (Prüfer draws with random.Random(2009_11665)).
* ``u13-2``, ``u14-2``, ``u15-2``, ``u16-2``: Prüfer draws with a fixed seed
  (``random_tree``), committed here as data.
* paths and stars of every size bracket SpMM-heavy and eMA-heavy shapes.
"""
from __future__ import annotations

import random


def path_template(k: int):
    return [(i, i + 1) for i in range(k - 1)]


def star_template(k: int):
    return [(0, i) for i in range(1, k)]


def random_tree(k: int, seed: int):
    """Uniform labelled tree on k vertices via a Prüfer sequence (k >= 2)."""
    if k == 1:
        return []
    if k == 2:
        return [(0, 1)]
    rnd = random.Random(seed)
    seq = [rnd.randrange(k) for _ in range(k - 2)]
    degree = [1] * k
    for x in seq:
        degree[x] += 1
    edges = []
    for x in seq:
        for leaf in range(k):
            if degree[leaf] == 1:
                edges.append((min(leaf, x), max(leaf, x)))
                degree[leaf] -= 1
                degree[x] -= 1
                break
    u, v = [i for i in range(k) if degree[i] == 1]
    edges.append((u, v))
    return sorted(edges)


TEMPLATES = {
    "u1": [],
    "u2": [(0, 1)],
    "u3-1": path_template(3),
    "u5-2": [(0, 1), (1, 2), (0, 3), (0, 4)],
    "u7-2": [(0, 4), (1, 2), (1, 4), (2, 5), (2, 6), (3, 6)],
    "u10-2": [(0, 1), (0, 3), (1, 6), (1, 7), (1, 9), (2, 9), (3, 4), (5, 9), (7, 8)],
    "u12-1": path_template(12),
    "u13-1": path_template(13),
    "u14-1": path_template(14),
    "u15-1": path_template(15),
    "u16-1": path_template(16),
    "u17-1": path_template(17),
    "u17": [(0, 15), (0, 16), (1, 13), (1, 14), (2, 3), (2, 9), (2, 14), (3, 6), (4, 13),
            (5, 10), (5, 12), (7, 16), (8, 10), (10, 13), (11, 15), (13, 16)],
    "u17-s22": [(0, 4), (0, 9), (1, 7), (2, 7), (3, 8), (4, 15), (5, 12), (6, 7), (6, 9),
                (8, 15), (9, 10), (9, 11), (9, 12), (10, 14), (12, 16), (13, 16)],
    "u20": [(0, 15), (1, 6), (1, 17), (2, 17), (3, 6), (4, 9), (4, 17), (5, 17), (6, 10),
            (6, 14), (6, 18), (7, 10), (8, 10), (8, 15), (11, 15), (12, 16), (12, 18),
            (13, 19), (14, 19)],
    "u13-2": random_tree(13, 2009_11665 + 13),
    "u14-2": random_tree(14, 2009_11665 + 14),
    "u15-2": random_tree(15, 2009_11665 + 15),
    "u16-2": random_tree(16, 2009_11665 + 16),
    "star4": star_template(4),
}
for _k in range(2, 21):
    TEMPLATES.setdefault(f"path{_k}", path_template(_k))
    TEMPLATES.setdefault(f"star{_k}", star_template(_k))


def template_edges(name: str):
    """(k, edges) for a named template."""
    e = TEMPLATES[name]
    k = 1 + max((max(a, b) for a, b in e), default=0)
    return k, list(e)


def _canon_free(k, edges):
    """Canonical string of an unrooted tree (centre + AHU nesting) for dedupe."""
    adj = [[] for _ in range(k)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)

    def enc(v, p):
        return "(" + "".join(sorted(enc(c, v) for c in adj[v] if c != p)) + ")"
    if k <= 2:
        return str(k)
    deg = [len(x) for x in adj]
    layer = [v for v in range(k) if deg[v] == 1]
    left = k
    while left > 2:
        left -= len(layer)
        nxt = []
        for v in layer:
            for u in adj[v]:
                deg[u] -= 1
                if deg[u] == 1:
                    nxt.append(u)
        layer = nxt
    if len(layer) == 1:
        return enc(layer[0], -1)
    a, b = layer
    return "".join(sorted([enc(a, b), enc(b, a)]))


def all_trees(k: int):
    """Every non-isomorphic tree on k vertices (k <= 9), as edge lists, in a fixed
    order (Prüfer enumeration, first representative of each isomorphism class).
    Counts: 1, 1, 1, 2, 3, 6, 11, 23, 47 (the paper's 47 size-9 treelets)."""
    import itertools
    if k == 1:
        return [[]]
    if k == 2:
        return [[(0, 1)]]
    seen, out = set(), []
    for seq in itertools.product(range(k), repeat=k - 2):
        degree = [1] * k
        for x in seq:
            degree[x] += 1
        edges = []
        for x in seq:
            for leaf in range(k):
                if degree[leaf] == 1:
                    edges.append((min(leaf, x), max(leaf, x)))
                    degree[leaf] -= 1
                    degree[x] -= 1
                    break
        u, v = [i for i in range(k) if degree[i] == 1]
        edges.append((u, v))
        c = _canon_free(k, edges)
        if c not in seen:
            seen.add(c)
            out.append(sorted(edges))
    return out
