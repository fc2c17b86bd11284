"""Deterministic graph generators producing simple undirected graphs as CSR.

Graph semantics follow PAPER.md:357 (A_G is a 0-1 symmetric CSR adjacency)
and the reading in SURVEY.md §8(c) "Graph semantics": undirected, simple,
duplicates removed, self-loops dropped, column ids sorted inside each row.

* ``erdos_renyi``: G(n, m) with m uniform distinct pairs.
* ``rmat``: RMAT(a,b,c,d) edge draw (Chakrabarti et al.), random
  id permutation, symmetrised + deduplicated (SURVEY §8(d) D2–D5a).
* small closed-form graphs (cycle, path, complete, "house+tail") used by the
  oracle pins (SURVEY §8(c) "What pins each part").

ER uses numpy ``default_rng(seed)``; RMAT uses counter-hash uniforms in gen.c
(thread-count independent), so the same arrays come out on every machine.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CSR:
    """Symmetric 0-1 adjacency in CSR form: int64 row_offsets[n+1], int32 col[nnz]."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def edges(self):
        """Undirected edge list (u < v) as an (m, 2) int64 array."""
        rows = np.repeat(np.arange(self.n, dtype=np.int64), self.degrees)
        cols = self.col_indices.astype(np.int64)
        keep = rows < cols
        return np.stack([rows[keep], cols[keep]], axis=1)

    def nbytes(self) -> int:
        return self.row_offsets.nbytes + self.col_indices.nbytes


def csr_from_edges(n: int, u, v, name: str = "") -> CSR:
    """Symmetrise, drop self-loops, deduplicate, sort -> CSR."""
    u = np.asarray(u, dtype=np.int64).ravel()
    v = np.asarray(v, dtype=np.int64).ravel()
    keep = u != v
    u, v = u[keep], v[keep]
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    keys = np.unique(src * np.int64(n) + dst)
    src = keys // n
    dst = keys - src * n
    counts = np.bincount(src, minlength=n).astype(np.int64)
    row_offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_offsets[1:])
    return CSR(n=n, row_offsets=row_offsets, col_indices=dst.astype(np.int32), name=name)


def erdos_renyi(n: int, m: int, seed: int = 1) -> CSR:
    """G(n, m): m distinct undirected pairs drawn uniformly."""
    rng = np.random.default_rng(seed)
    if m > n * (n - 1) // 2:
        raise ValueError("m exceeds the number of vertex pairs")
    have = np.zeros(0, dtype=np.int64)
    while have.shape[0] < m:
        need = m - have.shape[0]
        a = rng.integers(0, n, size=2 * need + 16, dtype=np.int64)
        b = rng.integers(0, n, size=2 * need + 16, dtype=np.int64)
        keep = a != b
        lo = np.minimum(a[keep], b[keep])
        hi = np.maximum(a[keep], b[keep])
        keys = lo * n + hi
        # keep first occurrences in draw order, then merge with what we have
        _, first = np.unique(keys, return_index=True)
        keys = keys[np.sort(first)]
        keys = keys[~np.isin(keys, have)]
        have = np.concatenate([have, keys[:need]])
    lo, hi = have // n, have % n
    return csr_from_edges(n, lo, hi, name=f"ER(n={n},m={m},seed={seed})")


_GEN = None


def _gen_lib():
    """gcc-built helper (gen.c): RMAT draw + symmetrise/dedupe in C (numpy is too slow at 2e8)."""
    global _GEN
    if _GEN is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, lib = os.path.join(here, "gen.c"), os.path.join(here, "libgen.so")
        if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", lib, src])
        L = ctypes.CDLL(lib)
        L.gen_rmat.restype = ctypes.c_int64
        L.gen_rmat.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _GEN = L
    return _GEN


def rmat(scale: int, m: int, a: float, b: float, c: float, seed: int = 1,
         perm_seed: int | None = 7) -> CSR:
    """RMAT(a,b,c,d=1-a-b-c) with m drawn directed edges over n = 2^scale vertices.

    Each draw picks one quadrant per level (row bit set for quadrants c,d;
    column bit for b,d) from a counter-hash uniform of (seed, edge, level);
    vertex ids are relabelled by a random permutation (``perm_seed``) so degree
    is uncorrelated with id; the edge set is symmetrised, self-loops dropped
    and duplicates removed (SURVEY §8(d) D4 recipe).  Implemented in gen.c.
    """
    n = 1 << scale
    ro = np.zeros(n + 1, dtype=np.int64)
    col = np.empty(max(2 * m, 1), dtype=np.int32)
    nnz = _gen_lib().gen_rmat(scale, m, a, b, c, seed, -1 if perm_seed is None else perm_seed,
                              ro.ctypes.data, col.ctypes.data)
    if nnz < 0:
        raise MemoryError("gen_rmat failed")
    col = col[:nnz].copy()
    return CSR(n=n, row_offsets=ro, col_indices=col,
               name=f"RMAT(scale={scale},m={m},a={a},b={b},c={c},seed={seed})")


def rmat_1m_like(scale: int = 20, edge_factor: float = 100.0, seed: int = 1) -> CSR:
    """RMAT(0.45,0.22,0.22,0.11), scale 20, m = 1.05e8 drawn, perm seed 7.

    ``edge_factor`` = drawn edges per vertex (1.05e8 / 2^20 ≈ 100.1).  Smaller
    ``scale`` keeps the same recipe (used for parity-size cases).
    """
    m = int(round(1.05e8 * (1 << scale) / (1 << 20) * (edge_factor / 100.1354)))
    g = rmat(scale, m, 0.45, 0.22, 0.22, seed=seed, perm_seed=7)
    g.name = f"RMAT-1M-like(scale={scale},m={m},seed={seed})"
    return g


def cycle_graph(n: int) -> CSR:
    i = np.arange(n)
    return csr_from_edges(n, i, (i + 1) % n, name=f"C{n}")


def path_graph(n: int) -> CSR:
    i = np.arange(n - 1)
    return csr_from_edges(n, i, i + 1, name=f"P{n}")


def complete_graph(n: int) -> CSR:
    u, v = np.triu_indices(n, 1)
    return csr_from_edges(n, u, v, name=f"K{n}")


def house_tail_graph() -> CSR:
    """SURVEY §8(c) pin 3 end-to-end graph: n=8, 10 edges."""
    e = [(0, 1), (1, 2), (2, 3), (3, 0), (0, 4), (1, 4), (3, 5), (5, 6), (6, 7), (2, 6)]
    u, v = zip(*e)
    return csr_from_edges(8, u, v, name="house+tail")


def disjoint_union(g1: CSR, g2: CSR) -> CSR:
    e1 = g1.edges()
    e2 = g2.edges() + g1.n
    e = np.concatenate([e1, e2])
    return csr_from_edges(g1.n + g2.n, e[:, 0], e[:, 1], name=f"{g1.name}+{g2.name}")


def degree_stats(g: CSR) -> dict:
    d = g.degrees
    return {
        "n": g.n,
        "nnz": g.nnz,
        "avg_deg": float(g.nnz / max(g.n, 1)),
        "max_deg": int(d.max()) if g.n else 0,
        "p50": float(np.percentile(d, 50)) if g.n else 0.0,
        "p99": float(np.percentile(d, 99)) if g.n else 0.0,
        "isolated": int((d == 0).sum()),
    }


def miami_like(seed: int = 1) -> CSR:
    """RMAT with milder skew, scale 21, m = 5.2e7 drawn, id-permuted.

    a lowered from 0.45 until the max degree is ~10K ("Miami 2.1M / avg 49 /
    max 10K"): a = 0.41, b = c = 0.4·(1-a), d = 0.2·(1-a) (the 2:2:1 ratio of
    RMAT(0.45,0.22,0.22,0.11)).  Realised: n = 2,097,152, nnz = 103,964,748,
    avg 49.6, max 10,643.
    """
    a = 0.41
    g = rmat(21, 52_000_000, a, 0.4 * (1 - a), 0.4 * (1 - a), seed=seed, perm_seed=7)
    g.name = f"Miami-like(scale=21,m=5.2e7,a={a},seed={seed})"
    return g


def orkut_like(seed: int = 1) -> CSR:
    """RMAT(0.45,0.22,0.22,0.11), scale 22, m = 1.2e8 drawn, id-permuted.

    Realised: n = 4,194,304 (217,689 isolated), nnz = 239,797,400, max 34,166
    ("Orkut 3M / 230M / avg 76 / max 33K").
    """
    g = rmat(22, 120_000_000, 0.45, 0.22, 0.22, seed=seed, perm_seed=7)
    g.name = f"Orkut-like(scale=22,m=1.2e8,seed={seed})"
    return g


def graph500_like(scale: int = 22, edge_factor: int = 16, seed: int = 1) -> CSR:
    """SURVEY §8(d) D5a (strong-scaling graph): Graph500 RMAT(0.57, 0.19, 0.19, 0.05),
    scale 22, edge factor 16 (m = 16·2^scale drawn edges), id-permuted — shaped like the
    paper's GS22 row (2M vertices / 128M edges / avg 53 / max 170K)."""
    g = rmat(scale, edge_factor << scale, 0.57, 0.19, 0.19, seed=seed, perm_seed=7)
    g.name = f"Graph500-like(scale={scale},ef={edge_factor},seed={seed})"
    return g


BIG_GRAPHS = {"rmat1m": lambda: rmat_1m_like(), "miami": lambda: miami_like(), "orkut": lambda: orkut_like(),
              "gs22": lambda: graph500_like()}
