"""Python face of the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with the
CUDA path (paper_2009_11665_b200/) and imports nothing from it.

* ``colors``/``count``: ctypes calls into liboracle.so (sg2v_oracle.c).
* ``alpha``: |Aut(T)| of the UNROOTED template (reading "α", SURVEY §8(c);
  P:153 "number of automorphisms of T_0"), by brute force over k! vertex
  permutations for k <= 8 and by the AHU canonical-form product above that.
* ``colorful_probability``: P = k!/k^k.
* ``estimate``: finalCount[j] = colorful_j/(P·α), averaged.

"parity unpinned" items: none in this module (see tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sg2v_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

FORM_TWO_STAGE, FORM_ALG2 = 0, 1
ARITH_U64, ARITH_F64 = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -fopenmp (no fast-math: IEEE RN-even)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        vp = ctypes.c_void_p
        L.oracle_color.restype = i32
        L.oracle_color.argtypes = [u64, i64, i64, i32]
        L.oracle_colors.restype = None
        L.oracle_colors.argtypes = [u64, i64, i64, i32, vp]
        L.oracle_binom.restype = i64
        L.oracle_binom.argtypes = [i32, i32]
        L.oracle_rank.restype = i32
        L.oracle_rank.argtypes = [i32, vp, i32]
        L.oracle_partition.restype = i32
        L.oracle_partition.argtypes = [i32, vp, i32, vp]
        L.oracle_spmm_f64.restype = None
        L.oracle_spmm_f64.argtypes = [i64, vp, vp, vp, i64, vp]
        L.oracle_ema_f64.restype = None
        L.oracle_ema_f64.argtypes = [i64, vp, vp, vp]
        L.oracle_count.restype = i32
        L.oracle_count.argtypes = [i64, vp, vp, i32, vp, i32, vp, i32, i32,
                                   vp, vp, vp, vp, vp]
        L.oracle_count_ex.restype = i32
        L.oracle_count_ex.argtypes = [i64, vp, vp, i32, vp, i32, vp, i32, i32,
                                      vp, vp, vp, vp, vp, vp]
        L.oracle_set_threads.restype = None
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_get_threads.restype = i32
        L.oracle_get_threads.argtypes = []
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(nt: int) -> None:
    lib().oracle_set_threads(int(nt))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def color(seed: int, j: int, v: int, k: int) -> int:
    return int(lib().oracle_color(seed & (2**64 - 1), j, v, k))


def colors(seed: int, j: int, n: int, k: int) -> np.ndarray:
    out = np.empty(max(n, 1), dtype=np.uint8)
    lib().oracle_colors(seed & (2**64 - 1), j, n, k, _ptr(out))
    return out[:n]


def rank(k: int, colour_set) -> int:
    s = np.ascontiguousarray(sorted(colour_set), dtype=np.int32)
    return int(lib().oracle_rank(k, _ptr(s), len(s)))


def partition(k: int, edges, root: int = 0):
    """SPEC-rule chain: list of (size, root, active, passive), children first."""
    if len(edges) != k - 1:
        raise ValueError("a tree on k vertices has k-1 edges")
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1)) if edges else np.zeros(1, np.int32)
    out = np.zeros(4 * 2 * max(k, 1), dtype=np.int32)
    m = lib().oracle_partition(k, _ptr(e), root, _ptr(out))
    if m < 0:
        raise ValueError(f"oracle_partition error {m}")
    return [tuple(int(x) for x in out[4 * i:4 * i + 4]) for i in range(m)]


def spmm(csr, X: np.ndarray) -> np.ndarray:
    """Alg. 4 / Alg. 6 semantics: B = A_G · X for an n x w fp64 block."""
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(csr.n, -1)
    B = np.empty_like(X)
    lib().oracle_spmm_f64(csr.n, _ptr(csr.row_offsets), _ptr(csr.col_indices), _ptr(X), X.shape[1], _ptr(B))
    return B


def ema(dst: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    dst = np.ascontiguousarray(dst, dtype=np.float64).copy()
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    lib().oracle_ema_f64(dst.shape[0], _ptr(dst), _ptr(a), _ptr(b))
    return dst


def count(csr, k: int, edges, cols: np.ndarray, root: int = 0, form: int = FORM_TWO_STAGE,
          arith: int = ARITH_U64, rows: bool = False, live: bool = False):
    """One colouring.  U64 -> int (mod 2^64); F64 -> (float, max_intermediate).

    With rows=True also returns the per-vertex values Σ_C M_0(i, I_C).
    With live=True (F64) the tuple gains max_live after max_intermediate: the max over
    every non-top table entry and every live B entry (I_p ∌ c(i)), the top's B
    excluded when its active child is a leaf — the entries any F32 layout holds in F32.
    """
    n = csr.n
    if len(edges) != k - 1:
        raise ValueError("a tree on k vertices has k-1 edges")
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1)) if len(edges) else np.zeros(1, np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.uint8)
    if cols.shape[0] < max(n, 1):
        cols = np.concatenate([cols, np.zeros(max(n, 1) - cols.shape[0], np.uint8)])
    ro = np.ascontiguousarray(csr.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(csr.col_indices, dtype=np.int32)
    if ci.shape[0] == 0:
        ci = np.zeros(1, np.int32)
    tot_u = np.zeros(1, np.uint64)
    tot_f = np.zeros(1, np.float64)
    vmax = np.zeros(1, np.float64)
    vlive = np.zeros(1, np.float64)
    rows_u = np.zeros(max(n, 1), np.uint64) if (rows and arith == ARITH_U64) else None
    rows_f = np.zeros(max(n, 1), np.float64) if (rows and arith == ARITH_F64) else None
    rc = lib().oracle_count_ex(n, _ptr(ro), _ptr(ci), k, _ptr(e), root, _ptr(cols), form, arith,
                               _ptr(tot_u), _ptr(rows_u) if rows_u is not None else None,
                               _ptr(tot_f), _ptr(rows_f) if rows_f is not None else None, _ptr(vmax),
                               _ptr(vlive) if live else None)
    if rc != 0:
        raise ValueError({-1: "EINVAL", -2: "ENOTTREE", -3: "ENOMEM"}.get(rc, rc))
    if arith == ARITH_U64:
        return (int(tot_u[0]), rows_u[:n]) if rows else int(tot_u[0])
    head = (float(tot_f[0]), float(vmax[0])) + ((float(vlive[0]),) if live else ())
    return head + (rows_f[:n],) if rows else head


# ---------------------------------------------------------------------------
# Normalisation: P = k!/k^k, α = |Aut(T)| unrooted.
# ---------------------------------------------------------------------------
def colorful_probability(k: int) -> Fraction:
    return Fraction(math.factorial(k), k ** k)


def alpha_bruteforce(k: int, edges) -> int:
    es = {frozenset(e) for e in edges}
    cnt = 0
    for p in itertools.permutations(range(k)):
        if all(frozenset((p[a], p[b])) in es for a, b in edges):
            cnt += 1
    return cnt


def _ahu(adj, v, parent):
    """(canonical string, |Aut| of the subtree rooted at v)."""
    kids = [_ahu(adj, c, v) for c in adj[v] if c != parent]
    kids.sort()
    aut = 1
    for _, a in kids:
        aut *= a
    i = 0
    while i < len(kids):
        j = i
        while j < len(kids) and kids[j][0] == kids[i][0]:
            j += 1
        aut *= math.factorial(j - i)
        i = j
    return "(" + "".join(c for c, _ in kids) + ")", aut


def alpha_ahu(k: int, edges) -> int:
    if k <= 2:
        return 1 if k == 1 else 2
    adj = [[] for _ in range(k)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)
    # centre(s) by repeatedly stripping leaves
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
    centres = layer  # the last layer of leaves left standing is the centre (1 or 2 vertices)
    if len(centres) == 1:
        return _ahu(adj, centres[0], -1)[1]
    a, b = centres
    ca, aa = _ahu(adj, a, b)
    cb, ab = _ahu(adj, b, a)
    return aa * ab * (2 if ca == cb else 1)


def alpha(k: int, edges) -> int:
    return alpha_bruteforce(k, edges) if k <= 8 else alpha_ahu(k, edges)


def final_count(colorful: int | float, k: int, edges) -> float:
    """finalCount[j] = colorful_j / (P·α)."""
    return float(Fraction(int(colorful)) / (colorful_probability(k) * alpha(k, edges))) \
        if isinstance(colorful, int) else float(colorful) / (float(colorful_probability(k)) * alpha(k, edges))


def run(csr, k: int, edges, seed: int, n_iter: int, iter_offset: int = 0, arith: int = ARITH_U64,
        root: int = 0):
    """Per-colouring colorful counts for j = iter_offset .. iter_offset+n_iter-1."""
    out = []
    for j in range(iter_offset, iter_offset + n_iter):
        c = colors(seed, j, csr.n, k)
        out.append(count(csr, k, edges, c, root=root, arith=arith))
    return out
