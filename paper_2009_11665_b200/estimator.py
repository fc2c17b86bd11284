"""Estimator extras around the colour-coding path.

Host-side arithmetic on the per-colouring counts the library returns; nothing
here touches the hot path.

* required_iterations: N = ⌈e^k · ln(1/δ) / ε²⌉ — Alg. 1 line 1 (P:146,
  N = O(e^k log(1/δ)/ε²)) with leading constant 1, N >= 1.
* std_error: sample standard deviation of finalCount[j] / √N.
* treelet_distribution: normalised estimates over a family of same-size trees
  (Fig. 1).
* compare_distributions: pairwise L1 distances (the paper names no
  metric).
"""
from __future__ import annotations

import math

import numpy as np


def required_iterations(epsilon: float, delta: float, k: int) -> int:
    if not (epsilon > 0 and 0 < delta < 1) or k < 1:
        raise ValueError("need epsilon > 0, 0 < delta < 1, k >= 1")
    return max(1, math.ceil(math.exp(k) * math.log(1.0 / delta) / epsilon ** 2 - 1e-12))


def final_counts(colorful, P: float, alpha: float) -> np.ndarray:
    """finalCount[j] = colorful_j / (P·α)."""
    return np.asarray(colorful, dtype=np.float64) / (P * alpha)


def std_error(colorful, P: float, alpha: float) -> float:
    f = final_counts(colorful, P, alpha)
    if f.size < 2:
        return float("nan")
    return float(np.std(f, ddof=1) / math.sqrt(f.size))


def treelet_distribution(estimates) -> np.ndarray:
    """estimates / Σ estimates; all-zero when the sum is 0."""
    e = np.asarray(estimates, dtype=np.float64)
    s = e.sum()
    return e / s if s > 0 else np.zeros_like(e)


def compare_distributions(dists) -> np.ndarray:
    """Symmetric matrix of L1 distances with zero diagonal."""
    d = [np.asarray(x, dtype=np.float64) for x in dists]
    m = len(d)
    if any(x.shape != d[0].shape for x in d):
        raise ValueError("distributions must have equal length")
    out = np.zeros((m, m))
    for a in range(m):
        for b in range(a + 1, m):
            out[a, b] = out[b, a] = float(np.abs(d[a] - d[b]).sum())
    return out


def estimate_distribution(graph, templates, n_iter: int, seed: int, precision: str = "f64", **kw):
    """Treelet distribution of `templates` (same k) on `graph` through sg2v_count_batch."""
    from .sg2v import count_batch
    est, colorful = count_batch(graph, templates, n_iter, seed, precision=precision, **kw)
    return treelet_distribution(est), est, colorful
