"""Estimator extras (host side) — SPEC examples S:150-152."""
import math

import numpy as np
import pytest

from paper_2009_11665_b200.estimator import (compare_distributions, required_iterations, std_error,
                                             treelet_distribution)
from sg2v_inputs import all_trees


def test_required_iterations_examples():
    assert required_iterations(1.0, 1 / math.e, 2) == 8          # ⌈e²⌉
    assert required_iterations(1.0, 1 / math.e, 1) == 3          # ⌈e⌉
    assert required_iterations(0.5, 0.1, 2) == 69                 # ⌈e²·ln10/0.25⌉
    assert required_iterations(0.3, 1 - 1e-15, 5) == 1            # δ→1: clamp to 1
    with pytest.raises(ValueError):
        required_iterations(0, 0.1, 3)


def test_distribution_examples():
    assert treelet_distribution([7.0]).tolist() == [1.0]
    assert treelet_distribution([3.0, 3.0]).tolist() == [0.5, 0.5]
    assert treelet_distribution([0.0, 0.0]).tolist() == [0.0, 0.0]
    d = compare_distributions([[1, 0], [0, 1], [0.5, 0.5], [0.75, 0.25]])
    assert d[0, 1] == 2.0 and d[2, 3] == 0.5 and np.allclose(d, d.T) and np.all(np.diag(d) == 0)
    with pytest.raises(ValueError):
        compare_distributions([[1, 0], [1, 0, 0]])


def test_std_error():
    assert math.isnan(std_error([5.0], 0.5, 2))
    se = std_error([2.0, 4.0, 6.0, 8.0], 0.5, 1.0)
    f = np.array([4.0, 8.0, 12.0, 16.0])
    assert math.isclose(se, f.std(ddof=1) / 2)


def test_all_trees_counts():
    # OEIS A000055: number of trees on k unlabelled vertices
    assert [len(all_trees(k)) for k in range(1, 9)] == [1, 1, 1, 2, 3, 6, 11, 23]
    for e in all_trees(7):
        assert len(e) == 6
