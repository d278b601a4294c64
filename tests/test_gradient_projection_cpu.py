"""Iterate records and the masked GPSR direction (host logic, no GPU) —
test_gradient_projection.py:34-88 restated against the drop-in module."""

import numpy as np
import pytest

from paper_1007_3753_b200.gradient_projection import BarrierIterate, SplitIterate, gpsr_direction


def test_split_iterate():
    for bad in (np.array([1.0, -0.1]), np.array([1.0, 2.0, 3.0])):
        with pytest.raises(ValueError):
            SplitIterate(bad)
    it = SplitIterate(np.array([3.0, 0.0, 1.0, 2.0]))
    assert it.n == 2
    np.testing.assert_allclose(it.recombined(), [2.0, -2.0])


def test_barrier_iterate_requires_strict_interior():
    BarrierIterate(np.array([0.5]), np.array([1.0]), 2.0)
    with pytest.raises(ValueError):
        BarrierIterate(np.array([1.0]), np.array([1.0]), 2.0)
    with pytest.raises(ValueError):
        BarrierIterate(np.array([0.0]), np.array([1.0]), 0.0)


def test_direction_cases():
    eq = np.testing.assert_array_equal
    eq(gpsr_direction(np.array([0.0, 1.0]), np.array([-1.0, 2.0])), [-1.0, 2.0])
    eq(gpsr_direction(np.array([0.0, 0.0]), np.array([1.0, 1.0])), [0.0, 0.0])
    eq(gpsr_direction(np.array([2.0, 0.0]), np.array([3.0, -4.0])), [3.0, -4.0])
    eq(gpsr_direction(SplitIterate(np.array([0.0, 1.0])), np.array([5.0, -1.0])), [0.0, -1.0])
    with pytest.raises(ValueError):
        gpsr_direction(np.zeros(4), np.zeros(2))
