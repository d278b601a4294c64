"""Scalar host helpers of the shrinkage boundary (no GPU): the reference's
test_shrinkage.py BB / schedule / momentum scenarios restated against
paper_1007_3753_b200.shrinkage (the fused kernels apply the same rules on the
device; their parity is covered by the -m gpu golden tests)."""

import numpy as np
import pytest

from paper_1007_3753_b200.shrinkage import (ContinuationSchedule, bb_alpha, fista_t_next,
                                            objective_delta)


def test_bb_alpha_formula_and_clamps():
    assert bb_alpha([1.0, 1.0], [2.0, 4.0]) == 3.0
    assert bb_alpha([1.0, 0.0], [0.0, 1.0]) == 1e-30
    assert bb_alpha([1e-20, 0.0], [1e20, 0.0]) == 1e30


def test_bb_alpha_is_rayleigh_quotient_on_quadratics():
    rng = np.random.default_rng(8)
    for _ in range(30):
        B = rng.standard_normal((6, 6))
        H = B @ B.T + 0.1 * np.eye(6)
        s = -0.01 * (H @ rng.standard_normal(6))
        assert bb_alpha(s, H @ s) == pytest.approx(float(s @ H @ s) / float(s @ s), rel=1e-12)


def test_schedule_validation_and_shapes():
    for args in ((1.0, 0.5, 0.0), (0.5, 0.5, 1.0), (1.0, 1.0, 0.5)):
        with pytest.raises(ValueError):
            ContinuationSchedule(*args)
    st = ContinuationSchedule(0.8, 0.5, 0.1).stages()
    assert len(st) == 5 and st[0] == 0.8 and st[-1] == 0.1
    assert all(a > b for a, b in zip(st, st[1:]))
    st = ContinuationSchedule(1000.0, 0.5, 1.0).stages()
    assert st[0] == 1000.0 and st[-1] == 1.0
    for prev, cur in zip(st, st[1:]):
        assert cur == max(0.5 * prev, 1.0)
    assert ContinuationSchedule(0.3, 0.5, 0.3).stages() == [0.3]


def test_t_next_values_and_invariants():
    assert fista_t_next(1.0) == pytest.approx(1.6180339887498949, rel=1e-15)
    assert fista_t_next(1.6180339887498949) == pytest.approx(2.193527085331054, rel=1e-12)
    t = 1.0
    for _ in range(3000):
        tn = fista_t_next(t)
        assert tn * tn - tn <= t * t and tn > t
        t = tn
    for t in np.random.default_rng(2).uniform(1.0, 1e6, 100):
        assert fista_t_next(float(t)) > t
    with pytest.raises(ValueError):
        fista_t_next(0.5)


def test_objective_delta_matches_direct_difference():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((7, 11))
    b = rng.standard_normal(7)
    lam = 0.3
    F = lambda v: 0.5 * float((b - A @ v) @ (b - A @ v)) + lam * float(np.abs(v).sum())
    for _ in range(20):
        x, c = rng.standard_normal(11), rng.standard_normal(11)
        g = A.T @ (A @ x - b)
        got = objective_delta(x, c, A @ x, A @ c, g, lam)
        assert got == pytest.approx(F(c) - F(x), rel=1e-10, abs=1e-10)
