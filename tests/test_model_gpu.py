"""Objective / KKT / default-lambda helpers on the device — the reference's
test_model.py objective and KKT scenarios (incl. its invariant properties)
restated against paper_1007_3753_b200.model, whose helpers evaluate A x and
A^T r through the solver library."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(rng, d=8, n=12):
    from paper_1007_3753_b200.model import ProblemInstance
    A = rng.standard_normal((d, n))
    A /= np.linalg.norm(A, axis=0)
    return ProblemInstance(A, rng.standard_normal(d))


def test_default_lambda():
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    P = ProblemInstance(np.eye(2), np.array([2.0, -5.0]))
    assert SolverConfig().resolved_lambda(P) == pytest.approx(0.05)


def test_objective_cases():
    from paper_1007_3753_b200 import model
    rng = np.random.default_rng(0)
    P = _problem(rng)
    assert model.objective(np.zeros(P.n), P, 0.3) == pytest.approx(0.5 * float(P.b @ P.b))
    E = model.ProblemInstance(np.eye(2), np.array([1.0, 0.0]))
    assert model.objective(np.array([1.0, 0.0]), E, 1.0) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        model.objective(np.zeros(P.n + 1), P, 0.1)


def test_objective_vs_extended_precision():
    from paper_1007_3753_b200 import model
    rng = np.random.default_rng(3)
    P = _problem(rng)
    x = rng.standard_normal(P.n)
    lam = 0.17
    r = np.asarray(P.b, np.longdouble) - np.asarray(P.A, np.longdouble) @ x
    want = 0.5 * float(np.sum(r * r)) + lam * float(np.sum(np.abs(np.asarray(x, np.longdouble))))
    assert model.objective(x, P, lam) == pytest.approx(want, rel=1e-13)


def test_kkt_cases():
    from paper_1007_3753_b200 import model, numerics
    rng = np.random.default_rng(9)
    Q, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    b = rng.standard_normal(6)
    xstar = numerics.soft_threshold(Q.T @ b, 0.4)
    assert model.kkt_residual(xstar, model.ProblemInstance(Q, b), 0.4) <= 1e-12
    P = _problem(np.random.default_rng(12))
    lmax = float(np.max(np.abs(P.A.T @ P.b)))
    assert model.kkt_residual(np.zeros(P.n), P, lmax * 1.01) == 0.0
    assert model.kkt_residual(np.zeros(P.n), P, 0.5 * lmax) == pytest.approx(0.5 * lmax)
    with pytest.raises(ValueError):
        model.kkt_residual(np.zeros(P.n), P, 0.0)


def test_objective_nonnegative_property():
    from paper_1007_3753_b200 import model
    rng = np.random.default_rng(50)
    for _ in range(60):
        P = _problem(rng, d=int(rng.integers(2, 10)), n=int(rng.integers(2, 14)))
        x = rng.standard_normal(P.n) * rng.uniform(0, 10)
        assert model.objective(x, P, rng.uniform(0, 2)) >= 0.0


def test_orthonormal_minimizer_property():
    """soft(Q^T b, lam) is the minimiser for orthonormal Q: KKT is zero and
    the point beats random perturbations (batched objective on the host)."""
    from paper_1007_3753_b200 import model, numerics
    rng = np.random.default_rng(51)
    for _ in range(40):
        n = int(rng.integers(2, 8))
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        b = rng.standard_normal(n)
        P = model.ProblemInstance(Q, b)
        lam = rng.uniform(0.1, 0.8)
        xstar = numerics.soft_threshold(Q.T @ b, lam)
        assert model.kkt_residual(xstar, P, lam) <= 1e-10
        fstar = model.objective(xstar, P, lam)
        deltas = rng.standard_normal((2000, n))
        deltas *= (rng.uniform(0, 1e-3, 2000) / np.linalg.norm(deltas, axis=1))[:, None]
        X = xstar[:, None] + deltas.T
        R = b[:, None] - Q @ X
        vals = 0.5 * np.sum(R * R, axis=0) + lam * np.sum(np.abs(X), axis=0)
        assert np.all(vals >= fstar - 1e-12)
