"""Shrinkage solvers on the B200 — the remaining scenarios of the reference's
test_shrinkage.py (objective agreement with the path solver, stopping rules,
the O(1/k^2) bound with exact L, shrinkage fixed points, backtracking
post-conditions, default schedule) restated against the drop-in API."""

import numpy as np
import pytest

import oracle
from tests.golden.cases import build_inputs

pytestmark = pytest.mark.gpu


def _path_problem():
    from paper_1007_3753_b200.model import ProblemInstance
    rng = np.random.default_rng(17)
    A = rng.standard_normal((100, 200))
    A /= np.linalg.norm(A, axis=0)
    x0 = np.zeros(200)
    x0[rng.choice(200, 10, replace=False)] = rng.standard_normal(10)
    P = ProblemInstance(A, A @ x0)
    return P, 0.01 * float(np.max(np.abs(A.T @ P.b)))


@pytest.mark.parametrize("which", ["ist", "fista"])
def test_matches_path_solver_objective(which):
    from paper_1007_3753_b200 import homotopy, model, shrinkage
    P, lam = _path_problem()
    F_ref = model.objective(homotopy.homotopy_solve(P, lam, model.SolverConfig()).x_star, P, lam)
    cfg = model.SolverConfig(lam=lam, tol=1e-7, max_iter=20000)
    r = shrinkage.ist_solve(P, None, cfg) if which == "ist" else shrinkage.fista_solve(P, cfg)
    assert r.converged
    assert abs(model.objective(r.x_star, P, lam) - F_ref) <= 1e-5 * abs(F_ref)


def test_ist_honors_stopping_rule():
    from paper_1007_3753_b200 import model, shrinkage
    rng = np.random.default_rng(21)
    A = rng.standard_normal((20, 40))
    A /= np.linalg.norm(A, axis=0)
    P = model.ProblemInstance(A, rng.standard_normal(20))
    lam = 0.1 * float(np.max(np.abs(A.T @ P.b)))
    rule = model.StoppingRule(kind="relative-objective", threshold=0.5)
    r = shrinkage.ist_solve(P, shrinkage.ContinuationSchedule(lam, 0.5, lam),
                            model.SolverConfig(lam=lam, stopping=rule))
    assert r.converged and r.iterations <= 3


def test_fista_objective_bound_with_exact_L():
    from paper_1007_3753_b200 import model, numerics, shrinkage
    rng = np.random.default_rng(23)
    A = rng.standard_normal((50, 100))
    A /= np.linalg.norm(A, axis=0)
    x0 = np.zeros(100)
    x0[rng.choice(100, 5, replace=False)] = rng.standard_normal(5)
    P = model.ProblemInstance(A, A @ x0)
    fixed = {"exact_L": True, "continuation": False}
    ref = shrinkage.fista_solve(P, model.SolverConfig(lam=0.05, tol=1e-15, max_iter=30000, options=fixed))
    F_star = model.objective(ref.x_star, P, 0.05)
    run = shrinkage.fista_solve(P, model.SolverConfig(lam=0.05, tol=1e-15, max_iter=300, options=fixed))
    L_f = numerics.spectral_norm_sq(A)
    dist0 = float(np.linalg.norm(ref.x_star)) ** 2
    assert len(run.trace) == 300
    for t in run.trace:
        assert t.objective - F_star <= 2.0 * L_f * dist0 / (t.iteration + 1) ** 2


def test_returned_solutions_are_shrinkage_fixed_points():
    from paper_1007_3753_b200 import model, numerics, shrinkage
    for seed in range(1600, 1606):
        A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=2, seed=seed, sigma=0.0))
        P = model.ProblemInstance(A, b)
        lam = 0.05 * float(np.max(np.abs(A.T @ b)))
        L = numerics.spectral_norm_sq(A) * 1.01
        cfg = model.SolverConfig(lam=lam, tol=1e-9, max_iter=20000)
        for r in (shrinkage.ist_solve(P, shrinkage.ContinuationSchedule(lam, 0.5, lam), cfg),
                  shrinkage.fista_solve(P, cfg)):
            assert r.converged
            assert model.kkt_residual(r.x_star, P, lam) <= 1e-8 * lam
            g = A.T @ (A @ r.x_star - b)
            step = oracle.soft(r.x_star - g / L, lam / L)
            assert np.linalg.norm(step - r.x_star) <= 1e-6 * max(1.0, np.linalg.norm(r.x_star))


def test_backtrack_postconditions_and_validation():
    from paper_1007_3753_b200 import model, numerics, shrinkage
    rng = np.random.default_rng(4)
    A = rng.standard_normal((10, 15))
    P = model.ProblemInstance(A, rng.standard_normal(10))
    L0 = numerics.spectral_norm_sq(A) * 1.01
    L, _ = shrinkage.backtrack_L(rng.standard_normal(15), L0, 2.0, 0.1, P)
    assert L == L0          # already a majoriser: no growth step
    rng = np.random.default_rng(14)
    for _ in range(10):
        A = rng.standard_normal((8, 12))
        b = rng.standard_normal(8)
        P = model.ProblemInstance(A, b)
        y = rng.standard_normal(12)
        lam = float(rng.uniform(0.01, 1.0))
        L, xn = shrinkage.backtrack_L(y, 0.5, 1.5, lam, P)
        r_y = A @ y - b
        dl = xn - y
        Qm = 0.5 * float(r_y @ r_y) + float((A.T @ r_y) @ dl) + 0.5 * L * float(dl @ dl) \
            + lam * float(np.abs(xn).sum())
        assert model.objective(xn, P, lam) <= Qm + 1e-9
    P = model.ProblemInstance(np.array([[1.0]]), np.array([1.0]))
    with pytest.raises(ValueError):
        shrinkage.backtrack_L(np.array([0.0]), 0.0, 2.0, 0.1, P)
    with pytest.raises(ValueError):
        shrinkage.backtrack_L(np.array([0.0]), 1.0, 1.0, 0.1, P)


def test_default_schedule_shape():
    from paper_1007_3753_b200 import model, shrinkage
    rng = np.random.default_rng(9)
    A = rng.standard_normal((10, 20))
    P = model.ProblemInstance(A, rng.standard_normal(10))
    cmax = float(np.max(np.abs(A.T @ P.b)))
    sch = shrinkage.default_schedule(P, 0.01 * cmax)
    assert sch.lambda_start == pytest.approx(0.9 * cmax)
    assert sch.lambda_target == 0.01 * cmax and sch.beta == 0.5
