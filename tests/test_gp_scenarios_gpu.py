"""GPSR / TNIPM scenarios of the reference's test_gradient_projection.py not
pinned by golden fixtures: the exact line-search step, agreement with the
path solver and with each other, budgets and truncation, stopping rules,
the first interior step, and the KKT contract / direction invariants."""

import numpy as np
import pytest

from tests.golden.cases import build_inputs

pytestmark = pytest.mark.gpu


def _gen(n, d, k, seed, sigma=0.0):
    from paper_1007_3753_b200.model import ProblemInstance
    A, b, x0 = build_inputs(dict(kind="genspec", n=n, d=d, k=k, seed=seed, sigma=sigma))
    return ProblemInstance(A, b, ground_truth=x0)


def _cfg(**kw):
    from paper_1007_3753_b200.model import SolverConfig
    return SolverConfig(**kw)


def _split_obj(z, A, b, lam):
    n = z.shape[0] // 2
    r = A @ (z[:n] - z[n:]) - b
    return 0.5 * float(r @ r) + lam * float(np.sum(z))


def _split_grad(z, A, b, lam):
    n = z.shape[0] // 2
    gx = A.T @ (A @ (z[:n] - z[n:]) - b)
    return np.concatenate([gx + lam, lam - gx])


def test_step_size_cases():
    from paper_1007_3753_b200.gradient_projection import gpsr_direction, gpsr_step_size
    A = np.array([[1.0], [1.0]])
    assert gpsr_step_size(np.array([1.0, 0.0]), A) == 0.5
    assert gpsr_step_size(np.array([1.0, 1.0]), A) == 1e8
    with pytest.raises(ValueError):
        gpsr_step_size(np.zeros(4), np.eye(2))
    rng = np.random.default_rng(31)
    for _ in range(20):
        A = rng.standard_normal((6, 4))
        b = rng.standard_normal(6)
        z = np.abs(rng.standard_normal(8)) * (rng.random(8) > 0.4)
        g = gpsr_direction(z, _split_grad(z, A, b, 0.3))
        if float(g @ g) == 0.0:
            continue
        alpha = gpsr_step_size(g, A)
        grid = np.linspace(0.0, 2.0 * alpha, 2001)
        best = grid[int(np.argmin([_split_obj(z - a * g, A, b, 0.3) for a in grid]))]
        assert abs(best - alpha) <= grid[1] - grid[0] + 1e-15


def _small_lambda_problem(seed):
    from paper_1007_3753_b200.model import ProblemInstance
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((100, 200)) / np.sqrt(100)
    x_true = np.zeros(200)
    x_true[rng.choice(200, 10, replace=False)] = rng.standard_normal(10)
    return ProblemInstance(A, A @ x_true)


def test_gpsr_matches_homotopy_at_small_lambda():
    from paper_1007_3753_b200.gradient_projection import gpsr_solve
    from paper_1007_3753_b200.homotopy import homotopy_solve
    from paper_1007_3753_b200.model import objective
    P = _small_lambda_problem(5)
    lam = 1e-3 * float(np.max(np.abs(P.A.T @ P.b)))
    ref = homotopy_solve(P, lam, _cfg(tol=1e-10, max_iter=5000))
    res = gpsr_solve(P, lam, _cfg(tol=1e-7, max_iter=50000))
    assert res.converged
    F_ref = objective(ref.x_star, P, lam)
    assert abs(objective(res.x_star, P, lam) - F_ref) <= 1e-6 * abs(F_ref)


def test_tnipm_matches_gpsr():
    from paper_1007_3753_b200.gradient_projection import gpsr_solve, tnipm_solve
    from paper_1007_3753_b200.model import objective
    P = _small_lambda_problem(6)
    lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
    F_gp = objective(gpsr_solve(P, lam, _cfg(tol=1e-7, max_iter=50000)).x_star, P, lam)
    res = tnipm_solve(P, lam, _cfg(tol=1e-7, max_iter=500))
    assert res.converged
    assert abs(objective(res.x_star, P, lam) - F_gp) <= 1e-5 * abs(F_gp)


def test_budgets_truncation_and_stopping_rule():
    from paper_1007_3753_b200.gradient_projection import gpsr_solve, tnipm_solve
    from paper_1007_3753_b200.model import ProblemInstance, StoppingRule
    res = gpsr_solve(_gen(60, 30, 5, 10), None, _cfg(tol=1e-12, max_iter=3))
    assert not res.converged and res.iterations == 3 and len(res.trace) == 4
    res = tnipm_solve(_gen(60, 30, 5, 11), None, _cfg(tol=1e-12, max_iter=2))
    assert not res.converged and res.iterations == 2
    small = np.abs(res.x_star) <= 1e-7 * float(np.max(np.abs(res.x_star)))
    assert np.all(res.x_star[small] == 0.0)
    rng = np.random.default_rng(12)
    A = rng.standard_normal((20, 40)) / np.sqrt(20)
    P = ProblemInstance(A, rng.standard_normal(20))
    lam = 0.1 * float(np.max(np.abs(A.T @ P.b)))
    res = gpsr_solve(P, lam, _cfg(stopping=StoppingRule(kind="relative-objective", threshold=0.5)))
    assert res.converged and res.iterations <= 3


def test_tnipm_interior_start_takes_a_clean_first_step():
    from paper_1007_3753_b200.gradient_projection import tnipm_solve
    seen = []
    tnipm_solve(_gen(30, 15, 3, 21), None, _cfg(max_iter=1), observer=seen.append)
    assert len(seen) == 1
    first = seen[0]
    assert np.all(np.abs(first.x) < first.u)
    assert np.all(np.isfinite(first.x)) and np.all(np.isfinite(first.u))


def test_gpsr_descent_and_direction_invariants():
    from paper_1007_3753_b200.gradient_projection import gpsr_direction, gpsr_solve
    total = 0
    for seed in range(1800, 1910):
        P = _gen(40, 20, 1 + seed % 5, seed, sigma=0.01)
        lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
        its = []
        res = gpsr_solve(P, lam, _cfg(tol=1e-7, max_iter=20000), observer=its.append)
        assert res.converged
        zs = [np.zeros(2 * P.n)] + [it.z for it in its]
        for z_prev, z_next in zip(zs, zs[1:]):
            assert np.all(z_next >= 0.0)
            grad = _split_grad(z_prev, P.A, P.b, lam)
            n = P.n
            dx = (z_next[:n] - z_next[n:]) - (z_prev[:n] - z_prev[n:])
            Adx = P.A @ dx
            dQ = float(grad @ (z_next - z_prev)) + 0.5 * float(Adx @ Adx)
            assert dQ <= 1e-15 * (1.0 + abs(_split_obj(z_prev, P.A, P.b, lam)))
            g_next = _split_grad(z_next, P.A, P.b, lam)
            assert float(gpsr_direction(z_next, g_next) @ g_next) >= 0.0
            total += 1
    assert total >= 100


def test_both_solvers_meet_the_kkt_contract():
    from paper_1007_3753_b200.gradient_projection import gpsr_solve, tnipm_solve
    from paper_1007_3753_b200.model import kkt_residual
    for seed in range(2200, 2255):
        P = _gen(50, 25, 1 + seed % 4, seed)
        lam = 1e-2 * float(np.max(np.abs(P.A.T @ P.b)))
        cfg = _cfg(tol=1e-6, max_iter=20000)
        for solver in (gpsr_solve, tnipm_solve):
            res = solver(P, lam, cfg)
            assert res.converged
            assert kkt_residual(res.x_star, P, lam) <= 10 * cfg.tol * lam
