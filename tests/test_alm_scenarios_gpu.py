"""PALM / DALM scenarios of the reference's test_alm.py not pinned by golden
fixtures, restated against the drop-in alm module: the two-variable LP value,
agreement with PDIPA and the path solver, the dense-spike regime, the
single-CG y-step mode, stopping rules and PALM/DALM l1-value agreement."""

import numpy as np
import pytest

from tests.golden.cases import build_inputs

pytestmark = pytest.mark.gpu


def _gen(n, d, k, seed, sigma=0.0):
    from paper_1007_3753_b200.model import ProblemInstance
    A, b, x0 = build_inputs(dict(kind="genspec", n=n, d=d, k=k, seed=seed, sigma=sigma))
    return ProblemInstance(A, b, ground_truth=x0)


def _two_var_lp():
    from paper_1007_3753_b200.model import ProblemInstance
    return ProblemInstance(np.array([[1.0, 1.0]]) / np.sqrt(2.0), np.array([np.sqrt(2.0)]))


def _cfg(**kw):
    from paper_1007_3753_b200.model import SolverConfig
    return SolverConfig(**kw)


def test_palm_two_variable_value():
    from paper_1007_3753_b200.alm import palm_solve
    res = palm_solve(_two_var_lp(), _cfg(tol=1e-8, max_iter=20000))
    assert res.converged
    assert abs(float(np.abs(res.x_star).sum()) - 2.0) <= 1e-6


def test_palm_matches_pdipa():
    from paper_1007_3753_b200.alm import palm_solve
    from paper_1007_3753_b200.pdipa import pdipa_solve
    P = _gen(200, 100, 5, 42)
    ref = pdipa_solve(P, _cfg(tol=1e-8, max_iter=200))
    res = palm_solve(P, _cfg(tol=1e-7, max_iter=20000))
    assert ref.converged and res.converged
    assert np.linalg.norm(res.x_star - ref.x_star) / np.linalg.norm(ref.x_star) <= 1e-4


def test_palm_budget_note():
    from paper_1007_3753_b200.alm import palm_solve
    res = palm_solve(_gen(100, 50, 4, 13), _cfg(tol=1e-12, max_iter=5))
    assert not res.converged and res.iterations <= 5
    assert "inner-iteration budget exhausted" in res.notes


def test_dalm_orthonormal_rows_matches_homotopy():
    from paper_1007_3753_b200.alm import dalm_solve
    from paper_1007_3753_b200.homotopy import homotopy_solve
    from paper_1007_3753_b200.model import ProblemInstance
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    A = Q[:20, :]
    x_true = np.zeros(40)
    x_true[[3, 11, 29]] = [1.2, -0.7, 0.4]
    P = ProblemInstance(A, A @ x_true)
    ref = homotopy_solve(P, 1e-10, _cfg(tol=1e-10, max_iter=1000))
    res = dalm_solve(P, _cfg(tol=1e-9, max_iter=2000))
    assert res.converged
    assert float(np.max(np.abs(res.x_star - ref.x_star))) <= 1e-6


def test_dalm_recovers_dense_spike_regime():
    from paper_1007_3753_b200.alm import dalm_solve
    P = _gen(2000, 1000, 200, 7)
    res = dalm_solve(P, _cfg(tol=1e-4, max_iter=3000, options={"beta": 0.004}))
    assert res.converged
    assert np.linalg.norm(res.x_star - P.ground_truth) / np.linalg.norm(P.ground_truth) <= 1e-3


def test_dalm_single_cg_mode():
    from paper_1007_3753_b200.alm import dalm_solve
    from paper_1007_3753_b200.model import ProblemInstance
    rng = np.random.default_rng(19)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    A = Q[:15, :]
    x_true = np.zeros(30)
    x_true[[2, 9]] = [1.0, -2.0]
    P = ProblemInstance(A, A @ x_true)
    exact = dalm_solve(P, _cfg(tol=1e-8, max_iter=2000))
    cg = dalm_solve(P, _cfg(tol=1e-8, max_iter=2000, options={"y_cg_step": True}))
    assert exact.converged and cg.converged
    np.testing.assert_allclose(cg.x_star, exact.x_star, atol=1e-10)
    P = _gen(120, 60, 6, 9)
    exact = dalm_solve(P, _cfg(tol=1e-7, max_iter=50000))
    cg = dalm_solve(P, _cfg(tol=1e-7, max_iter=50000, options={"y_cg_step": True}))
    assert exact.converged and cg.converged
    l1e, l1c = float(np.abs(exact.x_star).sum()), float(np.abs(cg.x_star).sum())
    assert abs(l1c - l1e) <= 1e-5 * l1e


def test_dalm_honors_stopping_rule():
    from paper_1007_3753_b200.alm import dalm_solve
    from paper_1007_3753_b200.model import StoppingRule
    rule = StoppingRule(kind="relative-estimate", threshold=0.9)
    res = dalm_solve(_gen(100, 50, 4, 23), _cfg(tol=1e-14, stopping=rule))
    assert res.converged and res.iterations <= 3


def test_palm_and_dalm_agree_on_the_l1_value():
    from paper_1007_3753_b200.alm import dalm_solve, palm_solve
    for seed in range(2600, 2700):
        P = _gen(100, 50, 1 + seed % 4, seed)
        rp = palm_solve(P, _cfg(tol=1e-7, max_iter=20000))
        rd = dalm_solve(P, _cfg(tol=1e-7, max_iter=20000, options={"beta": 0.2}))
        assert rp.converged and rd.converged
        l1p, l1d = float(np.abs(rp.x_star).sum()), float(np.abs(rd.x_star).sum())
        assert abs(l1p - l1d) <= 1e-4 * max(l1p, l1d)
