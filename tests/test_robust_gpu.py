"""Cross-and-bouquet solving on the B200 — the scenarios of the reference's
test_robust.py (TestExtendedDictionary, TestCabSolve) restated against the
drop-in cab_solve / ExtendedDictionary: exact recovery by the equality
backends, agreement of the penalized backends, the implicit [A, sI] operator
against the materialised stack, e_weight pricing, clean-data behaviour."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _corrupted(seed, n=120, d=60, k=6, frac=0.2, amp=1.0):
    A = oracle.gaussian_dict(d, n, seed)
    x0 = oracle.sparse_signal(n, k, seed)
    clean = A @ x0
    s = float(np.max(np.abs(clean)))
    bad, mask = oracle.corrupt(clean, frac, -amp * s, amp * s, seed + 100000)
    return A, x0, clean, bad, mask


def _cfg(**kw):
    from paper_1007_3753_b200.model import SolverConfig
    return SolverConfig(**kw)


def test_extended_dictionary_shape_mode_and_errors():
    from paper_1007_3753_b200.robust import ExtendedDictionary
    rng = np.random.default_rng(0)
    ext = ExtendedDictionary(rng.standard_normal((8, 12)))
    assert ext.shape == (8, 20)
    assert ext.T.shape == (20, 8)
    assert ext.T.T is ext
    assert ext.mode == "cab"
    with pytest.raises(ValueError):
        ExtendedDictionary(np.ones(4))
    with pytest.raises(ValueError):
        ExtendedDictionary(np.ones((2, 3)), identity_scale=0.0)


@pytest.mark.parametrize("seed", range(6))
def test_extended_dictionary_adjoint_consistency(seed):
    from paper_1007_3753_b200.robust import ExtendedDictionary
    rng = np.random.default_rng(seed)
    d, n = 4 + seed % 7, 3 + seed % 11
    ext = ExtendedDictionary(rng.standard_normal((d, n)), identity_scale=0.5 + rng.random())
    v = rng.standard_normal(n + d)
    u = rng.standard_normal(d)
    lhs = float(u @ (ext @ v))
    rhs = float((ext.T @ u) @ v)
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def test_cab_argument_errors():
    from paper_1007_3753_b200.robust import cab_solve
    with pytest.raises(ValueError):
        cab_solve(np.eye(3), np.ones(3), "magic", _cfg(tol=1e-6, max_iter=10))
    with pytest.raises(ValueError):
        cab_solve(np.eye(3), np.ones(3), "ist", _cfg(tol=1e-6, max_iter=10, options={"e_weight": -1.0}))


@pytest.mark.parametrize("backend", ["pdipa", "palm", "dalm"])
def test_equality_backends_recover_exactly(backend):
    from paper_1007_3753_b200.robust import cab_solve
    A, x0, clean, bad, mask = _corrupted(3)
    e0 = bad - clean
    x, e, _ = cab_solve(A, bad, backend, _cfg(tol=1e-8, max_iter=6000))
    assert np.linalg.norm(x - x0) <= 1e-6 * np.linalg.norm(x0)
    assert np.linalg.norm(e - e0) <= 1e-6 * max(np.linalg.norm(e0), 1.0)


def test_penalized_backends_agree():
    from paper_1007_3753_b200.robust import cab_solve
    A, x0, clean, bad, mask = _corrupted(3)
    cfg = _cfg(tol=1e-10, max_iter=8000)
    answers = [cab_solve(A, bad, name, cfg) for name in ("homotopy", "gp", "ist", "fista")]
    xr, er, _ = answers[0]
    for x, e, _ in answers[1:]:
        assert np.linalg.norm(x - xr) <= 1e-5 * (1.0 + np.linalg.norm(xr))
        assert np.linalg.norm(e - er) <= 1e-5 * (1.0 + np.linalg.norm(er))


def test_pure_corruption_lands_on_identity_block():
    from paper_1007_3753_b200.robust import cab_solve
    rng = np.random.default_rng(9)
    A = rng.standard_normal((40, 80))
    A /= np.linalg.norm(A, axis=0)
    b = np.zeros(40)
    spots = rng.choice(40, size=5, replace=False)
    b[spots] = 5.0 * rng.choice([-1.0, 1.0], size=5)
    x, e, _ = cab_solve(A, b, "pdipa", _cfg(tol=1e-8, max_iter=200))
    assert np.linalg.norm(e - b) <= 1e-6 * np.linalg.norm(b)
    assert np.linalg.norm(x) <= 1e-6 * np.linalg.norm(b)


def test_implicit_stack_matches_dense_lasso_and_e_weight():
    from paper_1007_3753_b200.model import ProblemInstance
    from paper_1007_3753_b200.robust import cab_solve
    from paper_1007_3753_b200.shrinkage import fista_solve
    A, x0, clean, bad, mask = _corrupted(5, n=60, d=30, k=3)
    lam = 1e-2 * float(np.max(np.abs(np.concatenate([A.T @ bad, bad]))))
    cfg = _cfg(tol=1e-10, max_iter=8000, lam=lam)
    x, e, _ = cab_solve(A, bad, "fista", cfg)
    res = fista_solve(ProblemInstance(np.hstack([A, np.eye(30)]), bad), cfg)
    np.testing.assert_allclose(x, res.x_star[:60], atol=1e-6)
    np.testing.assert_allclose(e, res.x_star[60:], atol=1e-6)
    # e_weight w prices the corruption block at lam * w: same optimum as [A, I / w]
    A, x0, clean, bad, mask = _corrupted(6, n=60, d=30, k=3)
    lam = 1e-2 * float(np.max(np.abs(A.T @ bad)))
    cfg = _cfg(tol=1e-10, max_iter=8000, lam=lam)
    x1, e1, _ = cab_solve(A, bad, "fista", cfg)
    xw, ew, _ = cab_solve(A, bad, "fista", _cfg(tol=1e-10, max_iter=8000, lam=lam, options={"e_weight": 2.0}))
    res = fista_solve(ProblemInstance(np.hstack([A, np.eye(30) / 2.0]), bad), cfg)
    np.testing.assert_allclose(xw, res.x_star[:60], atol=1e-6)
    np.testing.assert_allclose(ew, res.x_star[60:] / 2.0, atol=1e-6)
    assert np.sum(np.abs(ew)) < np.sum(np.abs(e1)) + 1e-12


@pytest.mark.parametrize("seed", [2700, 2701, 2702, 2703])
def test_clean_data_keeps_identity_block_negligible(seed):
    from paper_1007_3753_b200.robust import cab_solve
    A = oracle.gaussian_dict(30, 60, seed)
    b = A @ oracle.sparse_signal(60, 3, seed)
    x, e, _ = cab_solve(A, b, "homotopy", _cfg(tol=1e-8, max_iter=2000))
    assert np.sum(np.abs(e)) <= 1e-2 * np.sum(np.abs(b))
