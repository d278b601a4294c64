"""FISTA on the B200 vs the reference (golden fixtures) and the oracle.

Mirrors the reference's own FISTA tests (test_shrinkage.py:164-358) through
the drop-in entry points.
"""

import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, case_inputs, ids_for, make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shr():
    from paper_1007_3753_b200 import shrinkage
    return shrinkage


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


@pytest.mark.parametrize("cid", ids_for("fista"))
def test_fista_matches_reference_fp64(shr, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = shr.fista_solve(P, make_config(case, A, b))
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    assert res.notes == ()


@pytest.mark.parametrize("cid", [c for c in ids_for("fista") if not c.startswith("fista_small_budget")])
def test_fista_matches_reference_fp32(shr, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = shr.fista_solve(P, make_config(case, A, b, dtype="float32"))
    # fp32 dictionary storage (f64 accumulation): 1e-4 gate, iteration count may move
    from tests.gpu_util import rel_err, support
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])
    assert res.converged == bool(gold["converged"])


def test_fista_matches_oracle_random_small(shr, model):
    rng = np.random.default_rng(2024)
    for trial in range(6):
        d, n = int(rng.integers(5, 60)), int(rng.integers(5, 120))
        A = rng.standard_normal((d, n))
        b = rng.standard_normal(d)
        lam = float(rng.uniform(0.01, 0.3)) * float(np.max(np.abs(A.T @ b)))
        ref = oracle.fista(A, b, lam=lam, tol=1e-8, max_iter=3000)
        P = model.ProblemInstance(A, b)
        res = shr.fista_solve(P, model.SolverConfig(lam=lam, tol=1e-8, max_iter=3000))
        assert res.iterations == ref.iterations, (trial, d, n)
        assert np.linalg.norm(res.x_star - ref.x) <= 1e-9 * max(1.0, np.linalg.norm(ref.x))


def test_fista_zero_rhs(shr, model):
    r = shr.fista_solve(model.ProblemInstance(np.eye(4), np.zeros(4)), model.SolverConfig(lam=0.1))
    assert r.converged and r.iterations == 0
    assert np.all(r.x_star == 0.0)
    assert len(r.trace) == 1 and r.trace[0].residual_norm == 0.0


def test_fista_rejects_nonpositive_lambda(shr, model):
    P = model.ProblemInstance(np.eye(3), np.ones(3))
    with pytest.raises(ValueError):
        shr.fista_solve(P, model.SolverConfig(lam=0.0))


def test_fista_orthonormal_closed_form(shr, model):
    rng = np.random.default_rng(31)
    Q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    b = rng.standard_normal(8)
    r = shr.fista_solve(model.ProblemInstance(Q, b), model.SolverConfig(lam=0.25, tol=1e-9))
    assert r.converged
    assert np.max(np.abs(r.x_star - oracle.soft(Q.T @ b, 0.25))) <= 1e-6


def test_fista_step_invariants_with_observer(shr, model):
    # test_shrinkage.py:303-319 through the per-iteration observer path
    from tests.golden.cases import build_inputs
    for seed in (1400, 1401, 1402, 1403):
        A, b, gt = build_inputs(dict(kind="genspec", n=40, d=20, k=1 + seed % 5, seed=seed, sigma=0.02))
        P = model.ProblemInstance(A, b)
        lam = 0.05 * float(np.max(np.abs(A.T @ b)))
        log = []
        res = shr.fista_solve(P, model.SolverConfig(lam=lam, tol=1e-7, max_iter=2000),
                              observer=lambda st, y, la: log.append((st, y, la)))
        assert len(log) == res.iterations
        Ls = [st.L for st, _, _ in log]
        assert all(a <= c for a, c in zip(Ls, Ls[1:]))
        for st, y, la in log:
            assert st.t_cur ** 2 - st.t_cur <= st.t_prev ** 2
            F = model.objective(st.x_cur, P, la)
            r_y = A @ y - b
            g_y = A.T @ r_y
            dl = st.x_cur - y
            Qm = 0.5 * float(r_y @ r_y) + float(g_y @ dl) + 0.5 * st.L * float(dl @ dl) \
                + la * float(np.sum(np.abs(st.x_cur)))
            assert F <= Qm + 1e-9 * max(1.0, abs(F))
        ref = oracle.fista(A, b, lam=lam, tol=1e-7, max_iter=2000)
        assert res.iterations == ref.iterations
        np.testing.assert_allclose(res.x_star, ref.x, atol=1e-10)


def test_backtrack_scalar_case(shr, model):
    P = model.ProblemInstance(np.array([[2.0]]), np.array([2.0]))
    L, _ = shr.backtrack_L(np.array([0.0]), 1.0, 2.0, 0.0, P)
    assert L == 4.0


def test_backtrack_matches_oracle(shr, model):
    rng = np.random.default_rng(14)
    for _ in range(10):
        A = rng.standard_normal((8, 12))
        b = rng.standard_normal(8)
        P = model.ProblemInstance(A, b)
        y = rng.standard_normal(12)
        lam = float(rng.uniform(0.01, 1.0))
        L, xn = shr.backtrack_L(y, 0.5, 1.5, lam, P)
        Lr, xr = oracle.backtrack(A, b, y, 0.5, 1.5, lam)
        assert L == Lr
        np.testing.assert_allclose(xn, xr, atol=1e-12)


def test_backtrack_nonfinite_breaks_down(shr, model):
    from paper_1007_3753_b200.exceptions import NumericalBreakdownError
    P = model.ProblemInstance(np.array([[1.0]]), np.array([1.0]))
    with pytest.raises(NumericalBreakdownError):
        shr.backtrack_L(np.array([np.nan]), 1.0, 2.0, 0.1, P)


def test_spectral_norm_matches_oracle():
    from paper_1007_3753_b200 import device
    rng = np.random.default_rng(5)
    for shape in ((30, 50), (50, 30), (200, 700)):
        A = rng.standard_normal(shape)
        D = device.DeviceDictionary(A)
        assert D.norm_sq() == pytest.approx(oracle.power_norm_sq(A), rel=1e-9)


def test_fista_budget_cap(shr, model):
    rng = np.random.default_rng(19)
    A = rng.standard_normal((20, 40))
    A /= np.linalg.norm(A, axis=0)
    P = model.ProblemInstance(A, rng.standard_normal(20))
    r = shr.fista_solve(P, model.SolverConfig(lam=0.05, max_iter=2))
    assert not r.converged and r.iterations == 2


def test_fista_cab_matches_reference(model):
    from paper_1007_3753_b200.robust import cab_solve
    from tests.gpu_util import rel_err
    case, A, b, gt, gold = case_inputs("cab_small_fista")
    x, e, res = cab_solve(A, b, "fista", make_config(case, A, b))
    gw = dict(gold)
    gw["x"] = gold["w"]
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gw, 1e-6)
    assert rel_err(x, gold["x"]) <= 1e-6
