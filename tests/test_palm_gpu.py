"""Primal ALM on the B200 vs the reference (golden fixtures) and the oracle
(test_alm.py:44-93, 219-240 through the drop-in)."""

import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, case_inputs, gold_notes, ids_for, make_config, rel_err, support

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def alm():
    from paper_1007_3753_b200 import alm
    return alm


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


@pytest.mark.parametrize("cid", ids_for("palm"))
def test_palm_matches_reference_fp64(alm, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = alm.palm_solve(P, make_config(case, A, b))
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    assert res.notes == gold_notes(gold)


@pytest.mark.parametrize("cid", [c for c in ids_for("palm") if c.startswith("cfg")])
def test_palm_matches_reference_fp32(alm, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = alm.palm_solve(P, make_config(case, A, b, dtype="float32"))
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])


def test_palm_zero_data(alm, model):
    r = alm.palm_solve(model.ProblemInstance(np.eye(3), np.zeros(3)), model.SolverConfig())
    assert r.converged and r.iterations == 0 and np.all(r.x_star == 0)


def test_palm_rejects_bad_penalty_options(alm, model):
    P = model.ProblemInstance(np.eye(2), np.ones(2))
    with pytest.raises(ValueError):
        alm.palm_solve(P, model.SolverConfig(options={"mu0": 0.0}))
    with pytest.raises(ValueError):
        alm.palm_solve(P, model.SolverConfig(options={"rho": 1.0}))


def test_palm_budget_returns_best_iterate(alm, model):
    rng = np.random.default_rng(5)
    A = rng.standard_normal((10, 30))
    b = A @ np.where(rng.random(30) < 0.1, 1.0, 0.0)
    r = alm.palm_solve(model.ProblemInstance(A, b), model.SolverConfig(max_iter=5))
    ref = oracle.palm(A, b, max_iter=5)
    assert not r.converged and r.iterations == 5 == ref.iterations
    assert r.notes == ("inner-iteration budget exhausted",)
    np.testing.assert_allclose(r.x_star, ref.x, atol=1e-10)


def test_palm_penalty_grows_geometrically(alm, model):
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="genspec", n=60, d=30, k=3, seed=1700, sigma=0.0))
    log = []
    res = alm.palm_solve(model.ProblemInstance(A, b), model.SolverConfig(tol=1e-6, max_iter=3000),
                         observer=lambda st: log.append(st))
    assert len(log) == len(res.trace) - 1
    mus = [st.mu for st in log]
    for a, c in zip(mus, mus[1:]):
        assert c == pytest.approx(2.0 * a)
    ref = oracle.palm(A, b, tol=1e-6, max_iter=3000)
    assert res.iterations == ref.iterations
    np.testing.assert_allclose(res.x_star, ref.x, atol=1e-9)


def test_palm_matches_oracle_random(alm, model):
    rng = np.random.default_rng(7)
    for trial in range(4):
        d, n = int(rng.integers(5, 40)), int(rng.integers(45, 100))
        A = rng.standard_normal((d, n))
        x0 = np.zeros(n)
        x0[rng.choice(n, max(1, d // 5), replace=False)] = 1.0
        b = A @ x0
        ref = oracle.palm(A, b, tol=1e-7, max_iter=3000)
        res = alm.palm_solve(model.ProblemInstance(A, b), model.SolverConfig(tol=1e-7, max_iter=3000))
        assert res.iterations == ref.iterations, trial
        assert rel_err(res.x_star, ref.x) <= 1e-8
