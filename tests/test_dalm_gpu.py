"""Dual ALM on the B200 vs the reference (golden fixtures) and the oracle.

Mirrors test_alm.py:95-263 through the drop-in entry points.
"""

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


@pytest.mark.parametrize("cid", ids_for("dalm"))
def test_dalm_matches_reference_fp64(alm, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = alm.dalm_solve(P, make_config(case, A, b))
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    assert res.notes == gold_notes(gold)


@pytest.mark.parametrize("cid", [c for c in ids_for("dalm") if c.startswith("cfg")])
def test_dalm_matches_reference_fp32(alm, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    res = alm.dalm_solve(P, make_config(case, A, b, dtype="float32"))
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])


def test_dalm_zero_data(alm, model):
    r = alm.dalm_solve(model.ProblemInstance(np.eye(3), np.zeros(3)), model.SolverConfig())
    assert r.converged and r.iterations == 0 and np.all(r.x_star == 0)
    assert r.trace[0].residual_norm == 0.0


def test_dalm_rejects_rank_deficient_rows(alm, model):
    # test_alm.py:133-137: more rows than columns, A A^T cannot be positive definite
    from paper_1007_3753_b200.exceptions import IllConditionedError
    with pytest.raises(IllConditionedError):
        alm.dalm_solve(model.ProblemInstance(np.ones((3, 2)), np.ones(3)), model.SolverConfig())


def test_dalm_borderline_gram_matches_reference(alm, model):
    # a rank-1 row Gram whose last Cholesky pivot rounds to +1.8e-15: the
    # reference's numpy factor succeeds and the solve converges in 2 steps
    A = np.array([[1.0, 0.0, 1.0], [2.0, 0.0, 2.0]])
    r = alm.dalm_solve(model.ProblemInstance(A, np.array([1.0, 2.0])), model.SolverConfig())
    assert r.converged and r.iterations == 2


def test_dalm_two_variable_value(alm, model):
    # test_alm.py:143-146: min |x1| + |x2| s.t. x1 + 2 x2 = 2  ->  x = (0, 1)
    r = alm.dalm_solve(model.ProblemInstance(np.array([[1.0, 2.0]]), np.array([2.0])),
                       model.SolverConfig(tol=1e-9, max_iter=20000))
    assert np.allclose(r.x_star, [0.0, 1.0], atol=1e-6)


def test_dalm_step_identities_every_iteration(alm, model):
    # test_alm.py:243-263 through the observer path
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="genspec", n=60, d=30, k=3, seed=1700, sigma=0.0))
    P = model.ProblemInstance(A, b)
    log = []
    res = alm.dalm_solve(P, model.SolverConfig(tol=1e-6, max_iter=300),
                         observer=lambda st, xp: log.append((st, xp)))
    assert len(log) == res.iterations
    for st, xp in log:
        assert np.max(np.abs(st.z)) <= 1.0
        aty = A.T @ st.y
        np.testing.assert_allclose(st.x, xp - st.beta * (st.z - aty), atol=1e-9)
        rhs = A @ st.z - (A @ xp - b) / st.beta
        assert np.linalg.norm(rhs - A @ aty) <= 1e-9 * max(1.0, np.linalg.norm(rhs))
    ref = oracle.dalm(A, b, tol=1e-6, max_iter=300)
    assert res.iterations == ref.iterations
    np.testing.assert_allclose(res.x_star, ref.x, atol=1e-9)


def test_dalm_cab_matches_reference(model):
    from paper_1007_3753_b200.robust import cab_solve
    case, A, b, gt, gold = case_inputs("cab_small_dalm")
    cfg = make_config(case, A, b)
    x, e, res = cab_solve(A, b, "dalm", cfg)
    gw = dict(gold)
    gw["x"] = gold["w"]
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gw, 1e-6)
    assert rel_err(x, gold["x"]) <= 1e-6
    np.testing.assert_allclose(e, gold["e"], atol=1e-6 * np.linalg.norm(gold["w"]))


def test_dalm_matches_oracle_random(alm, model):
    rng = np.random.default_rng(99)
    for trial in range(5):
        d, n = int(rng.integers(4, 40)), int(rng.integers(45, 120))
        A = rng.standard_normal((d, n))
        x0 = np.zeros(n)
        x0[rng.choice(n, max(1, d // 5), replace=False)] = rng.standard_normal(max(1, d // 5))
        b = A @ x0
        ref = oracle.dalm(A, b, tol=1e-7, max_iter=4000, opts={"beta": 0.5})
        res = alm.dalm_solve(model.ProblemInstance(A, b),
                             model.SolverConfig(tol=1e-7, max_iter=4000, options={"beta": 0.5}))
        assert abs(res.iterations - ref.iterations) <= 1, (trial, res.iterations, ref.iterations)
        assert rel_err(res.x_star, ref.x) <= 1e-6
