"""IST on the B200 vs the reference (golden fixtures) and the oracle
(test_shrinkage.py:160-235 through the drop-in)."""

import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, case_inputs, ids_for, make_config, rel_err, support

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shr():
    from paper_1007_3753_b200 import shrinkage
    return shrinkage


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


def _schedule(shr, case, cfg):
    if case["extra"].get("schedule") == "flat":
        return shr.ContinuationSchedule(cfg.lam, 0.5, cfg.lam)
    return None


@pytest.mark.parametrize("cid", ids_for("ist"))
def test_ist_matches_reference_fp64(shr, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    cfg = make_config(case, A, b)
    res = shr.ist_solve(P, _schedule(shr, case, cfg), cfg)
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)


@pytest.mark.parametrize("cid", [c for c in ids_for("ist") if c.startswith("cfg")])
def test_ist_matches_reference_fp32(shr, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    cfg = make_config(case, A, b, dtype="float32")
    res = shr.ist_solve(P, _schedule(shr, case, cfg), cfg)
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])


def test_ist_zero_rhs(shr, model):
    r = shr.ist_solve(model.ProblemInstance(np.eye(4), np.zeros(4)), None, model.SolverConfig(lam=0.1))
    assert r.converged and r.iterations == 0 and np.all(r.x_star == 0.0)


def test_ist_orthonormal_closed_form(shr, model):
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    b = rng.standard_normal(8)
    r = shr.ist_solve(model.ProblemInstance(Q, b), shr.ContinuationSchedule(0.3, 0.5, 0.3),
                      model.SolverConfig(lam=0.3, tol=1e-8))
    assert r.converged
    assert np.max(np.abs(r.x_star - oracle.soft(Q.T @ b, 0.3))) <= 1e-6


def test_ist_budget_cap(shr, model):
    rng = np.random.default_rng(19)
    A = rng.standard_normal((20, 40))
    A /= np.linalg.norm(A, axis=0)
    b = rng.standard_normal(20)
    r = shr.ist_solve(model.ProblemInstance(A, b), None, model.SolverConfig(lam=0.05, max_iter=3))
    ref = oracle.ist(A, b, lam=0.05, max_iter=3)
    assert not r.converged and r.iterations == 3 == ref.iterations
    np.testing.assert_allclose(r.x_star, ref.x, atol=1e-12)


def test_ist_strict_descent_with_observer(shr, model):
    # test_shrinkage.py:215-235
    from tests.golden.cases import build_inputs
    for seed in (1200, 1201, 1203):
        A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=1 + seed % 5, seed=seed, sigma=0.02))
        P = model.ProblemInstance(A, b)
        lam = 0.05 * float(np.max(np.abs(A.T @ b)))
        xs = []
        res = shr.ist_solve(P, shr.ContinuationSchedule(lam, 0.5, lam),
                            model.SolverConfig(lam=lam, tol=1e-8, max_iter=3000),
                            observer=lambda x, la, dF: xs.append((x, dF)))
        assert len(xs) == res.iterations
        prev = np.zeros(P.n)
        for cur, dF in xs:
            assert dF < 0.0
            Ap, Ac = A @ prev, A @ cur
            assert oracle.obj_delta(prev, cur, Ap, Ac, A.T @ (Ap - b), lam) < 0.0
            prev = cur
        ref = oracle.ist(A, b, stages=[lam], lam=lam, tol=1e-8, max_iter=3000)
        assert res.iterations == ref.iterations


def test_ist_matches_oracle_random(shr, model):
    rng = np.random.default_rng(31)
    for trial in range(5):
        d, n = int(rng.integers(5, 50)), int(rng.integers(10, 120))
        A = rng.standard_normal((d, n))
        b = rng.standard_normal(d)
        lam = float(rng.uniform(0.01, 0.2)) * float(np.max(np.abs(A.T @ b)))
        ref = oracle.ist(A, b, lam=lam, tol=1e-8, max_iter=4000)
        res = shr.ist_solve(model.ProblemInstance(A, b), None,
                            model.SolverConfig(lam=lam, tol=1e-8, max_iter=4000))
        # near the optimum dF compares objective differences at machine precision, so a
        # different (deterministic) summation order may take a few more / fewer steps;
        # the north-star gates are the solution and its support
        assert res.converged == ref.converged
        assert rel_err(res.x_star, ref.x) <= 1e-6
        assert support(res.x_star) == support(ref.x)
