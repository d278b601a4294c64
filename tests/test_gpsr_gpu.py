"""GPSR on the B200 vs the reference (golden fixtures) and the oracle
(test_gradient_projection.py:128-183, 283-320 through the drop-in)."""

import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, case_inputs, gold_notes, ids_for, make_config, rel_err, support

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gp():
    from paper_1007_3753_b200 import gradient_projection
    return gradient_projection


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


@pytest.mark.parametrize("cid", ids_for("gpsr"))
def test_gpsr_matches_reference_fp64(gp, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    cfg = make_config(case, A, b)
    res = gp.gpsr_solve(P, cfg.lam, cfg)
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    assert res.notes == gold_notes(gold)


@pytest.mark.parametrize("cid", [c for c in ids_for("gpsr") if c.startswith("cfg")])
def test_gpsr_matches_reference_fp32(gp, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    P = model.ProblemInstance(A, b, ground_truth=gt)
    cfg = make_config(case, A, b, dtype="float32")
    res = gp.gpsr_solve(P, cfg.lam, cfg)
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])


def test_gpsr_zero_data(gp, model):
    r = gp.gpsr_solve(model.ProblemInstance(np.eye(3), np.zeros(3)), 0.1, model.SolverConfig())
    assert r.converged and r.iterations == 0


def test_gpsr_rejects_nonpositive_lambda(gp, model):
    with pytest.raises(ValueError):
        gp.gpsr_solve(model.ProblemInstance(np.eye(2), np.ones(2)), 0.0, model.SolverConfig())


def test_gpsr_orthonormal_closed_form(gp, model):
    rng = np.random.default_rng(8)
    Q, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    b = rng.standard_normal(10)
    r = gp.gpsr_solve(model.ProblemInstance(Q, b), 0.2, model.SolverConfig(tol=1e-10, max_iter=20000))
    assert r.converged
    assert np.max(np.abs(r.x_star - oracle.soft(Q.T @ b, 0.2))) <= 1e-6


def test_gpsr_iterates_feasible_and_descending(gp, model):
    # test_gradient_projection.py:283-306 via the observer
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=3, seed=1300, sigma=0.02))
    P = model.ProblemInstance(A, b)
    lam = 0.05 * float(np.max(np.abs(A.T @ b)))
    zs = []
    res = gp.gpsr_solve(P, lam, model.SolverConfig(tol=1e-7, max_iter=3000),
                        observer=lambda it: zs.append(it.z))
    assert len(zs) == res.iterations
    prevF = np.inf
    for z in zs:
        assert np.all(z >= 0)
        x = z[:P.n] - z[P.n:]
        F = model.objective(x, P, lam)
        assert F <= prevF + 1e-12
        prevF = F


def test_gpsr_matches_oracle_random(gp, model):
    rng = np.random.default_rng(41)
    for trial in range(5):
        d, n = int(rng.integers(5, 50)), int(rng.integers(10, 120))
        A = rng.standard_normal((d, n))
        b = rng.standard_normal(d)
        lam = float(rng.uniform(0.02, 0.3)) * float(np.max(np.abs(A.T @ b)))
        ref = oracle.gpsr(A, b, lam=lam, tol=1e-7, max_iter=3000)
        res = gp.gpsr_solve(model.ProblemInstance(A, b), lam, model.SolverConfig(tol=1e-7, max_iter=3000))
        assert abs(res.iterations - ref.iterations) <= max(3, ref.iterations // 20), trial
        assert rel_err(res.x_star, ref.x) <= 1e-6
        assert support(res.x_star) == support(ref.x)


def test_gpsr_cab_backend(model):
    from paper_1007_3753_b200.robust import cab_solve
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="cab", d=40, n=30, k=3, seed=7, m=4))
    x, e, res = cab_solve(A, b, "gp", model.SolverConfig(tol=1e-6, max_iter=5000))
    ref_x, ref_e, ref = oracle.cab(A, b, "gp", tol=1e-6, max_iter=5000)
    assert rel_err(np.concatenate([x, e]), np.concatenate([ref_x, ref_e])) <= 1e-6
