"""PDIPA on the B200 vs the reference (golden fixtures) and the oracle.

Mirrors test_pdipa.py through the drop-in entry points (pdipa_solve,
newton_kkt_step, cab_solve(..., "pdipa"), solve_named("pdipa"))."""

import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, case_inputs, gold_notes, ids_for, make_config, rel_err, support

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pd():
    from paper_1007_3753_b200 import pdipa
    return pdipa


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


@pytest.mark.parametrize("cid", ids_for("pdipa", sizes=("small", "cfg1", "cfg2")))
def test_pdipa_matches_reference(pd, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    res = pd.pdipa_solve(model.ProblemInstance(A, b, ground_truth=gt), make_config(case, A, b))
    # the primal residual column reaches rounding level (~1e-10) at convergence
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6,
                  trace_atol=1e-9 * max(1.0, float(np.abs(gold["trace"][:, 2]).max())))
    assert res.notes == gold_notes(gold)


def test_pdipa_cab_matches_reference(model):
    from paper_1007_3753_b200.robust import cab_solve
    case, A, b, gt, gold = case_inputs("cab_small_pdipa")
    x, e, res = cab_solve(A, b, "pdipa", make_config(case, A, b))
    assert res.iterations == int(gold["iterations"]) and res.converged == bool(gold["converged"])
    assert rel_err(res.x_star, gold["w"]) <= 1e-6
    np.testing.assert_allclose(x, gold["x"], rtol=0, atol=1e-6 * max(np.abs(gold["w"]).max(), 1.0))
    np.testing.assert_allclose(e, gold["e"], rtol=0, atol=1e-6 * max(np.abs(gold["w"]).max(), 1.0))


def test_pdipa_zero_rhs_budget_and_observer(pd, model):
    r = pd.pdipa_solve(model.ProblemInstance(np.eye(3), np.zeros(3)), model.SolverConfig())
    assert r.iterations == 0 and r.converged and len(r.trace) == 1 and np.all(r.x_star == 0)
    rng = np.random.default_rng(4)
    A = rng.standard_normal((20, 40))
    x0 = np.zeros(40)
    x0[[3, 11, 30]] = [1.0, -2.0, 0.5]
    P = model.ProblemInstance(A, A @ x0)
    states = []
    r = pd.pdipa_solve(P, model.SolverConfig(), observer=states.append)
    assert r.converged and len(states) == r.iterations
    assert all(np.all(s.x > 0) and np.all(s.z > 0) for s in states)
    mus = [s.mu for s in states]
    assert all(b < a for a, b in zip(mus, mus[1:]))
    ref = oracle.pdipa(A, A @ x0)
    assert r.iterations == ref.iterations
    assert rel_err(r.x_star, ref.x) <= 1e-8
    short = pd.pdipa_solve(P, model.SolverConfig(max_iter=2))
    assert short.iterations == 2 and not short.converged


@pytest.mark.parametrize("seed", range(3))
def test_newton_kkt_step_matches_oracle(pd, seed):
    rng = np.random.default_rng(200 + seed)
    d, N = 12, 30
    A = rng.standard_normal((d, N))
    b = rng.standard_normal(d)
    x = rng.uniform(0.5, 2.0, N)
    z = rng.uniform(0.5, 2.0, N)
    y = rng.standard_normal(d)
    st = pd.PdipaState(x, y, z, float(x @ z) / N)
    dx, dy, dz = pd.newton_kkt_step(st, A, b, 0.1 * st.mu)
    rx, ry, rz = oracle.pd_newton(x, y, z, A, b, 0.1 * st.mu)
    for got, ref in ((dx, rx), (dy, ry), (dz, rz)):
        np.testing.assert_allclose(got[: ref.shape[0]], ref, rtol=1e-9, atol=1e-11)
    # the Newton equations hold
    np.testing.assert_allclose(A @ dx[:N], b - A @ x, rtol=1e-8, atol=1e-10)


def test_solve_named_pdipa(model):
    from paper_1007_3753_b200.solvers import solve_named
    case, A, b, gt, gold = case_inputs("pdipa_small_1600")
    r = solve_named("pdipa", model.ProblemInstance(A, b), make_config(case, A, b))
    assert r.iterations == int(gold["iterations"])
