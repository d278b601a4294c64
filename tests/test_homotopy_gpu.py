"""Homotopy on the B200 vs the reference (golden fixtures) and the oracle
(test_homotopy.py:141-291 through the drop-in)."""

import numpy as np
import pytest

import oracle
from tests.golden.cases import resolve_lambda
from tests.gpu_util import assert_parity, case_inputs, gold_notes, ids_for, rel_err, support

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hom():
    from paper_1007_3753_b200 import homotopy
    return homotopy


@pytest.fixture(scope="module")
def model():
    from paper_1007_3753_b200 import model
    return model


def _target(case, A, b):
    lam = resolve_lambda(case["cfg"], A, b)
    return lam if lam is not None else 1e-2 * float(np.max(np.abs(A.T @ b)))


@pytest.mark.parametrize("cid", ids_for("homotopy"))
def test_homotopy_matches_reference_fp64(hom, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    res = hom.homotopy_solve(model.ProblemInstance(A, b), _target(case, A, b), model.SolverConfig())
    assert_parity(res.x_star, res.iterations, res.converged, res.trace, gold, 1e-6)
    assert res.notes == gold_notes(gold)


@pytest.mark.parametrize("cid", [c for c in ids_for("homotopy") if c.startswith("cfg")])
def test_homotopy_matches_reference_fp32(hom, model, cid):
    case, A, b, gt, gold = case_inputs(cid)
    res = hom.homotopy_solve(model.ProblemInstance(A, b), _target(case, A, b),
                             model.SolverConfig(options={"dtype": "float32"}))
    assert rel_err(res.x_star, gold["x"]) <= 1e-4
    assert support(res.x_star) == support(gold["x"])


def test_identity_reaches_soft_threshold(hom, model):
    # test_homotopy.py:141-146
    r = hom.homotopy_solve(model.ProblemInstance(np.eye(2), np.array([3.0, 1.0])), 1.0,
                           model.SolverConfig())
    assert r.converged
    np.testing.assert_allclose(r.x_star, [2.0, 0.0], atol=1e-12)
    assert len(r.trace) == r.iterations


def test_zero_rhs_and_target_above_start(hom, model):
    r = hom.homotopy_solve(model.ProblemInstance(np.eye(3), np.zeros(3)), 0.1, model.SolverConfig())
    assert r.converged and r.iterations == 0
    res, lam = hom.solve_path(np.eye(2), np.array([0.5, 0.2]), 2.0, model.SolverConfig())
    assert res.iterations == 0 and lam == 2.0


def test_negative_target_rejected(hom, model):
    with pytest.raises(ValueError):
        hom.homotopy_solve(model.ProblemInstance(np.eye(2), np.ones(2)), -1.0, model.SolverConfig())


def test_path_invariants_with_observer(hom, model):
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=3, seed=1300, sigma=0.02))
    target = 0.01 * float(np.max(np.abs(A.T @ b)))
    states = []
    res, lam = hom.solve_path(A, b, target, model.SolverConfig(), observer=lambda s: states.append(s))
    assert len(states) == res.iterations
    lams = [s.lam for s in states]
    assert all(x > y for x, y in zip(lams, lams[1:]))
    for s in states[:-1]:
        c = A.T @ (b - A @ s.x)
        np.testing.assert_allclose(c, s.c, atol=1e-9)
        G = A[:, s.support].T @ A[:, s.support]
        np.testing.assert_allclose(s.chol.R.T @ s.chol.R, G, atol=1e-8)
    ref, ref_lam = oracle.homotopy(A, b, target)
    assert res.iterations == ref.iterations and lam == pytest.approx(ref_lam)


def test_path_csv(hom, model, tmp_path):
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=3, seed=1301, sigma=0.02))
    target = 0.01 * float(np.max(np.abs(A.T @ b)))
    out = tmp_path / "path.csv"
    res = hom.homotopy_solve(model.ProblemInstance(A, b), target, model.SolverConfig(), path_csv=str(out))
    lines = out.read_text().splitlines()
    assert lines[0] == "lambda,support_size,objective"
    assert len(lines) == 1 + len(res.trace)


def test_matches_oracle_random(hom, model):
    rng = np.random.default_rng(51)
    for trial in range(5):
        d, n = int(rng.integers(10, 60)), int(rng.integers(20, 150))
        A = rng.standard_normal((d, n))
        A /= np.linalg.norm(A, axis=0)
        x0 = np.zeros(n)
        x0[rng.choice(n, max(1, d // 6), replace=False)] = rng.standard_normal(max(1, d // 6))
        b = A @ x0 + 0.01 * rng.standard_normal(d)
        target = 0.01 * float(np.max(np.abs(A.T @ b)))
        ref, _ = oracle.homotopy(A, b, target)
        res = hom.homotopy_solve(model.ProblemInstance(A, b), target, model.SolverConfig())
        assert res.iterations == ref.iterations, trial
        assert rel_err(res.x_star, ref.x) <= 1e-8


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_maintained_inverse_needs_no_refactorisation(seed):
    """homotopy.cu keeps W = R^{-1} next to R (appends extend it, deletes rotate
    it with R's Givens sequence).  If W drifted from R^{-1}, the drift check
    would trigger dense refactorisations (counted in state.rot[7]); a clean
    path — including remove events — must need none (the reference's
    test_no_fresh_factorization_on_clean_path, homotopy.py:53-64)."""
    import torch
    from paper_1007_3753_b200 import _lib, device as dv
    from paper_1007_3753_b200._runner import Buffers, Prepared, byref
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    rng = np.random.default_rng(40 + seed)
    d, n = 120, 400
    A = rng.standard_normal((d, n))
    A /= np.linalg.norm(A, axis=0)
    b = A @ oracle.sparse_signal(n, 30, 40 + seed) + 0.02 * rng.standard_normal(d)
    cfg = SolverConfig(lam=None, tol=1.0, max_iter=2000)
    prep = Prepared(ProblemInstance(A, b), cfg)
    L = _lib.lib()
    bufs = Buffers(prep, L.ell1_homotopy_workspace(byref(prep.view), 0), cfg.max_iter + 2)
    out = _lib.HomOut()
    cb = torch.zeros(prep.n, dtype=torch.float64, device=prep.dev)
    out.c = cb.data_ptr()
    lam = 1e-3 * float(np.max(np.abs(A.T @ b)))
    _lib.check(L.ell1_homotopy(byref(prep.view), dv.ptr(prep.b), lam, cfg.max_iter, byref(out),
                               byref(bufs.io(0)), prep.stream), "homotopy")
    st = bufs.read_all()
    ref, _ = oracle.homotopy(A, b, lam, max_iter=2000)
    removes = sum(1 for a0, a1 in zip(ref.trace, ref.trace[1:]) if a1[3] < a0[3])
    assert st.iterations == ref.iterations and removes > 0
    assert st.rot[7] == 0
    np.testing.assert_allclose(bufs.x_host(), ref.x, atol=1e-8 * max(1.0, np.abs(ref.x).max()))
