"""Batched shared-dictionary solvers: element j must equal the single-instance
reference solve on (A, b_j) (SURVEY §8(b) batched entry points)."""

import numpy as np
import pytest

import oracle
from tests.gpu_util import rel_err, support

pytestmark = pytest.mark.gpu


def _batch(d, n, ks, seed=5, noise=0.0):
    A = oracle.gaussian_dict(d, n, seed)
    cols, gts = [], []
    for j, k in enumerate(ks):
        g = np.random.default_rng(1000 + j)
        x0 = np.zeros(n)
        x0[g.choice(n, k, replace=False)] = g.standard_normal(k)
        b = A @ x0
        if noise:
            b = b + noise * g.standard_normal(d)
        cols.append(b)
        gts.append(x0)
    return A, np.stack(cols, axis=1), gts


@pytest.fixture(scope="module")
def bt():
    from paper_1007_3753_b200 import batched
    return batched


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batch_fista_equals_single_instances(bt, dtype):
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    A, Bm, _ = _batch(512, 2048, [16, 32, 64, 8, 48, 24, 1, 40])
    cfg = SolverConfig(lam=1e-3, tol=1e-6, stopping=StoppingRule("relative-estimate", 1e-6),
                       options={"dtype": dtype})
    res = bt.fista_solve_batch(A, Bm, cfg, with_trace=True).results()
    for j in range(Bm.shape[1]):
        ref = oracle.fista(A, Bm[:, j], lam=1e-3, tol=1e-6, stop=("relative-estimate", 1e-6))
        tol = 1e-6 if dtype == "float64" else 1e-4
        assert rel_err(res[j].x_star, ref.x) <= tol, j
        assert support(res[j].x_star) == support(ref.x), j
        assert res[j].converged == ref.converged
        if dtype == "float64":
            assert res[j].iterations == ref.iterations, (j, res[j].iterations, ref.iterations)
            tr = np.array([tuple(t) for t in res[j].trace])
            np.testing.assert_allclose(tr, np.array(ref.trace), rtol=1e-9, atol=1e-12)


def test_batch_fista_default_lambda_and_budget(bt):
    from paper_1007_3753_b200.model import SolverConfig
    A, Bm, _ = _batch(64, 200, [3, 5, 9, 2], noise=0.01)
    Bm = np.concatenate([Bm, np.zeros((64, 1))], axis=1)     # one zero-data instance
    for cap in (3, 5000):
        cfg = SolverConfig(tol=1e-7, max_iter=cap)
        res = bt.fista_solve_batch(A, Bm, cfg, with_trace=True).results()
        for j in range(Bm.shape[1]):
            ref = oracle.fista(A, Bm[:, j], lam=None, tol=1e-7, max_iter=cap)
            assert res[j].iterations == ref.iterations and res[j].converged == ref.converged
            assert rel_err(res[j].x_star, ref.x) <= 1e-9 if np.any(ref.x) else np.all(res[j].x_star == 0)


def test_batch_fista_cab(bt):
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import ExtendedDictionary
    A = oracle.gaussian_dict(40, 30, 7)
    g = np.random.default_rng(3)
    Bm = A @ (g.standard_normal((30, 5)) * (g.random((30, 5)) < 0.1)) + 0.3 * (g.random((40, 5)) < 0.1)
    cfg = SolverConfig(tol=1e-6, max_iter=5000)
    res = bt.fista_solve_batch(ExtendedDictionary(A, 1.0), Bm, cfg).results()
    for j in range(5):
        x, e, ref = oracle.cab(A, Bm[:, j], "fista", tol=1e-6, max_iter=5000)
        assert res[j].iterations == ref.iterations
        assert rel_err(res[j].x_star, ref.x) <= 1e-8


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batch_dalm_equals_single_instances(bt, dtype):
    from paper_1007_3753_b200.model import SolverConfig, StoppingRule
    A, Bm, _ = _batch(128, 512, [4, 8, 16, 2, 12, 6])
    cfg = SolverConfig(tol=1e-6, max_iter=3000, stopping=StoppingRule("relative-estimate", 1e-6),
                       options={"dtype": dtype})
    res = bt.dalm_solve_batch(A, Bm, cfg, with_trace=True).results()
    for j in range(Bm.shape[1]):
        ref = oracle.dalm(A, Bm[:, j], tol=1e-6, max_iter=3000, stop=("relative-estimate", 1e-6))
        tol = 1e-6 if dtype == "float64" else 1e-4
        assert rel_err(res[j].x_star, ref.x) <= tol, j
        assert support(res[j].x_star) == support(ref.x), j
        if dtype == "float64":
            assert res[j].iterations == ref.iterations, (j, res[j].iterations, ref.iterations)
            tr = np.array([tuple(t) for t in res[j].trace])
            np.testing.assert_allclose(tr, np.array(ref.trace), rtol=1e-8, atol=1e-10)


def test_batch_dalm_cab_matches_reference(bt):
    from paper_1007_3753_b200.model import SolverConfig
    from paper_1007_3753_b200.robust import ExtendedDictionary
    from tests.golden.cases import build_inputs
    A, b, _ = build_inputs(dict(kind="cab", d=40, n=30, k=3, seed=7, m=4))
    g = np.random.default_rng(11)
    Bm = np.stack([b] + [A @ (g.standard_normal(30) * (g.random(30) < 0.1)) + 0.5 * (g.random(40) < 0.1)
                         for _ in range(4)], axis=1)
    cfg = SolverConfig(tol=1e-6, max_iter=5000)
    res = bt.dalm_solve_batch(ExtendedDictionary(A, 1.0), Bm, cfg, with_trace=True).results()
    for j in range(Bm.shape[1]):
        x, e, ref = oracle.cab(A, Bm[:, j], "dalm", tol=1e-6, max_iter=5000)
        assert res[j].iterations == ref.iterations, j
        assert rel_err(res[j].x_star, ref.x) <= 1e-8
        assert res[j].notes == ref.notes


def _src_host(A, lab, b, w, s):
    n = A.shape[1]
    x, e = w[:n], s * w[n:]
    out = []
    for c in range(int(lab.max()) + 1):
        m = lab == c
        out.append(np.linalg.norm(b - e - A[:, m] @ x[m]))
    return int(np.argmin(out)), np.array(out)


def test_src_labels_match_reference_rule(bt):
    # a scaled-down config 3: 6 classes x 8 columns, d=96, 20% corrupted queries
    from paper_1007_3753_b200 import synth
    from paper_1007_3753_b200.model import SolverConfig
    A, lab = synth.cab_dictionary(d=96, classes=6, per_class=8, subspace=3, seed=2)
    Bq, truth = synth.cab_queries(A, lab, 10, fraction=0.2, seed=3)
    cfg = SolverConfig(tol=1e-4, max_iter=4000, options={"beta": 0.1})
    labels, resid, res = bt.src_classify(A, lab, Bq.T, cfg)
    for j in range(Bq.shape[0]):
        x, e, ref = oracle.cab(A, Bq[j], "dalm", tol=1e-4, max_iter=4000, opts={"beta": 0.1})
        want, wres = _src_host(A, lab, Bq[j], np.concatenate([x, e]), 1.0)
        assert labels[j] == want, j
        np.testing.assert_allclose(resid[j], wres, rtol=1e-5, atol=1e-8)
    assert np.mean(labels == truth) >= 0.8
