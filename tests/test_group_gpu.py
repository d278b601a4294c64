"""Group launches (one dictionary per solve, teams of CTAs walking the
trials) against the oracle and against the single-solve entry points:
every trial must take the iterations the reference takes and land within
the parity tolerance (fp64: 1e-6 relative)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SHAPES = [(20, 40), (30, 60), (25, 80), (40, 80)]


def _trials(count, sigma=0.01, seed0=500):
    from paper_1007_3753_b200.model import ProblemInstance
    out = []
    for t in range(count):
        d, n = SHAPES[t % len(SHAPES)]
        A = oracle.gaussian_dict(d, n, seed0 + t)
        x0 = oracle.sparse_signal(n, 1 + t % 4, seed0 + t)
        b = oracle.with_noise(A @ x0, sigma, seed0 + t)
        out.append(ProblemInstance(A, b, ground_truth=x0))
    return out


def _cfg(**kw):
    from paper_1007_3753_b200.model import SolverConfig
    return SolverConfig(**kw)


def _ref(name, P, lam, tol, max_iter):
    A, b = P.A, P.b
    if name == "fista":
        return oracle.fista(A, b, lam=lam, tol=tol, max_iter=max_iter)
    if name == "ist":
        return oracle.ist(A, b, lam=lam, tol=tol, max_iter=max_iter)
    if name == "gpsr":
        return oracle.gpsr(A, b, lam=lam, tol=tol, max_iter=max_iter)
    if name == "tnipm":
        return oracle.tnipm(A, b, lam=lam, tol=tol, max_iter=max_iter)
    if name == "palm":
        return oracle.palm(A, b, tol=tol, max_iter=max_iter)
    if name == "dalm":
        return oracle.dalm(A, b, tol=tol, max_iter=max_iter)
    return oracle.homotopy(A, b, lam, max_iter=max_iter)[0]


@pytest.mark.parametrize("name", ["fista", "ist", "gpsr", "tnipm", "palm", "dalm", "homotopy"])
def test_group_matches_oracle(name):
    from paper_1007_3753_b200.group import TrialGroup
    probs = _trials(12, sigma=0.0 if name in ("palm", "dalm") else 0.01)
    grp = TrialGroup(probs)
    c = grp.correlation_max()
    np.testing.assert_allclose(c, [np.max(np.abs(P.A.T @ P.b)) for P in probs], rtol=1e-13)
    lams = 0.05 * c
    tol, max_iter = 1e-6, 3000
    res = grp.solve(name, _cfg(tol=tol, max_iter=max_iter), lams=lams, want_trace=True)
    for P, lam, r in zip(probs, lams, res):
        ref = _ref(name, P, lam, tol, max_iter)
        assert r.iterations == ref.iterations, (name, r.iterations, ref.iterations)
        assert r.converged == ref.converged
        nrm = max(np.linalg.norm(ref.x), 1e-300)
        assert np.linalg.norm(r.x_star - ref.x) <= 1e-6 * nrm
        assert len(r.trace) == len(ref.trace)


def test_group_agrees_with_single_solves():
    from paper_1007_3753_b200.group import TrialGroup
    from paper_1007_3753_b200.shrinkage import fista_solve
    probs = _trials(8)
    res = TrialGroup(probs).solve("fista", _cfg(tol=1e-6, max_iter=3000))
    for P, r in zip(probs, res):
        s = fista_solve(P, _cfg(tol=1e-6, max_iter=3000))
        assert r.iterations == s.iterations
        np.testing.assert_allclose(r.x_star, s.x_star, rtol=0, atol=1e-10 * max(1.0, np.abs(s.x_star).max()))


def test_group_multi_cta_teams_and_norms():
    """Dictionaries too large for one CTA's shared memory run on teams of
    several CTAs (team barrier path)."""
    from paper_1007_3753_b200 import _lib
    from paper_1007_3753_b200.group import TrialGroup
    from paper_1007_3753_b200.model import ProblemInstance
    probs = []
    for t in range(5):
        A = oracle.gaussian_dict(200, 400, 900 + t)
        x0 = oracle.sparse_signal(400, 10, 900 + t)
        probs.append(ProblemInstance(A, A @ x0))
    grp = TrialGroup(probs)
    team = int(_lib.lib().ell1_group_team(_lib.SOLVER_FISTA, grp.dicts[0]))
    assert team > 1
    ns = grp.norm_sq()
    for P, v in zip(probs, ns):
        assert abs(v - oracle.power_norm_sq(P.A)) <= 1e-12 * v
    res = grp.solve("fista", _cfg(tol=1e-6, max_iter=3000))
    for P, r in zip(probs, res):
        ref = oracle.fista(P.A, P.b, tol=1e-6, max_iter=3000)
        assert r.iterations == ref.iterations
        assert np.linalg.norm(r.x_star - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


def test_group_cross_and_bouquet():
    from paper_1007_3753_b200.group import TrialGroup
    from paper_1007_3753_b200.model import ProblemInstance
    probs = []
    for t in range(6):
        A = oracle.gaussian_dict(30, 50, 700 + t)
        x0 = oracle.sparse_signal(50, 2, 700 + t)
        b, _ = oracle.corrupt(A @ x0, 0.1, -1.0, 1.0, 700 + t)
        probs.append(ProblemInstance(A, b))
    grp = TrialGroup(probs, ext=True)
    res = grp.solve("homotopy", _cfg(tol=1e-6, max_iter=2000), lams=np.zeros(6))
    for P, r in zip(probs, res):
        _, _, ref = oracle.cab(P.A, P.b, "homotopy", lam=0.0, tol=1e-6, max_iter=2000)
        assert r.iterations == ref.iterations
        np.testing.assert_allclose(r.x_star, ref.x, atol=1e-6 * max(1.0, np.abs(ref.x).max()))


def test_group_errors():
    from paper_1007_3753_b200.group import TrialGroup
    probs = _trials(2)
    with pytest.raises(ValueError):
        TrialGroup(probs).solve("pdipa", _cfg())
    with pytest.raises(ValueError):
        TrialGroup(probs).solve("gpsr", _cfg(), lams=np.array([0.1, 0.0]))
