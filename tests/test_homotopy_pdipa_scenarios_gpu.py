"""Homotopy and PDIPA scenarios of the reference's test_homotopy.py and
test_pdipa.py not pinned by golden fixtures: direction / breakpoint helpers
(frozen cases, exhaustive enumeration, singular Gram), exact recovery,
budgets, support recovery rate, the Newton step against the assembled
three-block KKT system, LP vertices, trace contracts and the interior-point
termination certificates."""

import math

import numpy as np
import pytest

import oracle
from tests.golden.cases import build_inputs

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from paper_1007_3753_b200.model import SolverConfig
    return SolverConfig(**kw)


def _P(A, b, gt=None):
    from paper_1007_3753_b200.model import ProblemInstance
    return ProblemInstance(A, b, ground_truth=gt)


def _state(A, support, x, lam, c):
    from paper_1007_3753_b200.homotopy import PathState
    from paper_1007_3753_b200.numerics import chol_factor
    G = A[:, support].T @ A[:, support]
    return PathState(x, list(support), lam, c, chol_factor(G))


def _random_state(seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((10, 20))
    A /= np.linalg.norm(A, axis=0)
    support = [3, 7, 12, 18]
    x = np.zeros(20)
    x[support] = rng.standard_normal(4)
    lam = 0.7
    c = rng.uniform(-0.6, 0.6, size=20)
    c[support] = lam * np.sign(x[support])
    return _state(A, support, x, lam, c), A


def test_direction_cases():
    from paper_1007_3753_b200.exceptions import DegenerateSupportError
    from paper_1007_3753_b200.homotopy import PathState, update_direction
    from paper_1007_3753_b200.numerics import chol_factor
    A = np.eye(3)
    d = update_direction(_state(A, [1], np.zeros(3), 0.9, np.array([0.2, 0.9, -0.1])), A)
    assert d[1] == 1.0 and d[0] == 0.0 and d[2] == 0.0
    A = np.array([[1.0, 0.5], [0.0, np.sqrt(0.75)]])
    d = update_direction(_state(A, [0, 1], np.zeros(2), 1.0, np.array([1.0, 1.0])), A)
    assert np.allclose(d, [2.0 / 3.0, 2.0 / 3.0], rtol=0, atol=1e-12)
    st, A = _random_state(1234)
    d = update_direction(st, A)
    assert np.all(d[np.setdiff1d(np.arange(20), st.support)] == 0.0)
    # a stale factor over a duplicated column: refactorization finds it singular
    A = np.array([[1.0, 1.0], [0.0, 0.0]])
    st = PathState(np.zeros(2), [0, 1], 1.0, np.array([1.0, 1.0]), chol_factor(np.eye(2)))
    with pytest.raises(DegenerateSupportError):
        update_direction(st, A)


def test_direction_repairs_a_drifted_factor():
    from paper_1007_3753_b200.homotopy import PathState, update_direction
    from paper_1007_3753_b200.numerics import chol_factor
    st, A = _random_state(77)
    stale = PathState(st.x, st.support, st.lam, st.c, chol_factor(np.eye(len(st.support))))
    np.testing.assert_allclose(update_direction(stale, A), update_direction(st, A), rtol=1e-10, atol=1e-12)


def test_gammas_cases():
    from paper_1007_3753_b200.homotopy import breakpoint_gammas, update_direction
    A = np.eye(2)
    gp, ip, gm, im = breakpoint_gammas(_state(A, [0], np.array([2.0, 0.0]), 1.0, np.array([1.0, 0.3])),
                                       np.array([-0.5, 0.0]), A)
    assert gm == 4.0 and im == 0
    assert gp == pytest.approx(0.7, abs=1e-15) and ip == 1
    gp, ip, _, _ = breakpoint_gammas(_state(A, [0, 1], np.array([2.0, 1.0]), 1.0, np.array([1.0, 1.0])),
                                     np.array([1.0, 1.0]), A)
    assert gp == np.inf and ip == -1
    st, A = _random_state(1234)
    gp, ip, gm, im = breakpoint_gammas(st, update_direction(st, A), A)
    assert gp == pytest.approx(0.062196515846916718, rel=1e-12) and ip == 14
    assert gm == np.inf and im == -1
    st, A = _random_state(1235)
    gp, ip, gm, im = breakpoint_gammas(st, update_direction(st, A), A)
    assert gp == pytest.approx(0.10713572596767527, rel=1e-12) and ip == 1
    assert gm == pytest.approx(0.19888143972140085, rel=1e-12) and im == 12


def _enumerate_gammas(lam, c, x, d, w, support):
    floor = 1e-10 * lam
    gp, ip = math.inf, -1
    for i in range(c.shape[0]):
        if i in support:
            continue
        for num, den in ((lam - c[i], 1.0 - w[i]), (lam + c[i], 1.0 + w[i])):
            if den != 0.0:
                r = num / den
                if math.isfinite(r) and floor < r < gp:
                    gp, ip = r, i
    gm, im = math.inf, -1
    for i in support:
        if d[i] != 0.0:
            r = -x[i] / d[i]
            if math.isfinite(r) and 0.0 < r < gm:
                gm, im = r, i
    return gp, ip, gm, im


def test_gammas_match_exhaustive_enumeration():
    from paper_1007_3753_b200.homotopy import breakpoint_gammas, update_direction
    for seed in range(3000, 3030):
        st, A = _random_state(seed)
        d = update_direction(st, A)
        w = A.T @ (A[:, st.support] @ d[st.support])
        want = _enumerate_gammas(st.lam, st.c, st.x, d, w, set(st.support))
        got = breakpoint_gammas(st, d, A)
        assert got[1] == want[1] and got[3] == want[3]
        assert got[0] == pytest.approx(want[0], rel=1e-12)
        assert got[2] == pytest.approx(want[2], rel=1e-12)


def test_homotopy_recovery_and_budget():
    from paper_1007_3753_b200.homotopy import homotopy_solve
    rng = np.random.default_rng(7)
    A = rng.standard_normal((100, 200))
    A /= np.linalg.norm(A, axis=0)
    x0 = np.zeros(200)
    sup = rng.choice(200, 5, replace=False)
    x0[sup] = rng.standard_normal(5)
    r = homotopy_solve(_P(A, A @ x0), 0.0, _cfg())
    assert r.converged and r.iterations <= 8
    assert np.linalg.norm(r.x_star - x0) <= 1e-8 * np.linalg.norm(x0)
    assert set(np.flatnonzero(np.abs(r.x_star) > 1e-10 * np.max(np.abs(r.x_star)))) == set(sup)
    r = homotopy_solve(_P(np.eye(2), np.array([3.0, 1.0])), 0.0, _cfg(max_iter=1))
    assert not r.converged and r.iterations == 1
    assert np.allclose(r.x_star, [2.0, 0.0], atol=1e-12)


def test_homotopy_support_recovery_rate():
    from paper_1007_3753_b200.homotopy import homotopy_solve
    n, hits, trials = 256, 0, 100
    for trial in range(trials):
        rng = np.random.default_rng(oracle.trial_seed(91, trial))
        k = int(rng.integers(1, 11))
        d = int(np.ceil(4 * k * np.log(n)))
        A, b, x0 = build_inputs(dict(kind="genspec", n=n, d=d, k=k, seed=oracle.trial_seed(92, trial), sigma=0.0))
        r = homotopy_solve(_P(A, b), 0.0, _cfg(max_iter=400))
        hits += r.converged and set(np.flatnonzero(np.abs(r.x_star) > 1e-8)) == set(np.flatnonzero(x0))
    assert hits >= 0.95 * trials


def _dense_kkt(A_ext, b, st, mu_hat):
    m, d = st.x.shape[0], A_ext.shape[0]
    K = np.zeros((2 * m + d, 2 * m + d))
    K[:d, :m] = A_ext
    K[d:d + m, m:m + d] = A_ext.T
    K[d:d + m, m + d:] = np.eye(m)
    K[d + m:, :m] = np.diag(st.z)
    K[d + m:, m + d:] = np.diag(st.x)
    rhs = np.concatenate([b - A_ext @ st.x, np.ones(m) - A_ext.T @ st.y - st.z, mu_hat - st.x * st.z])
    sol = np.linalg.solve(K, rhs)
    return sol[:m], sol[m:m + d], sol[m + d:]


def test_newton_step_cases():
    from paper_1007_3753_b200.exceptions import IllConditionedError
    from paper_1007_3753_b200.pdipa import PdipaState, newton_kkt_step
    A_ext = np.array([[1.0, -1.0]])
    st = PdipaState(np.array([1.5, 0.5]), np.array([0.5]), np.array([0.5, 1.5]), 0.75)
    dx, dy, dz = newton_kkt_step(st, A_ext, np.array([1.0]), 0.75)
    assert max(np.max(np.abs(dx)), np.max(np.abs(dy)), np.max(np.abs(dz))) <= 1e-14
    st = PdipaState(np.array([1.0, 2.0]), np.array([0.3]), np.array([0.7, 1.2]), 0.0)
    dx, dy, dz = newton_kkt_step(st, A_ext, np.array([1.0]), 0.05)
    assert dx == pytest.approx([-0.55769230769230793, -2.5576923076923075], rel=1e-10)
    assert dy == pytest.approx([0.25961538461538436], rel=1e-10)
    assert dz == pytest.approx([-0.25961538461538436, 0.35961538461538445], rel=1e-10)
    rng = np.random.default_rng(42)
    for _ in range(20):
        A_ext = rng.standard_normal((4, 12))
        b = rng.standard_normal(4)
        st = PdipaState(rng.uniform(0.1, 3.0, 12), rng.standard_normal(4), rng.uniform(0.1, 3.0, 12), 0.0)
        mu_hat = float(rng.uniform(0.01, 0.5))
        for g, w in zip(newton_kkt_step(st, A_ext, b, mu_hat), _dense_kkt(A_ext, b, st, mu_hat)):
            assert np.allclose(g, w, rtol=1e-8, atol=1e-10)
    rng = np.random.default_rng(5)
    A_ext = rng.standard_normal((3, 10))
    b = rng.standard_normal(3)
    st = PdipaState(np.full(10, 2.0), np.zeros(3), np.full(10, 0.5), 0.0)
    dx, _, _ = newton_kkt_step(st, A_ext, b, 0.1)
    rp = b - A_ext @ st.x
    assert np.linalg.norm(A_ext @ dx - rp) <= 1e-10 * max(1.0, np.linalg.norm(rp))
    st = PdipaState(np.array([1.0, 1.0]), np.zeros(1), np.array([1.0, 1.0]), 0.0)
    with pytest.raises(IllConditionedError):
        newton_kkt_step(st, np.array([[0.0, 0.0]]), np.array([1.0]), 0.1)


def test_pdipa_small_problems():
    from paper_1007_3753_b200.homotopy import homotopy_solve
    from paper_1007_3753_b200.pdipa import pdipa_solve
    P = _P(np.array([[1.0, 2.0]]), np.array([2.0]))
    r = pdipa_solve(P, _cfg())
    assert r.converged and np.allclose(r.x_star, [0.0, 1.0], atol=1e-5)
    assert len(r.trace) == r.iterations + 1 and r.trace[-1].residual_norm <= 2e-8
    r = pdipa_solve(P, _cfg(max_iter=2))
    assert not r.converged and r.iterations == 2 and r.x_star.shape == (2,)
    r = pdipa_solve(_P(np.array([[1.0]]), np.array([1.0])), _cfg())
    assert r.converged and r.x_star[0] == pytest.approx(1.0, abs=1e-8)
    rng = np.random.default_rng(11)
    A = rng.standard_normal((50, 100))
    A /= np.linalg.norm(A, axis=0)
    x0 = np.zeros(100)
    x0[rng.choice(100, 5, replace=False)] = rng.standard_normal(5)
    r = pdipa_solve(_P(A, A @ x0), _cfg())
    assert r.converged and np.linalg.norm(r.x_star - x0) <= 1e-6 * np.linalg.norm(x0)
    h = homotopy_solve(_P(A, A @ x0), 0.0, _cfg())
    assert np.linalg.norm(r.x_star - h.x_star) <= 1e-6 * np.linalg.norm(h.x_star)


def test_pdipa_termination_certificates():
    from paper_1007_3753_b200.pdipa import pdipa_solve
    for seed in range(900, 1010):
        A, b, _ = build_inputs(dict(kind="genspec", n=40, d=20, k=1 + seed % 5, seed=seed, sigma=0.0))
        states = []
        r = pdipa_solve(_P(A, b), _cfg(), observer=states.append)
        assert r.converged
        mus = [st.mu for st in states]
        assert all(a > c for a, c in zip(mus, mus[1:]))
        assert all(np.min(st.x) > 0 and np.min(st.z) > 0 for st in states)
        st = states[-1]
        rp = b - A @ (st.x[:40] - st.x[40:])
        assert np.linalg.norm(rp) <= 1e-8 * max(1.0, np.linalg.norm(b))
        obj = float(np.sum(st.x))
        assert obj - float(b @ st.y) <= 1e-6 * (1.0 + abs(obj))
