"""Device numerics / operator utilities
against the oracle restatement and the reference's own known answers
(test_numerics.py, test_accel.py cases restated)."""

import numpy as np
import pytest

import oracle.l1_oracle as O

pytestmark = pytest.mark.gpu


def spd(rng, n):
    B = rng.standard_normal((n, n))
    return B @ B.T + n * np.eye(n)


# ------------------------------------------------------------ _accel seam
@pytest.mark.parametrize("seed", range(4))
def test_accel_elementwise_bitwise(seed):
    from paper_1007_3753_b200 import _accel
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(1000) * 3
    u[::7] = 0.5                          # exactly at the threshold
    a = 0.5
    np.testing.assert_array_equal(_accel.soft_threshold(u, a), O.soft(u, a))
    np.testing.assert_array_equal(_accel.project_box_linf(u), np.clip(u, -1.0, 1.0))


@pytest.mark.parametrize("seed", range(3))
def test_accel_rank1_matches_oracle(seed):
    from paper_1007_3753_b200 import _accel
    rng = np.random.default_rng(100 + seed)
    m = 12
    R = np.ascontiguousarray(np.linalg.cholesky(spd(rng, m)).T)
    v = rng.standard_normal(m)
    R1, v1 = R.copy(), v.copy()
    R2, v2 = R.copy(), v.copy()
    assert _accel.chol_update(R1, v1) == 0
    O.rank1_update(R2, v2)
    np.testing.assert_allclose(R1, R2, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(v1, v2, rtol=1e-12, atol=1e-12)
    # downdate back
    w = v.copy()
    R3 = R1.copy()
    assert _accel.chol_downdate(R3, w) == 0
    np.testing.assert_allclose(R3.T @ R3, R.T @ R, rtol=1e-10, atol=1e-10)


def test_accel_downdate_failure_status():
    from paper_1007_3753_b200 import _accel
    R = np.eye(3)
    v = np.array([0.0, 2.0, 0.0])
    R1, v1 = R.copy(), v.copy()
    R2, v2 = R.copy(), v.copy()
    assert _accel.chol_downdate(R1, v1) == O.rank1_downdate(R2, v2) == 2


# ------------------------------------------------------------ numerics
def test_soft_threshold_contract():
    from paper_1007_3753_b200 import numerics
    np.testing.assert_array_equal(numerics.soft_threshold(np.array([3.0, -3.0, 0.5, -0.5]), 1.0),
                                  [2.0, -2.0, 0.0, 0.0])
    out = numerics.soft_threshold(np.arange(6.0).reshape(2, 3) - 2.5, 1.0)
    assert out.shape == (2, 3)
    with pytest.raises(ValueError):
        numerics.soft_threshold(np.ones(3), -1.0)
    with pytest.raises(ValueError):
        numerics.soft_threshold(np.ones(3), np.ones(2))
    np.testing.assert_array_equal(numerics.project_box_linf(np.array([2.0, -3.0, 0.25])), [1.0, -1.0, 0.25])


def test_chol_factor_and_solve():
    from paper_1007_3753_b200 import numerics
    from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError
    rng = np.random.default_rng(5)
    for n in (1, 8, 40, 100):
        M = spd(rng, n)
        F = numerics.chol_factor(M)
        np.testing.assert_allclose(F.matrix(), M, rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(F.R, np.linalg.cholesky(M).T, rtol=1e-10, atol=1e-12)
        rhs = rng.standard_normal(n)
        np.testing.assert_allclose(F.solve(rhs), np.linalg.solve(M, rhs), rtol=1e-9, atol=1e-11)
    with pytest.raises(NotPositiveDefiniteError):
        numerics.chol_factor(np.diag([1.0, -1.0]))


@pytest.mark.parametrize("d", [1, 5, 31, 32, 33, 64, 70, 257, 1024])
def test_dense_cholesky_abi_ragged_sizes(d):
    """ell1_chol_factor_dense / ell1_chol_solve_dense(_multi) through the C ABI
    (pdipa.py:43-62's factor + solve; chol.cu): blocked 64-column panels and the
    32-column solve blocks with one step of lookahead, at sizes that are not
    multiples of either block, against numpy's factor and solve."""
    import ctypes
    import torch
    from paper_1007_3753_b200 import _lib
    L_ = _lib.lib()
    rng = np.random.default_rng(100 + d)
    M = spd(rng, d)
    dev = torch.device("cuda", 0)
    Md = torch.from_numpy(M).to(dev)                          # symmetric: row- or column-major alike
    Lf = torch.zeros((d, d), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())               # noqa: E731
    assert L_.ell1_chol_factor_dense(d, P(Md), d, 0.0, P(Lf), d, P(info), st) == 0
    assert int(info.item()) == 0
    Lh = np.tril(Lf.cpu().numpy().T)                          # column-major lower factor
    np.testing.assert_allclose(Lh, np.linalg.cholesky(M), rtol=1e-11, atol=1e-12)
    nrhs = 3
    R = rng.standard_normal((nrhs, d))                        # nrhs right-hand sides, pitch d
    Rd = torch.from_numpy(R).to(dev)
    Xd = torch.empty_like(Rd)
    assert L_.ell1_chol_solve_dense_multi(d, P(Lf), d, nrhs, P(Rd), d, P(Xd), d, st) == 0
    X = Xd.cpu().numpy()
    for k in range(nrhs):
        np.testing.assert_allclose(X[k], np.linalg.solve(M, R[k]), rtol=1e-9, atol=1e-12)
    x1 = torch.empty(d, dtype=torch.float64, device=dev)
    assert L_.ell1_chol_solve_dense(d, P(Lf), d, P(Rd), P(x1), st) == 0
    np.testing.assert_array_equal(x1.cpu().numpy(), X[0])
    # not positive definite: LAPACK's status convention (failing column + 1)
    Mb = M.copy()
    k = d // 2
    Mb[k, k] = -1.0
    assert L_.ell1_chol_factor_dense(d, P(torch.from_numpy(Mb).to(dev)), d, 0.0, P(Lf), d, P(info), st) == 0
    assert int(info.item()) == k + 1


def test_chol_rank1_append_delete():
    from paper_1007_3753_b200 import numerics
    from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError
    rng = np.random.default_rng(9)
    B = rng.standard_normal((30, 10))
    M = B.T @ B
    F = numerics.chol_factor(M[:9, :9])
    F2 = numerics.chol_append(F, M[:9, 9], M[9, 9])
    np.testing.assert_allclose(F2.R, O.chol_grow(F.R, M[:9, 9], M[9, 9]), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(F2.matrix(), M, rtol=1e-9, atol=1e-9)
    for k in (0, 4, 9):
        F3 = numerics.chol_delete(F2, k)
        keep = [i for i in range(10) if i != k]
        np.testing.assert_allclose(F3.matrix(), M[np.ix_(keep, keep)], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(F3.R, O.chol_drop(F2.R, k), rtol=1e-12, atol=1e-12)
    v = rng.standard_normal(10)
    Fu = numerics.chol_rank1(F2, v, 1)
    np.testing.assert_allclose(Fu.matrix(), M + np.outer(v, v), rtol=1e-9, atol=1e-9)
    Fd = numerics.chol_rank1(Fu, v, -1)
    np.testing.assert_allclose(Fd.matrix(), M, rtol=1e-8, atol=1e-8)
    with pytest.raises(NotPositiveDefiniteError):
        numerics.chol_rank1(numerics.chol_factor(np.eye(2)), np.array([2.0, 0.0]), -1)
    with pytest.raises(NotPositiveDefiniteError):
        numerics.chol_append(numerics.chol_factor(np.eye(2)), np.array([1.0, 0.0]), 1.0)
    with pytest.raises(ValueError):
        numerics.chol_rank1(F2, v, 2)
    F0 = numerics.chol_append(numerics.CholFactor(np.zeros((0, 0))), np.zeros(0), 4.0)
    np.testing.assert_allclose(F0.R, [[2.0]])


def test_pcg_known_answers():
    from paper_1007_3753_b200 import numerics
    res = numerics.pcg_solve(np.eye(3), np.array([1.0, -2.0, 3.0]), tol=1e-10, max_iter=10)
    assert res.converged and res.iterations == 1
    np.testing.assert_allclose(res.x, [1.0, -2.0, 3.0], atol=1e-12)
    res = numerics.pcg_solve(np.diag([1.0, 2.0]), np.array([1.0, 2.0]), tol=1e-10, max_iter=10)
    np.testing.assert_allclose(res.x, [1.0, 1.0], atol=1e-10)
    res = numerics.pcg_solve(np.diag([1.0, -1.0]), np.array([1.0, 1.0]), tol=1e-10, max_iter=5)
    assert not res.converged
    rng = np.random.default_rng(31)
    dg = rng.uniform(1, 1e4, 30)
    b = rng.standard_normal(30)
    res = numerics.pcg_solve(np.diag(dg), b, precond=dg, tol=1e-12, max_iter=5)
    assert res.converged
    np.testing.assert_allclose(res.x, b / dg, rtol=1e-10)
    res = numerics.pcg_solve(np.eye(4), np.zeros(4))
    assert res.converged and res.iterations == 0


@pytest.mark.parametrize("seed", range(6))
def test_pcg_matches_oracle(seed):
    from paper_1007_3753_b200 import numerics
    rng = np.random.default_rng(42 + seed)
    n = int(rng.integers(2, 300))
    M = spd(rng, n)
    b = rng.standard_normal(n)
    diag = np.diag(M).copy() if seed % 2 else None
    res = numerics.pcg_solve(M, b, precond=diag, tol=1e-12, max_iter=n)
    x, conv, its, rr = O.pcg(lambda v: M @ v, b, diag=diag, tol=1e-12, max_iter=n)
    assert res.converged == conv
    assert abs(res.iterations - its) <= 1
    exact = np.linalg.solve(M, b)
    assert np.linalg.norm(res.x - exact) / np.linalg.norm(exact) <= 1e-8
    # budget exhaustion returns the best iterate, not converged
    res2 = numerics.pcg_solve(M, b, tol=1e-30, max_iter=3)
    x2, conv2, its2, rr2 = O.pcg(lambda v: M @ v, b, tol=1e-30, max_iter=3)
    assert not res2.converged and res2.iterations == its2 == 3
    np.testing.assert_allclose(res2.x, x2, rtol=1e-9, atol=1e-12)
    assert abs(res2.residual - rr2) <= 1e-9 * max(rr2, 1.0)


def test_spectral_norm_matches_oracle():
    from paper_1007_3753_b200 import numerics
    rng = np.random.default_rng(3)
    for shape in ((20, 40), (40, 20), (300, 700)):
        A = rng.standard_normal(shape)
        got = numerics.spectral_norm_sq(A)
        assert abs(got - O.power_norm_sq(A)) <= 1e-9 * got
        assert abs(got - np.linalg.eigvalsh(A.T @ A).max()) <= 1e-5 * got
    with pytest.raises(ValueError):
        numerics.spectral_norm_sq(np.zeros((3, 3)))


# ------------------------------------------------------------ operators
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_dense_dictionary_methods(dtype):
    from paper_1007_3753_b200.operators import DenseDictionary
    rng = np.random.default_rng(7)
    A = rng.standard_normal((50, 120))
    D = DenseDictionary(A, dtype=dtype)
    Ah = A if dtype == "float64" else A.astype(np.float32).astype(np.float64)
    tol = 1e-12 if dtype == "float64" else 1e-12
    w = rng.standard_normal(120)
    r = rng.standard_normal(50)
    idx = np.array([3, 7, 100])
    c = rng.standard_normal(3)
    assert D.shape == (50, 120)
    np.testing.assert_allclose(D.apply(w), Ah @ w, rtol=tol, atol=tol * 50)
    np.testing.assert_allclose(D.adjoint(r), Ah.T @ r, rtol=tol, atol=tol * 50)
    np.testing.assert_allclose(D.apply_columns(idx, c), Ah[:, idx] @ c, rtol=tol, atol=tol * 50)
    np.testing.assert_allclose(D.columns_dot(idx, r), Ah[:, idx].T @ r, rtol=tol, atol=tol * 50)
    np.testing.assert_array_equal(D.column(7), Ah[:, 7])
    np.testing.assert_allclose(D.gram_column(idx, 5), Ah[:, idx].T @ Ah[:, 5], rtol=tol, atol=tol * 50)
    np.testing.assert_allclose(D.column_norms_sq(), np.sum(Ah * Ah, axis=0), rtol=1e-12)
    np.testing.assert_allclose(D.gram_dd(), Ah @ Ah.T, rtol=1e-11, atol=1e-10)
    np.testing.assert_allclose(D.weighted_gram_dd(w), (Ah * w) @ Ah.T, rtol=1e-11, atol=1e-10)
    assert abs(D.norm_sq() - O.power_norm_sq(Ah)) <= 1e-9 * D.norm_sq()


def test_solvers_accept_dense_dictionary():
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    from paper_1007_3753_b200.operators import DenseDictionary
    from paper_1007_3753_b200.shrinkage import fista_solve
    rng = np.random.default_rng(2)
    A = rng.standard_normal((40, 90))
    A /= np.linalg.norm(A, axis=0)
    b = A[:, :3] @ np.array([1.0, -2.0, 0.5])
    cfg = SolverConfig(lam=1e-3, tol=1e-7)
    ref = fista_solve(ProblemInstance(A, b), cfg)
    P = ProblemInstance.__new__(ProblemInstance)
    P.A, P.b, P.ground_truth, P.noise_sigma = DenseDictionary(A), b, None, None
    got = fista_solve(P, cfg)
    assert got.iterations == ref.iterations
    np.testing.assert_allclose(got.x_star, ref.x_star, rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------ dual_y_solve, solve_named
def test_dual_y_solve_matches_dense():
    from paper_1007_3753_b200.alm import DalmState, dual_y_solve
    from paper_1007_3753_b200.numerics import chol_factor
    rng = np.random.default_rng(4)
    A = rng.standard_normal((30, 80))
    b = rng.standard_normal(30)
    x = rng.standard_normal(80)
    z = np.clip(rng.standard_normal(80), -1, 1)
    st = DalmState(x=x, y=np.zeros(30), z=z, beta=0.7, gram_chol=chol_factor(A @ A.T))
    y = dual_y_solve(st, A, z, b)
    rhs = A @ z - (A @ x - b) / 0.7
    np.testing.assert_allclose(y, np.linalg.solve(A @ A.T, rhs), rtol=1e-9, atol=1e-10)


def test_solve_named_dispatch():
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    from paper_1007_3753_b200.shrinkage import fista_solve
    from paper_1007_3753_b200.gradient_projection import gpsr_solve
    from paper_1007_3753_b200.solvers import SOLVER_NAMES, solve_named
    rng = np.random.default_rng(8)
    A = rng.standard_normal((30, 60))
    A /= np.linalg.norm(A, axis=0)
    b = A[:, :2] @ np.array([1.0, -1.0])
    P = ProblemInstance(A, b)
    cfg = SolverConfig(lam=1e-2, tol=1e-6)
    assert solve_named("fista", P, cfg).iterations == fista_solve(P, cfg).iterations
    g = solve_named("gp", P, cfg)
    assert g.iterations == gpsr_solve(P, 1e-2, cfg).iterations
    for name in SOLVER_NAMES:
        r = solve_named(name, P, cfg)
        assert r.x_star.shape == (60,)
    with pytest.raises(ValueError):
        solve_named("nope", P, cfg)


# ------------------------------------------------------------ reference-API helpers on the device
def test_extended_dictionary_operator_methods():
    from paper_1007_3753_b200.robust import ExtendedDictionary
    rng = np.random.default_rng(12)
    A = rng.standard_normal((30, 50))
    s = 0.7
    E = ExtendedDictionary(A, s)
    B = np.hstack([A, s * np.eye(30)])
    w = rng.standard_normal(80)
    r = rng.standard_normal(30)
    idx = np.array([1, 49, 50, 79])
    c = rng.standard_normal(4)
    np.testing.assert_allclose(E.apply(w), B @ w, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E @ w, B @ w, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.adjoint(r), B.T @ r, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.T @ r, B.T @ r, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.apply_columns(idx, c), B[:, idx] @ c, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.columns_dot(idx, r), B[:, idx].T @ r, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.column(60), B[:, 60])
    np.testing.assert_allclose(E.gram_column(idx, 3), B[:, idx].T @ B[:, 3], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E.column_norms_sq(), np.sum(B * B, axis=0), rtol=1e-12)
    ww = rng.uniform(0.1, 1.0, 80)
    np.testing.assert_allclose(E.weighted_gram_dd(ww), (B * ww) @ B.T, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(E.gram_dd(), B @ B.T, rtol=1e-11, atol=1e-11)
    assert abs(E.norm_sq() - (O.power_norm_sq(A) + s * s)) <= 1e-9 * E.norm_sq()


def test_model_and_solver_helpers_on_device():
    from paper_1007_3753_b200 import model
    from paper_1007_3753_b200.gradient_projection import gpsr_step_size
    from paper_1007_3753_b200.homotopy import PathState, breakpoint_gammas, update_direction
    from paper_1007_3753_b200.numerics import chol_factor
    rng = np.random.default_rng(13)
    A = rng.standard_normal((25, 60))
    b = rng.standard_normal(25)
    x = np.zeros(60)
    x[[2, 9]] = [0.5, -1.0]
    P = model.ProblemInstance(A, b)
    r = b - A @ x
    assert abs(model.objective(x, P, 0.1) - (0.5 * r @ r + 0.1 * np.abs(x).sum())) <= 1e-12
    assert abs(model.kkt_residual(x, P, 0.1) - O.kkt_of(x, A.T @ r, 0.1)) <= 1e-12
    assert abs(model.default_lambda(P) - 1e-2 * np.max(np.abs(A.T @ b))) <= 1e-14
    g = rng.standard_normal(120)
    Av = A @ (g[:60] - g[60:])
    assert abs(gpsr_step_size(g, A) - (g @ g) / (Av @ Av)) <= 1e-12 * (g @ g) / (Av @ Av)
    sup = [2, 9]
    c = A.T @ r
    st = PathState(x, sup, 1.5, c, chol_factor(A[:, sup].T @ A[:, sup]))
    d = update_direction(st, A)
    ref_dI = np.linalg.solve(A[:, sup].T @ A[:, sup], np.sign(c[sup]))
    np.testing.assert_allclose(d[sup], ref_dI, rtol=1e-10)
    mask = np.zeros(60, bool)
    mask[sup] = True
    w = A.T @ (A[:, sup] @ d[sup])
    got = breakpoint_gammas(st, d, A)
    ref = O.step_lengths(1.5, c, x, d, w, mask)
    assert got[1] == ref[1] and got[3] == ref[3]
    np.testing.assert_allclose([got[0], got[2]], [ref[0], ref[2]], rtol=1e-10)
