"""Shared numerical kernels with the reference's interface (ell1.numerics,
numerics.py:1-261): shrinkage, box projection, the Cholesky machinery,
preconditioned CG and the spectral norm — every computation runs in
libell1b200.so on the GPU (csrc/kernels_misc.cu, csrc/linalg.cu,
csrc/fista.cu power iteration).  Inputs and outputs are host float64 arrays
like the reference's; argument checks and exceptions are the reference's.
"""

from collections import namedtuple

import numpy as np

from paper_1007_3753_b200 import _accel, _lib, device
from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError, NumericalBreakdownError

_POWER_SEED = 218751   # numerics.py:224


def _as_vector(u):
    v = np.ascontiguousarray(u, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError("expected a 1-d real vector, got shape %r" % (v.shape,))
    return v


def soft_threshold(u, a):
    """sgn(u) * max(|u| - a, 0) componentwise (numerics.py:24-37); exact zeros
    for |u_i| <= a; any shape, float64 out."""
    if not np.isscalar(a) and not isinstance(a, np.floating):
        raise ValueError("threshold a must be a scalar")
    a = float(a)
    if not a >= 0.0:
        raise ValueError("threshold a must be nonnegative, got %g" % a)
    arr = np.ascontiguousarray(u, dtype=np.float64)
    out = _accel.soft_threshold(arr.ravel(), a)
    return np.asarray(out).reshape(arr.shape)


def project_box_linf(z):
    """Clamp to [-1, 1] (numerics.py:40-44)."""
    arr = np.ascontiguousarray(z, dtype=np.float64)
    out = _accel.project_box_linf(arr.ravel())
    return np.asarray(out).reshape(arr.shape)


def _dev(a):
    torch = device._torch()
    a = np.ascontiguousarray(a, dtype=np.float64)
    return torch.from_numpy(a).to(device.current_device())


def _stream():
    return device.stream_ptr(device.current_device())


class CholFactor:
    """Upper factor R with R^T R = G (numerics.py:47-72)."""

    __slots__ = ("R",)

    def __init__(self, R):
        R = np.ascontiguousarray(R, dtype=np.float64)
        if R.ndim != 2 or R.shape[0] != R.shape[1]:
            raise ValueError("factor must be square, got shape %r" % (R.shape,))
        self.R = R

    @property
    def dim(self):
        return self.R.shape[0]

    def solve(self, rhs):
        """(R^T R) x = rhs by two triangular solves on the device."""
        rhs = np.asarray(rhs, dtype=np.float64)
        m = self.dim
        if rhs.shape[0] != m:
            raise ValueError("right-hand side length %d does not match factor dim %d" % (rhs.shape[0], m))
        if m == 0:
            return np.zeros_like(rhs)
        torch = device._torch()
        Rd = _dev(self.R)
        cols = rhs.reshape(m, -1)
        out = np.empty_like(cols)
        for c in range(cols.shape[1]):
            bd = _dev(cols[:, c])
            od = torch.empty_like(bd)
            _lib.check(_lib.lib().ell1_chol_solve(device.ptr(Rd), device.ptr(bd), device.ptr(od), m, _stream()),
                       "ell1_chol_solve")
            out[:, c] = od.cpu().numpy()
        return out.reshape(rhs.shape)

    def matrix(self):
        return self.R.T @ self.R

    def copy(self):
        return CholFactor(self.R.copy())


def chol_factor(M):
    """Dense upper Cholesky (numerics.py:75-87); NotPositiveDefiniteError
    when M is not positive definite."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("matrix must be square, got shape %r" % (M.shape,))
    torch = device._torch()
    m = M.shape[0]
    Gd = _dev(M)
    Rd = torch.zeros_like(Gd)
    st = torch.zeros(1, dtype=torch.int32, device=Gd.device)
    _lib.check(_lib.lib().ell1_chol_factor(device.ptr(Gd), device.ptr(Rd), m, device.ptr(st), _stream()),
               "ell1_chol_factor")
    if int(st.item()) != 0:
        raise NotPositiveDefiniteError("Matrix is not positive definite")
    return CholFactor(Rd.cpu().numpy())


def chol_rank1(factor, v, sign):
    """R'^T R' = R^T R + sign v v^T, non-destructive (numerics.py:90-112)."""
    if sign not in (1, -1):
        raise ValueError("sign must be +1 or -1, got %r" % (sign,))
    v = _as_vector(v)
    if v.shape[0] != factor.dim:
        raise ValueError("vector length %d does not match factor dim %d" % (v.shape[0], factor.dim))
    R = factor.R.copy()
    w = v.copy()
    if sign == 1:
        _accel.chol_update(R, w)
    else:
        status = _accel.chol_downdate(R, w)
        if status != 0:
            raise NotPositiveDefiniteError(
                "rank-1 downdate lost positive definiteness at pivot %d" % (status - 1))
    return CholFactor(R)


def chol_append(factor, gram_col, diag):
    """Factor of [[G, g], [g^T, diag]] (numerics.py:115-137)."""
    m = factor.dim
    g = _as_vector(gram_col)
    if g.shape[0] != m:
        raise ValueError("gram column length %d does not match factor dim %d" % (g.shape[0], m))
    torch = device._torch()
    dev = device.current_device()
    Rd = _dev(factor.R) if m else torch.zeros(1, dtype=torch.float64, device=dev)
    gd = _dev(g) if m else torch.zeros(1, dtype=torch.float64, device=dev)
    Rout = torch.zeros((m + 1) * (m + 1), dtype=torch.float64, device=dev)
    work = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().ell1_chol_append(device.ptr(Rd), m, device.ptr(gd), float(diag), device.ptr(Rout),
                                           device.ptr(work), device.ptr(st), _stream()), "ell1_chol_append")
    if int(st.item()) != 0:
        raise NotPositiveDefiniteError("appended column makes the matrix singular")
    return CholFactor(Rout.cpu().numpy().reshape(m + 1, m + 1))


def chol_delete(factor, k):
    """Remove row/column k: block permutation + one rank-1 update of the
    trailing block (numerics.py:140-158)."""
    m = factor.dim
    if not 0 <= k < m:
        raise ValueError("index %d out of range for factor dim %d" % (k, m))
    R = factor.R
    out = np.zeros((m - 1, m - 1))
    out[:k, :k] = R[:k, :k]
    out[:k, k:] = R[:k, k + 1:]
    if k < m - 1:
        trailing = np.ascontiguousarray(R[k + 1:, k + 1:].copy())
        w = R[k, k + 1:].copy()
        _accel.chol_update(trailing, w)
        out[k:, k:] = trailing
    return CholFactor(out)


PcgResult = namedtuple("PcgResult", "x converged iterations residual")


def pcg_solve(op, rhs, precond=None, tol=1e-8, max_iter=None):
    """Jacobi-preconditioned CG for a dense SPD op (numerics.py:164-221) as one
    persistent kernel (ell1_pcg_dense).  op: dense symmetric matrix (host
    array or DeviceDictionary); precond: None or the positive diagonal.
    Matvec callables are host code and have no device form here."""
    torch = device._torch()
    rhs = _as_vector(rhs)
    n = rhs.shape[0]
    if callable(op) and not hasattr(op, "view"):
        raise TypeError("the device pcg_solve takes the dense matrix, not a matvec callable")
    if precond is not None and callable(precond):
        raise TypeError("the device pcg_solve takes a diagonal preconditioner vector")
    dvec = None
    if precond is not None:
        dvec = _as_vector(precond)
        if dvec.shape[0] != n or np.any(dvec <= 0):
            raise ValueError("diagonal preconditioner must be positive, length n")
    if max_iter is None:
        max_iter = n
    M = op if isinstance(op, device.DeviceDictionary) else device.DeviceDictionary(np.asarray(op, np.float64))
    if M.d != n or M.n != n:
        raise ValueError("operator must be n x n")
    dev = M.device
    L = _lib.lib()
    view = M.view()
    rd = device.to_device_vec(rhs, n, dev)
    dd = device.to_device_vec(dvec, n, dev) if dvec is not None else None
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    wsb = L.ell1_pcg_workspace(_lib.ctypes.byref(view))
    ws = device.alloc_bytes(wsb, dev)
    _lib.check(L.ell1_pcg_dense(_lib.ctypes.byref(view), device.ptr(rd), device.ptr(dd), float(tol),
                                int(max_iter), device.ptr(x), device.ptr(out), device.ptr(ws), wsb,
                                device.stream_ptr(dev)), "ell1_pcg_dense")
    o = out.cpu().numpy()
    if int(o[3]) == _lib.ERR_TIMEOUT:
        from paper_1007_3753_b200.exceptions import DeviceError
        raise DeviceError("ell1_pcg_dense: grid barrier timed out")
    if int(o[3]) == _lib.BREAKDOWN:
        raise NumericalBreakdownError("non-finite curvature or residual in PCG")
    return PcgResult(x.cpu().numpy(), bool(o[0]), int(o[1]), float(o[2]))


def spectral_norm_sq(A, tol=1e-6, max_iter=1000):
    """Largest eigenvalue of A^T A by power iteration on the smaller Gram side
    with the reference's fixed start vector (numerics.py:227-261)."""
    if isinstance(A, device.DeviceDictionary):
        return device.spectral_norm_sq_device(A, tol, max_iter)
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2:
        raise ValueError("expected a matrix, got shape %r" % (A.shape,))
    if not np.any(A):
        raise ValueError("spectral norm of the zero matrix is not meaningful here")
    return device.spectral_norm_sq_device(device.DeviceDictionary(A), tol, max_iter)
