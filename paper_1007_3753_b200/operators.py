"""Dictionary operator with the reference's interface (ell1.operators.DenseDictionary,
operators.py:13-58), backed by a device copy of A.

Every method computes on the GPU through libell1b200.so (panel GEMV /
GEMV^T, column norms, the Gram GEMM) and returns host float64 arrays like the
reference's.  The solvers accept a DenseDictionary wherever they accept A
(it carries the DeviceDictionary upload, so repeated solves reuse it).
"""

import ctypes

import numpy as np

from paper_1007_3753_b200 import _lib, device


class DenseDictionary:
    """Explicit dense dictionary D of shape (d, N) resident on the device."""

    def __init__(self, A, dtype="float64", device_ordinal=None):
        if isinstance(A, device.DeviceDictionary):
            self._dev = A
        else:
            A = np.ascontiguousarray(A, dtype=np.float64)
            if A.ndim != 2:
                raise ValueError("dictionary must be a matrix")
            self._dev = device.DeviceDictionary(A, dtype=dtype, device=device_ordinal)
        self._norm_sq = None
        self._ws = None

    # the solvers' hook: run on this device copy
    def device_dictionary(self):
        return self._dev

    @property
    def shape(self):
        return self._dev.shape

    def _gws(self):
        D = self._dev
        if self._ws is None:
            v = D.view()
            wsb = _lib.lib().ell1_gemv_workspace(ctypes.byref(v))
            self._ws = (device.alloc_bytes(wsb, D.device), wsb)
        return self._ws

    def _apply_dev(self, xd):
        torch = device._torch()
        D = self._dev
        v = D.view()
        ws, wsb = self._gws()
        y = torch.zeros(D.ld, dtype=torch.float64, device=D.device)
        _lib.check(_lib.lib().ell1_gemv(ctypes.byref(v), device.ptr(xd), device.ptr(y), device.ptr(ws), wsb,
                                        device.stream_ptr(D.device)), "ell1_gemv")
        return y

    def _adjoint_dev(self, rd):
        torch = device._torch()
        D = self._dev
        v = D.view()
        ws, wsb = self._gws()
        g = torch.zeros(D.n, dtype=torch.float64, device=D.device)
        _lib.check(_lib.lib().ell1_gemv_t(ctypes.byref(v), device.ptr(rd), device.ptr(g), device.ptr(ws), wsb,
                                          device.stream_ptr(D.device)), "ell1_gemv_t")
        return g

    def apply(self, w):
        """D w (operators.py:26-27)."""
        D = self._dev
        w = np.asarray(w, dtype=np.float64)
        if w.ndim == 2:
            return np.stack([self.apply(w[:, j]) for j in range(w.shape[1])], axis=1)
        if w.shape[0] != D.n:
            raise ValueError("operand length %d does not match %d columns" % (w.shape[0], D.n))
        return self._apply_dev(device.to_device_vec(w, D.n, D.device))[: D.d].cpu().numpy()

    def adjoint(self, r):
        """D^T r (operators.py:29-30)."""
        D = self._dev
        r = np.asarray(r, dtype=np.float64)
        if r.ndim == 2:
            return np.stack([self.adjoint(r[:, j]) for j in range(r.shape[1])], axis=1)
        if r.shape[0] != D.d:
            raise ValueError("operand length %d does not match %d rows" % (r.shape[0], D.d))
        return self._adjoint_dev(device.to_device_vec(r, D.ld, D.device)).cpu().numpy()

    def apply_columns(self, idx, coeffs):
        """D[:, idx] @ coeffs (operators.py:32-33): a GEMV over a scattered x."""
        D = self._dev
        idx = np.asarray(idx, dtype=np.int64)
        coeffs = np.asarray(coeffs, dtype=np.float64)
        x = np.zeros(D.n)
        np.add.at(x, idx, coeffs)
        return self.apply(x)

    def columns_dot(self, idx, v):
        """D[:, idx]^T v (operators.py:35-36)."""
        return self.adjoint(v)[np.asarray(idx, dtype=np.int64)]

    def column(self, j):
        """D[:, j] (operators.py:38-39), read back from the device copy."""
        D = self._dev
        j = int(j)
        if not -D.n <= j < D.n:
            raise IndexError("column %d out of range" % j)
        j %= D.n
        return D.storage.view(D.n, D.ld)[j, : D.d].double().cpu().numpy()

    def gram_column(self, idx, j):
        """D[:, idx]^T D[:, j] (operators.py:41-42)."""
        return self.columns_dot(idx, self.column(j))

    def column_norms_sq(self):
        """sum_i D_ij^2 per column (operators.py:44-45)."""
        torch = device._torch()
        D = self._dev
        v = D.view()
        out = torch.zeros(D.n, dtype=torch.float64, device=D.device)
        _lib.check(_lib.lib().ell1_column_norms_sq(ctypes.byref(v), device.ptr(out),
                                                   device.stream_ptr(D.device)), "ell1_column_norms_sq")
        return out.cpu().numpy()

    def norm_sq(self):
        """Largest eigenvalue of D^T D, cached (operators.py:47-51)."""
        if self._norm_sq is None:
            self._norm_sq = self._dev.norm_sq()
        return self._norm_sq

    def _gram(self, w):
        torch = device._torch()
        D = self._dev
        v = D.view()
        L = _lib.lib()
        wsb = L.ell1_gram_dd_workspace(ctypes.byref(v))
        ws = device.alloc_bytes(wsb, D.device)
        G = torch.zeros(D.d * D.d, dtype=torch.float64, device=D.device)
        wd = device.to_device_vec(w, D.n, D.device) if w is not None else None
        _lib.check(L.ell1_gram_dd(ctypes.byref(v), device.ptr(wd), device.ptr(G), device.ptr(ws), wsb,
                                  device.stream_ptr(D.device)), "ell1_gram_dd")
        return G.view(D.d, D.d).cpu().numpy()

    def weighted_gram_dd(self, w):
        """D diag(w) D^T (operators.py:53-55)."""
        w = np.asarray(w, dtype=np.float64)
        if w.shape != (self._dev.n,):
            raise ValueError("weights must have length n")
        return self._gram(w)

    def gram_dd(self):
        """D D^T (operators.py:57-58)."""
        return self._gram(None)


def _device_op(A):
    """A device operator for whatever a caller passed as a dictionary, or None
    for a user-supplied host operator (which then keeps its own arithmetic)."""
    if isinstance(A, DenseDictionary):
        return A
    if isinstance(A, device.DeviceDictionary):
        return DenseDictionary(A)
    if hasattr(A, "device_extension"):          # robust.ExtendedDictionary
        return A
    if isinstance(A, np.ndarray):
        return DenseDictionary(A)
    return None


def apply_any(A, x):
    """A @ x with the product on the device when A is a dense / device /
    extended dictionary (the helper functions of the reference API use it)."""
    op = _device_op(A)
    if op is None:
        return A @ x
    return op.apply(np.asarray(x, dtype=np.float64))


def adjoint_any(A, r):
    """A^T @ r, on the device like apply_any."""
    op = _device_op(A)
    if op is None:
        return A.T @ r
    return op.adjoint(np.asarray(r, dtype=np.float64))
