"""Device-state manager: dictionaries uploaded once, workspaces, streams.

PyTorch is used here only as plumbing — device allocation, host<->device
copies and the current CUDA stream.  All arithmetic happens in
libell1b200.so (csrc/).
"""

import ctypes

import numpy as np

from paper_1007_3753_b200 import _lib
from paper_1007_3753_b200.exceptions import DeviceError

_POWER_SEED = 218751   # numerics.py:224


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available (the B200 path has no CPU fallback)")
    return torch


def current_device(ordinal=None):
    torch = _torch()
    if ordinal is None:
        ordinal = torch.cuda.current_device()
    return torch.device("cuda", int(ordinal))


def stream_ptr(dev):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def alloc_bytes(nbytes, dev):
    torch = _torch()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def to_device_vec(v, length, dev):
    """float64 host vector -> zero-padded device vector of `length` entries."""
    torch = _torch()
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = torch.zeros(length, dtype=torch.float64, device=dev)
    if v.shape[0]:
        # stream-ordered: from pinned memory the copy overlaps the host work that follows
        out[: v.shape[0]].copy_(torch.from_numpy(v), non_blocking=False)
    return out


def _pad32(d):
    return (int(d) + 31) // 32 * 32


class DeviceDictionary:
    """Read-only device copy of a dense dictionary A (d x n).

    Layout: column-major, ld = d rounded up to 32 rows, float64 or float32
    storage (``dtype``).  Pass an instance as ``ProblemInstance.A`` (or to
    ``cab_solve``) to reuse the upload across solves; plain numpy arrays are
    uploaded per call.  ``norm_sq`` mirrors DenseDictionary.norm_sq
    (operators.py:53-56, cached spectral_norm_sq).
    """

    def __init__(self, A, dtype="float64", device=None, _overlap=False):
        torch = _torch()
        L = _lib.lib()
        self.device = current_device(device)
        if isinstance(A, DeviceDictionary):
            raise TypeError("already a DeviceDictionary")
        if isinstance(A, torch.Tensor):
            src = A.to(device=self.device, dtype=torch.float64).contiguous()
        else:
            host = np.ascontiguousarray(A, dtype=np.float64)
            if host.ndim != 2:
                raise ValueError("dictionary must be a matrix")
            # _overlap (solver-internal uploads only): the H2D is left in flight so it
            # overlaps the host-side setup of the solve; safe because the caller's
            # array is used in place (no temporary), stays referenced by the
            # problem, and the solve synchronises before it returns.  Stream
            # order puts ell1_dict_build below after the copy.
            src = torch.from_numpy(host).to(self.device, non_blocking=bool(_overlap and host is A))
        if src.ndim != 2:
            raise ValueError("dictionary must be a matrix")
        self.d, self.n = int(src.shape[0]), int(src.shape[1])
        self.ld = _pad32(self.d)
        self.dtype = {"float64": _lib.F64, "float32": _lib.F32}[str(dtype)]
        tdt = torch.float64 if self.dtype == _lib.F64 else torch.float32
        self.storage = torch.empty(self.n * self.ld, dtype=tdt, device=self.device)
        rc = L.ell1_dict_build(ptr(src), self.d, self.n, self.ld, self.dtype,
                               ptr(self.storage), stream_ptr(self.device))
        _lib.check(rc, "ell1_dict_build")
        self._norm_sq = None

    @classmethod
    def wrap(cls, storage, d):
        """Adopt a device tensor already in the library layout: ``storage`` is
        (n, ld) row-major (= column-major A with leading dimension ld, the
        first d rows of each column used, padding rows zero), float64 or
        float32.  No copy (large dictionaries generated on the device)."""
        torch = _torch()
        _lib.lib()
        if storage.ndim != 2 or not storage.is_cuda or not storage.is_contiguous():
            raise ValueError("storage must be a contiguous (n, ld) CUDA tensor")
        ld = int(storage.shape[1])
        if ld % 32 or ld < int(d):
            raise ValueError("ld must be a multiple of 32 and >= d")
        self = cls.__new__(cls)
        self.device = storage.device
        self.d, self.n, self.ld = int(d), int(storage.shape[0]), ld
        self.dtype = {torch.float64: _lib.F64, torch.float32: _lib.F32}[storage.dtype]
        self.storage = storage.view(-1)
        self._norm_sq = None
        return self

    # -- C ABI view --------------------------------------------------------
    def view(self, ext=False, scale=0.0):
        v = _lib.Dict()
        v.A = self.storage.data_ptr()
        v.dtype = self.dtype
        v.ext = 1 if ext else 0
        v.d, v.n, v.ld = self.d, self.n, self.ld
        v.ext_scale = float(scale)
        return v

    @property
    def shape(self):
        return (self.d, self.n)

    # -- row-Gram factorisation for the dual ALM (alm.py:162-169) ----------
    def gram_factor(self, ext=False, scale=0.0):
        """(M, Ginv, L, G) with G = A A^T (+ s^2 I), L its lower Cholesky factor,
        Ginv = G^{-1} and G (column-major, ld rows, float64) and M = Ginv A in
        the dictionary's layout / dtype.  Computed once per (ext, scale) from the
        device copy of A (so float32 storage factors the rounded A).
        Raises IllConditionedError when G is not positive definite."""
        key = (bool(ext), float(scale) if ext else 0.0)
        cache = self.__dict__.setdefault("_gram", {})
        if key in cache:
            return cache[key]
        torch = _torch()
        from paper_1007_3753_b200.exceptions import IllConditionedError
        L_ = _lib.lib()
        st = stream_ptr(self.device)
        d, n, ld = self.d, self.n, self.ld
        f64 = dict(dtype=torch.float64, device=self.device)
        A64 = self.storage.view(n, ld).to(torch.float64)        # column-major A, ld rows
        G = torch.empty(d * d, **f64)
        # G = A A^T (+ s^2 I) on the DMMA path, its Cholesky factor, G^-1 and
        # M = G^-1 A: the library's own kernels (dmma_gemm.cu, chol.cu)
        _lib.check(L_.ell1_gemm_f64(0, 1, d, d, n, ptr(A64), ld, ptr(A64), ld, ptr(G), d, st), "ell1_gemm_f64")
        if ext:
            tr = torch.zeros(1, **f64)
            ones = torch.ones(d, **f64)
            _lib.check(L_.ell1_pd_diag(d, d, ptr(G), float(scale) ** 2, ptr(ones), ptr(tr), st), "ell1_pd_diag")
        Lf = torch.empty(d * d, **f64)
        info = torch.zeros(1, dtype=torch.int32, device=self.device)
        _lib.check(L_.ell1_chol_factor_dense(d, ptr(G), d, 0.0, ptr(Lf), d, ptr(info), st), "ell1_chol_factor_dense")
        if int(info.item()) != 0:
            raise IllConditionedError("row Gram A A^T is not positive definite; the dual "
                                      "solver needs full row rank")
        eye = torch.eye(d, **f64)
        Gcm = torch.zeros(d, ld, **f64)                         # G^-1, column-major (symmetric)
        _lib.check(L_.ell1_chol_solve_dense_multi(d, ptr(Lf), d, d, ptr(eye), d, ptr(Gcm), ld, st),
                   "ell1_chol_solve_dense_multi")
        M64 = torch.zeros(n, ld, **f64)                         # M = G^-1 A, column-major, ld rows
        _lib.check(L_.ell1_gemm_f64(0, 0, d, n, d, ptr(Gcm), ld, ptr(A64), ld, ptr(M64), ld, st), "ell1_gemm_f64")
        MT = M64 if self.storage.dtype == torch.float64 else M64.to(self.storage.dtype)
        Llow = torch.tril(Lf.view(d, d).T)                     # lower factor (row-major view), observers
        Gld = torch.zeros(d, ld, **f64)                         # G itself, column-major (batched certificate)
        Gld[:, :d] = G.view(d, d)
        cache[key] = (MT, Gcm, Llow, Gld)
        return cache[key]

    # -- operator-protocol hooks ------------------------------------------
    def norm_sq(self):
        """Largest eigenvalue of A^T A (numerics.spectral_norm_sq), cached."""
        if self._norm_sq is None:
            self._norm_sq = spectral_norm_sq_device(self)
        return self._norm_sq


def as_device_dictionary(A, config=None):
    """Return (DeviceDictionary, owned) for whatever the caller passed as A."""
    if isinstance(A, DeviceDictionary):
        return A, False
    if hasattr(A, "device_dictionary"):          # operators.DenseDictionary
        return A.device_dictionary(), False
    dtype = "float64"
    dev = None
    if config is not None:
        dtype = config.opt("dtype", "float64")
        dev = config.opt("device", None)
    return DeviceDictionary(A, dtype=dtype, device=dev, _overlap=True), True


def correlation_max(A, b, device=None):
    """max |A^T b| computed on the device (model.py:126-129)."""
    D, _ = as_device_dictionary(A) if not isinstance(A, DeviceDictionary) else (A, False)
    return _corr(D, D.view(), b)[0]


def _corr(D, view, b):
    torch = _torch()
    L = _lib.lib()
    bd = to_device_vec(b, D.ld, D.device)
    out = torch.zeros(2, dtype=torch.float64, device=D.device)
    wsb = L.ell1_correlation_workspace(ctypes.byref(view))
    ws = alloc_bytes(wsb, D.device)
    rc = L.ell1_correlation_max(ctypes.byref(view), ptr(bd), ptr(out), ptr(ws), wsb,
                                stream_ptr(D.device))
    _lib.check(rc, "ell1_correlation_max")
    o = out.cpu().numpy()
    if np.isnan(o[0]):
        raise DeviceError("ell1_correlation_max: grid barrier timed out")
    return float(o[0]), float(o[1])


def spectral_norm_sq_device(D, tol=1e-6, max_iter=1000):
    """Power iteration on the device with the reference's fixed start vector
    (numerics.py:245-247: default_rng(218751), normalised; redraws follow the
    same generator stream)."""
    torch = _torch()
    L = _lib.lib()
    dim = D.d if D.d <= D.n else D.n
    rng = np.random.default_rng(_POWER_SEED)
    draws = []
    for _ in range(4):
        v = rng.standard_normal(dim)
        v /= np.linalg.norm(v)
        draws.append(v)
    # start vector + 3 redraws, packed with stride dim (kernel indexes v0[k*dim + i])
    vd = to_device_vec(np.concatenate(draws), 4 * dim, D.device)
    out = torch.zeros(2, dtype=torch.float64, device=D.device)
    view = D.view()
    wsb = L.ell1_power_workspace(ctypes.byref(view))
    ws = alloc_bytes(wsb, D.device)
    rc = L.ell1_spectral_norm_sq(ctypes.byref(view), ptr(vd), 3, float(tol), int(max_iter),
                                 ptr(out), ptr(ws), wsb, stream_ptr(D.device))
    _lib.check(rc, "ell1_spectral_norm_sq")
    o = out.cpu().numpy()
    if np.isnan(o[0]):
        raise DeviceError("ell1_spectral_norm_sq: grid barrier timed out")
    return float(o[0])
