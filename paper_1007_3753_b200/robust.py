"""Cross-and-bouquet solving on the implicit [A, s I] dictionary — drop-in for
the CAB half of ell1.robust (robust.py:36-220).

The identity block is never materialised: the device kernels treat the
extension columns as slice-owned (column n + i lives with row i), so D x adds
s * x_ext in the row reduction and D^T r appends s * r (robust.py:91-96).
"""

import numpy as np

from paper_1007_3753_b200 import device
from paper_1007_3753_b200.model import SolverResult

_CAB_BACKENDS = ("pdipa", "homotopy", "gp", "ist", "fista", "palm", "dalm")


class _AdjointView:
    """Transpose-shaped face of an implicit operator (robust.py:36-54)."""

    __slots__ = ("_op",)

    def __init__(self, op):
        self._op = op

    @property
    def shape(self):
        d, w = self._op.shape
        return (w, d)

    @property
    def T(self):
        return self._op

    def __matmul__(self, r):
        return self._op.adjoint(np.asarray(r, dtype=np.float64))


class ExtendedDictionary:
    """Implicit stack [A, s I] of width n + d (robust.py:57-155).

    Solvers of this package read it through ``device_extension()`` (the
    device copy of A plus the scale).  The operator methods of the reference
    API (apply / adjoint / column protocol / Gram hooks / norm_sq) run their
    dictionary products on the device as well.
    """

    mode = "cab"

    def __init__(self, A, identity_scale=1.0, dtype="float64", device_ordinal=None):
        if isinstance(A, device.DeviceDictionary):
            self._dev = A
            self.A = None
        else:
            self.A = np.ascontiguousarray(A, dtype=np.float64)
            if self.A.ndim != 2:
                raise ValueError("dictionary must be a matrix")
            self._dev = None
        if not identity_scale > 0:
            raise ValueError("identity_scale must be positive")
        self.scale = float(identity_scale)
        self._dtype = dtype
        self._ordinal = device_ordinal
        self._norm_sq = None

    # -- device view -------------------------------------------------------
    def device_extension(self):
        if self._dev is None:
            self._dev = device.DeviceDictionary(self.A, dtype=self._dtype, device=self._ordinal)
        return self._dev, self.scale

    def _op(self):
        from paper_1007_3753_b200.operators import DenseDictionary
        if getattr(self, "_dd", None) is None:
            self._dd = DenseDictionary(self.device_extension()[0])
        return self._dd

    # -- operator protocol (products on the device; the identity block is O(d))
    @property
    def shape(self):
        if self.A is not None:
            d, n = self.A.shape
        else:
            d, n = self._dev.d, self._dev.n
        return (d, n + d)

    @property
    def T(self):
        return _AdjointView(self)

    def __matmul__(self, w):
        return self.apply(np.asarray(w, dtype=np.float64))

    def apply(self, w):
        w = np.asarray(w, dtype=np.float64)
        n = self.shape[1] - self.shape[0]
        return self._op().apply(w[:n]) + self.scale * w[n:]

    def adjoint(self, r):
        r = np.asarray(r, dtype=np.float64)
        return np.concatenate([self._op().adjoint(r), self.scale * r])

    def column(self, j):
        d, N = self.shape
        n = N - d
        if j < n:
            return self._op().column(j)
        out = np.zeros(d)
        out[j - n] = self.scale
        return out

    def apply_columns(self, idx, coeffs):
        d, N = self.shape
        n = N - d
        idx = np.asarray(idx, dtype=np.intp)
        coeffs = np.asarray(coeffs, dtype=np.float64)
        out = np.zeros(d)
        lo = idx < n
        if np.any(lo):
            out += self._op().apply_columns(idx[lo], coeffs[lo])
        if np.any(~lo):
            out[idx[~lo] - n] += self.scale * coeffs[~lo]
        return out

    def columns_dot(self, idx, v):
        d, N = self.shape
        n = N - d
        idx = np.asarray(idx, dtype=np.intp)
        out = np.empty(idx.shape[0])
        lo = idx < n
        if np.any(lo):
            out[lo] = self._op().columns_dot(idx[lo], v)
        if np.any(~lo):
            out[~lo] = self.scale * np.asarray(v, dtype=np.float64)[idx[~lo] - n]
        return out

    def gram_column(self, idx, j):
        return self.columns_dot(idx, self.column(j))

    def column_norms_sq(self):
        d = self.shape[0]
        return np.concatenate([self._op().column_norms_sq(), np.full(d, self.scale ** 2)])

    def norm_sq(self):
        """||A||^2 + s^2 (robust.py:139-143), power iteration on the device."""
        if self._norm_sq is None:
            D, s = self.device_extension()
            self._norm_sq = D.norm_sq() + s ** 2
        return self._norm_sq

    def weighted_gram_dd(self, w):
        w = np.asarray(w, dtype=np.float64)
        d, N = self.shape
        n = N - d
        M = self._op().weighted_gram_dd(w[:n])
        M[np.diag_indices(d)] += self.scale ** 2 * w[n:]
        return M

    def gram_dd(self):
        d = self.shape[0]
        M = self._op().gram_dd()
        M[np.diag_indices(d)] += self.scale ** 2
        return M


class _OperatorProblem:
    """Problem shim whose dictionary is an implicit operator (robust.py:158-175)."""

    def __init__(self, op, b):
        self.A = op
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        self.ground_truth = None
        self.noise_sigma = 0.0
        if self.b.shape != (op.shape[0],):
            raise ValueError("b must have length d")

    @property
    def d(self):
        return self.A.shape[0]

    @property
    def n(self):
        return self.A.shape[1]


def _resolved_lambda(config, prob):
    if config.lam is not None:
        return float(config.lam)
    D, s = prob.A.device_extension()
    return 1e-2 * device._corr(D, D.view(ext=True, scale=s), prob.b)[0]


def cab_solve(A, b, solver, config):
    """Solve the corruption-extended system with the chosen backend
    (robust.py:181-220).  Returns (x, e, record) with e = s * w[n:].

    A may be a numpy matrix or a DeviceDictionary (reused across queries).
    """
    if solver not in _CAB_BACKENDS:
        raise ValueError("unknown cab backend %r (choose from %s)"
                         % (solver, ", ".join(_CAB_BACKENDS)))
    e_weight = float(config.opt("e_weight", 1.0))
    if not e_weight > 0:
        raise ValueError("e_weight must be positive")
    scale = 1.0 / e_weight
    ext = ExtendedDictionary(A, identity_scale=scale, dtype=config.opt("dtype", "float64"),
                             device_ordinal=config.opt("device", None))
    prob = _OperatorProblem(ext, b)
    n = ext.shape[1] - ext.shape[0]
    if solver == "dalm":
        from paper_1007_3753_b200.alm import dalm_solve
        res = dalm_solve(prob, config)
    elif solver == "palm":
        from paper_1007_3753_b200.alm import palm_solve
        res = palm_solve(prob, config)
    elif solver == "fista":
        from paper_1007_3753_b200.shrinkage import fista_solve
        res = fista_solve(prob, config)
    elif solver == "ist":
        from paper_1007_3753_b200.shrinkage import ist_solve
        res = ist_solve(prob, None, config)
    elif solver == "gp":
        from paper_1007_3753_b200.gradient_projection import gpsr_solve
        res = gpsr_solve(prob, _resolved_lambda(config, prob), config)
    elif solver == "homotopy":
        from paper_1007_3753_b200.homotopy import solve_path
        res, _ = solve_path(ext, prob.b, _resolved_lambda(config, prob), config)
    else:                                                   # "pdipa" (robust.py:204-205)
        from paper_1007_3753_b200.pdipa import pdipa_solve
        res = pdipa_solve(prob, config)
    w = res.x_star
    return w[:n], scale * w[n:], res


# ---------------------------------------------------------------- alignment
# the alignment solvers (robust.py:223-515), batched
# across images on the device (csrc/align.cu, one CTA per image).

_POWER_SEED = 218751     # numerics.py:224 (IST step size)


class AlignmentProblem:
    """Tall regression b ~ B w with sparse gross error e (robust.py:223-252)."""

    def __init__(self, B, b, ground_truth_w=None, ground_truth_e=None):
        self.B = np.ascontiguousarray(B, dtype=np.float64)
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        self.ground_truth_w = ground_truth_w
        self.ground_truth_e = ground_truth_e
        if self.B.ndim != 2:
            raise ValueError("B must be a matrix")
        if self.B.shape[0] <= self.B.shape[1]:
            raise ValueError("B must be tall: more rows than columns")
        if self.b.shape != (self.B.shape[0],):
            raise ValueError("b must have length d")

    @property
    def d(self):
        return self.B.shape[0]

    @property
    def m(self):
        return self.B.shape[1]


def align_batch_device(kind, Bd, bd, config, lam=None, v0=None):
    """Batched alignment on device-resident images (new; e.g. images coming
    from a GPU pipeline).  Bd: CUDA float64 (count, d, m) row-major images,
    bd: (count, d).  kind: "palm" | "ist" | "homotopy" | "gp".  Returns device
    tensors (W (count, m), E (count, d), iterations (count,)) without syncing;
    raises on a failed image after reading the statuses back."""
    import ctypes
    from paper_1007_3753_b200 import _lib
    from paper_1007_3753_b200._runner import raise_for
    torch = device._torch()
    L = _lib.lib()
    if Bd.ndim != 3 or bd.ndim != 2 or tuple(bd.shape) != tuple(Bd.shape[:2]):
        raise ValueError("need B of shape (count, d, m) and b of shape (count, d)")
    count, d, m = (int(x) for x in Bd.shape)
    if d <= m:
        raise ValueError("B must be tall: more rows than columns")
    if m > 32 or d > 8192:
        raise ValueError("device alignment supports m <= 32 parameters and d <= 8192 rows")
    dev = Bd.device
    Bd = Bd.to(torch.float64).contiguous()
    bd = bd.to(device=dev, dtype=torch.float64).contiguous()
    W = torch.empty((count, m), dtype=torch.float64, device=dev)
    E = torch.empty((count, d), dtype=torch.float64, device=dev)
    st = torch.full((count,), -1, dtype=torch.int32, device=dev)
    its = torch.zeros((count,), dtype=torch.int32, device=dev)
    a = _lib.Align()
    a.count, a.d, a.m, a.max_iter = count, d, m, int(config.max_iter)
    a.B, a.ldb, a.b_stride = Bd.data_ptr(), m, d * m
    a.rhs, a.ld_rhs = bd.data_ptr(), d
    a.tol = float(config.tol)
    a.mu0 = float(config.opt("mu0", 1.0))
    a.rho = float(config.opt("rho", 2.0))
    a.lam = -1.0 if lam is None else float(lam)
    if kind == "ist":
        if v0 is None:
            rng = np.random.default_rng(_POWER_SEED)      # spectral_norm_sq's start vector + redraws
            draws = []
            for _ in range(4):
                v = rng.standard_normal(m)
                draws.append(v / np.linalg.norm(v))
            v0 = torch.from_numpy(np.concatenate(draws)).to(dev)
        a.v0 = v0.data_ptr()
    a.w, a.e, a.status, a.iterations = W.data_ptr(), E.data_ptr(), st.data_ptr(), its.data_ptr()
    kid = {"palm": 0, "ist": 1, "homotopy": 2, "gp": 3}[kind]
    stage = None
    sb = int(L.ell1_align_stage_bytes(kid, count, d, m)) if count else 0
    if sb:                          # B does not fit in shared memory: stage it in global memory
        stage = torch.empty(sb // 8, dtype=torch.float64, device=dev)
        a.Bstage = stage.data_ptr()
    fn = {"palm": L.ell1_align_palm_batch, "ist": L.ell1_align_ist_batch,
          "homotopy": L.ell1_align_homotopy_batch, "gp": L.ell1_align_gp_batch}[kind]
    _lib.check(fn(ctypes.byref(a), device.stream_ptr(dev)), "ell1_align_%s_batch" % kind)
    W._ell1_keep = (Bd, bd, v0, st, stage)                       # operands live until the caller syncs
    W._ell1_status = st
    return W, E, its


def _check_align_status(st):
    from paper_1007_3753_b200 import _lib
    from paper_1007_3753_b200._runner import raise_for
    status = st.cpu().numpy()
    if np.any(status == _lib.NOT_PD):                 # robust.py:254-258
        from paper_1007_3753_b200.exceptions import IllConditionedError
        raise IllConditionedError("B must have full column rank")
    for s in np.unique(status):
        raise_for(int(s), {_lib.ILL_CONDITIONED: "reduced alignment system lost definiteness",
                           _lib.BREAKDOWN: "alignment barrier line search exhausted",
                           _lib.LAMBDA_NONPOS: "lambda must be positive"})


def _align_batch(kind, Bs, bs, config, lam=None):
    """One batched alignment from host arrays.  Bs: (count, d, m), bs: (count, d).
    Returns host (W (count, m), E (count, d), iterations (count,))."""
    torch = device._torch()
    Bs = np.asarray(Bs, dtype=np.float64)
    bs = np.asarray(bs, dtype=np.float64)
    if Bs.ndim != 3 or bs.ndim != 2 or bs.shape != Bs.shape[:2]:
        raise ValueError("need B of shape (count, d, m) and b of shape (count, d)")
    dev = device.current_device(config.opt("device", None))
    Bd = torch.from_numpy(np.ascontiguousarray(Bs)).to(dev)      # row-major images, as given
    bd = torch.from_numpy(np.ascontiguousarray(bs)).to(dev)
    W, E, its = align_batch_device(kind, Bd, bd, config, lam)
    _check_align_status(W._ell1_status)
    return W.cpu().numpy(), E.cpu().numpy(), its.cpu().numpy()


def _palm_options(config):
    mu = float(config.opt("mu0", 1.0))
    rho = float(config.opt("rho", 2.0))
    if not mu > 0 or not rho > 1:
        raise ValueError("mu0 must be positive and rho must exceed 1")


def ist_block_step(B, b, w, e, lam, alpha):
    """One block soft-threshold sweep on the alignment objective
    (robust.py:433-445): r = b - B w - e, w_next = w + B^T r / alpha,
    e_next = soft(e + r / alpha, lam / alpha).  Returns (w_next, e_next);
    ValueError unless alpha > 0.  Runs on the device (ell1_align_ist_step)."""
    import ctypes
    from paper_1007_3753_b200 import _lib
    if not alpha > 0:
        raise ValueError("alpha must be positive")
    torch = device._torch()
    B = np.ascontiguousarray(B, dtype=np.float64)
    d, m = B.shape
    if m > 32:
        raise ValueError("ist_block_step on the device supports m <= 32 columns")
    dev = device.current_device()
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev)  # noqa: E731
    Bd, bd, wd, ed = t(B), t(b), t(w), t(e)
    wn = torch.empty(m, dtype=torch.float64, device=dev)
    en = torch.empty(d, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().ell1_align_ist_step(d, m, Bd.data_ptr(), m, bd.data_ptr(), wd.data_ptr(), ed.data_ptr(),
                                              float(lam), float(alpha), wn.data_ptr(), en.data_ptr(),
                                              device.stream_ptr(dev)), "ell1_align_ist_step")
    return wn.cpu().numpy(), en.cpu().numpy()


def align_palm_solve_batch(Bs, bs, config):
    """align_palm_solve for a batch of images (element j == align_palm_solve
    on (Bs[j], bs[j])).  Returns (W, E)."""
    _palm_options(config)
    W, E, _ = _align_batch("palm", Bs, bs, config)
    return W, E


def align_ist_solve_batch(Bs, bs, lam, config):
    """align_ist_solve for a batch of images; lam=None: per-image default."""
    if lam is not None and not lam > 0:
        raise ValueError("lambda must be positive")
    W, E, _ = _align_batch("ist", Bs, bs, config, lam)
    return W, E


def align_palm_solve(prob, config):
    """Multiplier method for min ||e||_1 s.t. b = B w + e (robust.py:470-515);
    options mu0 (1.0), rho (2.0).  Returns (w, e)."""
    _palm_options(config)
    W, E, _ = _align_batch("palm", prob.B[None], prob.b[None], config)
    return W[0], E[0]


def align_ist_solve(prob, lam, config):
    """Block soft-thresholding on the alignment objective (robust.py:427-467).
    Returns (w, e)."""
    if lam is not None and not lam > 0:
        raise ValueError("lambda must be positive")
    W, E, _ = _align_batch("ist", prob.B[None], prob.b[None], config, lam)
    return W[0], E[0]


def align_homotopy_solve_batch(Bs, bs, config):
    """align_homotopy_solve for a batch of images (target config.lam, default
    1e-2 of each image's peak least-squares residual)."""
    W, E, _ = _align_batch("homotopy", Bs, bs, config, config.lam)
    return W, E


def align_homotopy_solve(prob, config):
    """Path-following in the error block with w re-solved at every step, then
    a block-coordinate cleanup at the target weight (robust.py:374-424).
    Returns (w, e)."""
    W, E, _ = _align_batch("homotopy", prob.B[None], prob.b[None], config, config.lam)
    return W[0], E[0]


def align_gp_solve_batch(Bs, bs, lam, config):
    """align_gp_solve for a batch of images; lam=None: per-image default."""
    if lam is not None and not lam > 0:
        raise ValueError("lambda must be positive")
    W, E, _ = _align_batch("gp", Bs, bs, config, lam)
    return W, E


def align_gp_solve(prob, lam, config):
    """Log-barrier Newton solve of the alignment objective (robust.py:276-371):
    central path in (w, e, u) with -u <= e <= u, one m x m factorisation per
    Newton step, polished exit.  Returns (w, e)."""
    if lam is not None and not lam > 0:
        raise ValueError("lambda must be positive")
    W, E, _ = _align_batch("gp", prob.B[None], prob.b[None], config, lam)
    return W[0], E[0]

