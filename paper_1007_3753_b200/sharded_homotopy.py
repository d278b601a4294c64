"""Column-sharded single-instance Homotopy.

The LASSO path of homotopy.solve_path (reference homotopy.py:128-244) for a
dictionary whose columns are split across ranks (one process per GPU, the
same ShardedDictionary as the sharded FISTA):

* sharded — the two A^T passes of every breakpoint, the correlation
  c = A^T (b - A_I x_I) (homotopy.py:186-188, 226) and w = A^T v
  (homotopy.py:225), run on each rank's column panel; the add-event step
  lengths (homotopy.py:78-105) are computed per rank and folded across ranks
  with the reference's tie rules (first index of the ra pass wins, rb only if
  strictly smaller);
* replicated — the active columns A_I (broadcast by their owner when they
  enter the path, one d-vector), the upper factor of A_I^T A_I, x_I, the
  direction d_I = (A_I^T A_I)^-1 sgn(c_I) with the reference's drift check,
  dense refactorisation and ridge fallback (homotopy.py:41-64, 118-125),
  v = A_I d_I and the residual; every rank runs the identical device
  arithmetic, so all ranks take identical decisions.

Collectives per breakpoint: the correlation exchange (c on the support
columns + max|c|), the step-length exchange, and on an add the column
broadcast.  The device work is libell1b200.so (gemv / gemv_t panels,
chol_* factor kernels, csrc/shard_hom.cu reductions, the DMMA GEMM for
dense refactorisations); this module is the host control loop, as in the
reference.  Every rank returns the same (SolverResult, lambda reached).
"""

import ctypes
import math
import time

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError
from paper_1007_3753_b200.model import SolverResult, TraceEntry
from paper_1007_3753_b200.sharded import TorchCollective, column_range

TIE = 1e-12            # homotopy.py:22 (removal wins ties within 1e-12)
DRIFT = 1e-6           # homotopy.py:50
LAM_WINDOW = 1e-9      # homotopy.py:231


class _Degenerate(Exception):
    pass


class DeviceHomShardOps:
    """One rank's device state: its column panel plus the replicated active
    set.  Vectors are float64 torch tensors; factors are row-major m x m."""

    SLOT = 4

    def __init__(self, shard, coll=None):
        torch = device._torch()
        self.torch = torch
        self.L = _lib.lib()
        D = shard.local
        self.D = D
        self.view = D.view()
        self.dev = D.device
        self.stream = device.stream_ptr(self.dev)
        self.d, self.nl, self.ld = D.d, D.n, D.ld
        self.n = shard.n
        self.coll = coll if coll is not None else TorchCollective(shard.group)
        self.world, self.rank = self.coll.world, self.coll.rank
        self.c0, c1 = column_range(shard.n, self.rank, self.world)
        if (shard.c0, shard.c1) != (self.c0, c1):
            raise ValueError("shard columns differ from column_range(n, rank, world)")
        self.maxcap = min(self.d, self.n) + 32
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.gws = int(self.L.ell1_gemv_workspace(ctypes.byref(self.view)))
        self.ws = torch.zeros(max(self.gws, 256), dtype=torch.uint8, device=self.dev)
        self.cap = 0
        self.S = None                                               # active columns (column-major, ld)
        self._ensure(min(256, self.maxcap))
        self.c = torch.zeros(max(self.nl, 1), **f64)
        self.w = torch.zeros(max(self.nl, 1), **f64)
        self.mask = torch.zeros(max(self.nl, 1), dtype=torch.uint8, device=self.dev)
        self.small = torch.zeros(8, **f64)
        self.st = torch.zeros(1, dtype=torch.int32, device=self.dev)

    # ---- helpers
    def _ensure(self, m):
        """Room for m active columns (grown by doubling, at most min(d, n) + 32)."""
        if m <= self.cap:
            return
        torch = self.torch
        cap = min(max(m, 2 * self.cap), self.maxcap)
        S = torch.zeros(cap, self.ld, dtype=torch.float64, device=self.dev)
        if self.S is not None:
            S[: self.cap] = self.S
        self.S, self.cap = S, cap
        v = self._Sview(cap)
        self.sws = int(self.L.ell1_gemv_workspace(ctypes.byref(v)))
        self.sws_t = torch.zeros(max(self.sws, 256), dtype=torch.uint8, device=self.dev)

    def _Sview(self, m):
        v = _lib.Dict()
        v.A, v.dtype, v.ext, v.d, v.n, v.ld = self.S.data_ptr(), _lib.F64, 0, self.d, max(m, 1), self.ld
        return v

    def vec_d(self):
        return self.torch.zeros(self.ld, dtype=self.torch.float64, device=self.dev)

    def vec_m(self, m):
        return self.torch.zeros(max(m, 1), dtype=self.torch.float64, device=self.dev)

    def set_b(self, b):
        self.b = device.to_device_vec(b, self.ld, self.dev)
        self.bnorm = float(np.linalg.norm(b))

    # ---- sharded passes and exchanges
    def corr(self, r):
        """c = A_r^T r on this rank's columns."""
        _lib.check(self.L.ell1_gemv_t(ctypes.byref(self.view), device.ptr(r), device.ptr(self.c),
                                      device.ptr(self.ws), self.gws, self.stream), "ell1_gemv_t")

    def corr_exchange(self, sup):
        """-> (c_I (device, m), max|c|, first argmax (global index))."""
        torch = self.torch
        m = len(sup)
        buf = torch.zeros(m + self.SLOT * self.world, dtype=torch.float64, device=self.dev)
        mine = [(p, j - self.c0) for p, j in enumerate(sup) if self.c0 <= j < self.c0 + self.nl]
        if mine:
            pos = torch.tensor([p for p, _ in mine], dtype=torch.int64, device=self.dev)
            loc = torch.tensor([q for _, q in mine], dtype=torch.int64, device=self.dev)
            buf[pos] = self.c[loc]
        _lib.check(self.L.ell1_hom_absmax(self.nl, device.ptr(self.c), device.ptr(self.small), self.stream),
                   "ell1_hom_absmax")
        slot = buf[m + self.SLOT * self.rank: m + self.SLOT * (self.rank + 1)]
        slot[:2] = self.small[:2]
        slot[1] += self.c0
        if self.nl == 0:
            slot[0], slot[1] = -1.0, -1.0
        self.coll.allreduce_(buf)
        sl = buf[m:].view(self.world, self.SLOT).cpu().numpy()
        best, arg = -1.0, -1
        for r in range(self.world):                 # ranks own increasing column ranges
            if sl[r, 1] >= 0 and sl[r, 0] > best:
                best, arg = float(sl[r, 0]), int(sl[r, 1])
        return buf[:m].clone(), max(best, 0.0), arg

    def wpass(self, v):
        _lib.check(self.L.ell1_gemv_t(ctypes.byref(self.view), device.ptr(v), device.ptr(self.w),
                                      device.ptr(self.ws), self.gws, self.stream), "ell1_gemv_t")

    def gammas(self, lam):
        """Add events over all ranks' off-support columns -> (gamma+, index)."""
        torch = self.torch
        buf = torch.zeros(self.SLOT * self.world, dtype=torch.float64, device=self.dev)
        _lib.check(self.L.ell1_hom_gammas(self.nl, device.ptr(self.c), device.ptr(self.w), device.ptr(self.mask),
                                          float(lam), device.ptr(self.small), self.stream), "ell1_hom_gammas")
        slot = buf[self.SLOT * self.rank: self.SLOT * (self.rank + 1)]
        slot[:] = self.small[:4]
        self.coll.allreduce_(buf)
        sl = buf.view(self.world, self.SLOT).cpu().numpy()
        ga, ia, gb, ib = math.inf, -1, math.inf, -1
        for r in range(self.world):
            if sl[r, 1] >= 0 and sl[r, 0] < ga:
                ga, ia = float(sl[r, 0]), int(sl[r, 1]) + column_range(self.n, r, self.world)[0]
            if sl[r, 3] >= 0 and sl[r, 2] < gb:
                gb, ib = float(sl[r, 2]), int(sl[r, 3]) + column_range(self.n, r, self.world)[0]
        if gb < ga:                                   # homotopy.py:92-100: the rb pass must be strictly smaller
            return gb, ib
        return ga, ia

    def fetch_column(self, j):
        """Column j of A on every rank (its owner broadcasts it)."""
        col = self.vec_d()
        if self.c0 <= j < self.c0 + self.nl:
            src = self.D.storage.view(self.nl, self.ld)[j - self.c0]
            col.copy_(src.to(self.torch.float64))
        self.coll.allreduce_(col)
        return col

    def set_mask(self, j, on):
        if self.c0 <= j < self.c0 + self.nl:
            self.mask[j - self.c0] = 1 if on else 0

    # ---- replicated active-set arithmetic
    def store_put(self, m, col):
        self._ensure(m + 1)
        self.S[m].copy_(col)

    def store_drop(self, pos, m):
        if pos < m - 1:
            self.S[pos:m - 1] = self.S[pos + 1:m].clone()
        self.S[m - 1].zero_()

    def S_times(self, m, xI):
        """A_I x_I (d)."""
        out = self.vec_d()
        if m:
            _lib.check(self.L.ell1_gemv(ctypes.byref(self._Sview(m)), device.ptr(xI), device.ptr(out),
                                        device.ptr(self.sws_t), self.sws, self.stream), "ell1_gemv")
        return out

    def St_times(self, m, v):
        """A_I^T v (m)."""
        out = self.vec_m(m)
        if m:
            _lib.check(self.L.ell1_gemv_t(ctypes.byref(self._Sview(m)), device.ptr(v), device.ptr(out),
                                          device.ptr(self.sws_t), self.sws, self.stream), "ell1_gemv_t")
        return out[:m]

    def resid(self, m, xI):
        r = self.S_times(m, xI)
        _lib.check(self.L.ell1_axpby(self.ld, 1.0, device.ptr(self.b), -1.0, device.ptr(r), device.ptr(r),
                                     self.stream), "ell1_axpby")
        return r

    def sumsq(self, v, n):
        _lib.check(self.L.ell1_sumsq(n, device.ptr(v), device.ptr(self.small), self.stream), "ell1_sumsq")
        return float(self.small[0].item())

    def norm(self, v, n):
        return math.sqrt(self.sumsq(v, n))

    def matvec(self, G, m, x):
        """G (m x m, symmetric) x on the DMMA path."""
        out = self.vec_m(m)
        _lib.check(self.L.ell1_gemm_f64(0, 0, m, 1, m, device.ptr(G), m, device.ptr(x), m, device.ptr(out), m,
                                        self.stream), "ell1_gemm_f64")
        return out[:m]

    def gram_ridge(self, m):
        """homotopy.py:118-125: A_I^T A_I + 1e-12 max(trace, 1) I."""
        G = self.gram(m)
        Gm = G.view(m, m)
        tr = float(Gm.diagonal().sum().item())
        Gm.diagonal().add_(1e-12 * max(tr, 1.0))
        return G

    def remove_entry(self, x, pos, m):
        keep = [q for q in range(m) if q != pos]
        return x[keep].clone() if keep else self.vec_m(1)[:0]

    def append_zero(self, x, m):
        xn = self.vec_m(m + 1)
        xn[:m] = x[:m]
        return xn

    def gram(self, m):
        """G = A_I^T A_I (m x m) on the DMMA path."""
        G = self.torch.empty(m * m, dtype=self.torch.float64, device=self.dev)
        _lib.check(self.L.ell1_gemm_f64(1, 0, m, m, self.d, device.ptr(self.S), self.ld, device.ptr(self.S),
                                        self.ld, device.ptr(G), m, self.stream), "ell1_gemm_f64")
        return G

    def chol(self, G, m):
        R = self.torch.zeros(m * m, dtype=self.torch.float64, device=self.dev)
        _lib.check(self.L.ell1_chol_factor(device.ptr(G), device.ptr(R), m, device.ptr(self.st), self.stream),
                   "ell1_chol_factor")
        if int(self.st.item()) != 0:
            raise NotPositiveDefiniteError("active-set Gram is not positive definite")
        return R

    def solve(self, R, m, rhs):
        out = self.vec_m(m)
        _lib.check(self.L.ell1_chol_solve(device.ptr(R), device.ptr(rhs), device.ptr(out), m, self.stream),
                   "ell1_chol_solve")
        return out[:m]

    def grow(self, R, m, g, diag):
        Rout = self.torch.zeros((m + 1) * (m + 1), dtype=self.torch.float64, device=self.dev)
        work = self.vec_m(m)
        Rin = R if m else self.vec_m(1)
        gin = g if m else self.vec_m(1)
        _lib.check(self.L.ell1_chol_append(device.ptr(Rin), m, device.ptr(gin), float(diag), device.ptr(Rout),
                                           device.ptr(work), device.ptr(self.st), self.stream), "ell1_chol_append")
        if int(self.st.item()) != 0:
            raise NotPositiveDefiniteError("appended column makes the Gram singular")
        return Rout

    def drop(self, R, m, k):
        """numerics.chol_delete (numerics.py:140-158): block permutation and
        one rank-1 update of the trailing block."""
        torch = self.torch
        Rm = R.view(m, m)
        out = torch.zeros(m - 1, m - 1, dtype=torch.float64, device=self.dev)
        out[:k, :k] = Rm[:k, :k]
        out[:k, k:] = Rm[:k, k + 1:]
        if k < m - 1:
            tail = Rm[k + 1:, k + 1:].contiguous()
            v = Rm[k, k + 1:].contiguous()
            _lib.check(self.L.ell1_chol_update(device.ptr(tail), device.ptr(v), m - 1 - k, device.ptr(self.st),
                                               self.stream), "ell1_chol_update")
            out[k:, k:] = tail.view(m - 1 - k, m - 1 - k)
        return out.view(-1)

    def gamma_minus(self, m, xI, dI, sup):
        """Remove events over the support; ties go to the lowest column index
        (the reference scans the support mask in index order)."""
        keys = self.torch.tensor(sup, dtype=self.torch.int64, device=self.dev)
        _lib.check(self.L.ell1_hom_gamma_minus(m, device.ptr(xI), device.ptr(dI), device.ptr(keys),
                                               device.ptr(self.small), self.stream), "ell1_hom_gamma_minus")
        h = self.small[:2].cpu().numpy()
        return float(h[0]), int(h[1])

    def xstats(self, m, xI):
        _lib.check(self.L.ell1_hom_xstats(m, device.ptr(xI), device.ptr(self.small), self.stream),
                   "ell1_hom_xstats")
        h = self.small[:2].cpu().numpy()
        return float(h[0]), int(round(h[1]))

    def axpy(self, a, x, y):
        """y += a x (device, m entries)."""
        n = int(y.numel())
        _lib.check(self.L.ell1_axpby(n, float(a), device.ptr(x), 1.0, device.ptr(y), device.ptr(y), self.stream),
                   "ell1_axpby")

    def sign(self, v):
        return self.torch.sign(v)

    def to_host(self, v):
        return v.cpu().numpy().copy()


def _direction(o, R, m, sgn):
    """homotopy.py:41-64: d_I from the maintained factor, checked against the
    Gram; dense refactor on drift, Degenerate when that fails too."""
    dI = o.solve(R, m, sgn)
    v = o.S_times(m, dI)
    Gd = o.St_times(m, v)
    tol = DRIFT * max(1.0, o.norm(sgn, m))
    diff = Gd - sgn
    if o.norm(diff, m) <= tol:
        return dI, R, v
    G = o.gram(m)
    try:
        Rf = o.chol(G, m)
    except NotPositiveDefiniteError as exc:
        raise _Degenerate() from exc
    dI = o.solve(Rf, m, sgn)
    if o.norm(o.matvec(G, m, dI) - sgn, m) > tol:
        raise _Degenerate()
    return dI, Rf, o.S_times(m, dI)


def _ridge(o, m, notes):
    """homotopy.py:118-125: dense Gram + 1e-12 max(trace, 1) on the diagonal."""
    G = o.gram_ridge(m)
    if "ridge-regularized gram" not in notes:
        notes.append("ridge-regularized gram")
    return o.chol(G, m)


def sharded_solve_path(P, target_lambda, config, ops=None):
    """LASSO path to target_lambda on a column-sharded dictionary
    (homotopy.solve_path contract, homotopy.py:128-244).  Call collectively on
    every rank; every rank returns (SolverResult with the full x, lambda)."""
    t0 = time.perf_counter()
    if target_lambda < 0:
        raise ValueError("target lambda must be nonnegative")
    shard = P.A
    o = ops if ops is not None else DeviceHomShardOps(shard)
    n = shard.n
    b = np.asarray(P.b, dtype=np.float64)
    o.set_b(b)
    notes = []
    trace = []
    o.corr(o.b)                                            # c = A^T b
    _, lam0, j0 = o.corr_exchange([])
    target = float(target_lambda)

    def log(k, lam_k, rnorm, m, xI):
        l1, cnt = o.xstats(m, xI) if m else (0.0, 0)
        trace.append(TraceEntry(k, 0.5 * rnorm ** 2 + lam_k * l1, rnorm, cnt))

    if lam0 <= target or lam0 == 0.0:
        lam = max(lam0, target)
        trace.append(TraceEntry(0, 0.5 * o.bnorm ** 2, o.bnorm, 0))
        return SolverResult(np.zeros(n), 0, time.perf_counter() - t0, True, trace, ()), lam
    lam = lam0
    sup = [j0]
    col = o.fetch_column(j0)
    o.store_put(0, col)
    o.set_mask(j0, True)
    R = o.grow(None, 0, None, o.sumsq(col, o.d))
    xI = o.vec_m(1)[:1]
    cI, _, _ = o.corr_exchange(sup)
    done = False
    it = 0
    floor = max(target, 1e-12 * lam0)
    while it < config.max_iter:
        it += 1
        m = len(sup)
        sgn = o.sign(cI)
        try:
            dI, R, v = _direction(o, R, m, sgn)
        except _Degenerate:
            R = _ridge(o, m, notes)
            dI = o.solve(R, m, sgn)
            v = o.S_times(m, dI)
        o.wpass(v)
        gp, ip = o.gammas(lam)
        gm, im_pos = o.gamma_minus(m, xI, dI, sup)
        ge = min(gp, gm)
        cap = lam - target
        if cap <= ge:                                      # final partial step (homotopy.py:208-215)
            o.axpy(cap, dI, xI)
            lam = target
            r = o.resid(m, xI)
            log(it, lam, o.norm(r, o.d), m, xI)
            done = True
            break
        remove = gm <= gp + TIE
        gam = gm if remove else gp
        o.axpy(gam, dI, xI)
        if remove:
            pos = im_pos
            j = sup.pop(pos)
            o.set_mask(j, False)
            xI = o.remove_entry(xI, pos, m)
            o.store_drop(pos, m)
            R = o.drop(R, m, pos)
        else:
            col = o.fetch_column(ip)
            gcol = o.St_times(m, col)
            dg = o.sumsq(col, o.d)
            o.store_put(m, col)
            try:
                R = o.grow(R, m, gcol, dg)
                sup.append(ip)
            except NotPositiveDefiniteError:
                sup.append(ip)
                R = _ridge(o, m + 1, notes)
            o.set_mask(ip, True)
            xI = o.append_zero(xI, m)
        m = len(sup)
        r = o.resid(m, xI)
        o.corr(r)
        cI, lam_emp, _ = o.corr_exchange(sup)
        lam_step = lam - gam
        if abs(lam_emp - lam_step) <= LAM_WINDOW * max(lam_step, 1e-30) or not sup:
            lam = lam_step
        else:
            lam = lam_emp
        log(it, lam, o.norm(r, o.d), m, xI)
        if lam <= floor:
            done = True
            break
    x = np.zeros(n)
    if sup:
        x[np.asarray(sup)] = o.to_host(xI)[: len(sup)]
    return SolverResult(x, it, time.perf_counter() - t0, done, trace, tuple(notes)), lam


def sharded_homotopy_solve(P, target_lambda, config, ops=None):
    """homotopy_solve (homotopy.py:257-261) on a ShardedInstance."""
    res, _ = sharded_solve_path(P, target_lambda, config, ops)
    return res
