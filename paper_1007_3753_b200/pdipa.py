"""Primal-dual interior-point solver — drop-in for ell1.pdipa (pdipa.py:1-185).

min ||x||_1 s.t. A x = b as the split LP min 1'v, [A, -A] v = b, v >= 0.
Per Newton step the device runs: two dictionary products (panel GEMV /
GEMV^T), the weighted row Gram M = A diag(w+ + w-) A^T (the library's DMMA
GEMM, ``ell1_gram_dd``), the fused residual / elimination / step-to-boundary /
duality-measure kernels of csrc/pdipa.cu, and one d x d Cholesky factor +
solve of M (csrc/chol.cu: blocked panels, DMMA trailing updates, with the
reference's one jitter retry).  The host loop here only sequences those calls and reads
back a few scalars per step; it follows the reference's control flow
exactly (jitter retry, non-finite / stalled-measure stops, notes, trace).
"""

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200.exceptions import IllConditionedError
from paper_1007_3753_b200.model import SolverResult, TraceEntry

_BOUNDARY = 0.99   # pdipa.py:19
_SIGMA = 0.1       # pdipa.py:20
_FEAS_TOL = 1e-8   # pdipa.py:21
_GAP_TOL = 1e-6    # pdipa.py:22


@dataclass
class PdipaState:
    """Strictly interior primal-dual iterate of the split LP (pdipa.py:26-32)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    mu: float


class _Ops:
    """Device operator for the LP: plain A (n columns) or the implicit
    [A, sI] of robust.ExtendedDictionary (N = n + d columns)."""

    def __init__(self, A, config):
        torch = device._torch()
        self.torch = torch
        self.L = _lib.lib()
        ext = getattr(A, "device_extension", None)
        if ext is not None:
            D, s = ext()
            self.s = float(s)
            self.ext = True
        else:
            D, _ = device.as_device_dictionary(A, config)
            self.s = 0.0
            self.ext = False
        self.D = D
        self.view = D.view()
        self.dev = D.device
        self.st = device.stream_ptr(self.dev)
        self.d, self.n, self.ld = D.d, D.n, D.ld
        self.N = self.n + (self.d if self.ext else 0)
        wsb = self.L.ell1_gemv_workspace(ctypes.byref(self.view))
        self.gws, self.gwsb = device.alloc_bytes(wsb, self.dev), wsb
        gb = self.L.ell1_gram_dd_workspace(ctypes.byref(self.view))
        self.grws, self.grwsb = device.alloc_bytes(gb, self.dev), gb
        self.pws = device.alloc_bytes(self.L.ell1_pd_workspace(), self.dev)

    def zeros(self, k):
        return self.torch.zeros(max(int(k), 1), dtype=self.torch.float64, device=self.dev)

    def apply(self, u, out):
        """out[:d] = A_ext u  (u: N)."""
        _lib.check(self.L.ell1_gemv(ctypes.byref(self.view), device.ptr(u), device.ptr(out),
                                    device.ptr(self.gws), self.gwsb, self.st), "ell1_gemv")
        if self.ext:                                        # robust.py:91-93
            _lib.check(self.L.ell1_axpby(self.d, self.s, device.ptr(u[self.n:]), 1.0, device.ptr(out),
                                         device.ptr(out), self.st), "ell1_axpby")

    def adjoint(self, r, out):
        """out[:N] = A_ext^T r."""
        _lib.check(self.L.ell1_gemv_t(ctypes.byref(self.view), device.ptr(r), device.ptr(out),
                                      device.ptr(self.gws), self.gwsb, self.st), "ell1_gemv_t")
        if self.ext:                                        # robust.py:95-96
            _lib.check(self.L.ell1_axpby(self.d, self.s, device.ptr(r), 0.0, None, device.ptr(out[self.n:]),
                                         self.st), "ell1_axpby")

    def gram(self, wsum, M):
        """M = A_ext diag(wsum) A_ext^T (robust.py:145-149 for [A, sI])."""
        _lib.check(self.L.ell1_gram_dd(ctypes.byref(self.view), device.ptr(wsum), device.ptr(M),
                                       device.ptr(self.grws), self.grwsb, self.st), "ell1_gram_dd")
        tr = self.zeros(1)
        v = wsum[self.n:] if self.ext else None
        _lib.check(self.L.ell1_pd_diag(self.d, self.d, device.ptr(M), self.s ** 2, device.ptr(v),
                                       device.ptr(tr), self.st), "ell1_pd_diag")
        return tr

    def factor_solve(self, M, rhs, tr):
        """dy = M^-1 rhs with the reference's one jitter retry (pdipa.py:43-52):
        the library's blocked Cholesky (chol.cu; DMMA trailing updates) and
        triangular solves."""
        torch = self.torch
        d = self.d
        if getattr(self, "_Lf", None) is None:
            self._Lf = torch.empty(d * d, dtype=torch.float64, device=self.dev)
            self._cst = torch.zeros(1, dtype=torch.int32, device=self.dev)
        Lf, cst = self._Lf, self._cst
        _lib.check(self.L.ell1_chol_factor_dense(d, device.ptr(M), d, 0.0, device.ptr(Lf), d, device.ptr(cst),
                                                 self.st), "ell1_chol_factor_dense")
        if int(cst.item()) != 0:
            jit = 1e-12 * max(float(tr.item()) / d, 1.0)
            _lib.check(self.L.ell1_chol_factor_dense(d, device.ptr(M), d, jit, device.ptr(Lf), d, device.ptr(cst),
                                                     self.st), "ell1_chol_factor_dense")
            if int(cst.item()) != 0:
                raise IllConditionedError("weighted normal matrix is singular")
        out = torch.empty(d, dtype=torch.float64, device=self.dev)
        _lib.check(self.L.ell1_chol_solve_dense(d, device.ptr(Lf), d, device.ptr(rhs), device.ptr(out), self.st),
                   "ell1_chol_solve_dense")
        return out


def pdipa_solve(P, config, observer=None):
    """Interior-point solve of min ||x||_1 s.t. A x = b (pdipa.py:97-185).

    Returns the recombined signed estimate; observer, when given, receives
    the PdipaState after every accepted step."""
    t0 = time.perf_counter()
    b_host = np.asarray(P.b, dtype=np.float64)
    o = _Ops(P.A, config)
    L, st = o.L, o.st
    torch = o.torch
    d, N = o.d, o.N
    if float(np.linalg.norm(b_host)) == 0.0:
        return SolverResult(np.zeros(N), 0, time.perf_counter() - t0, True, [TraceEntry(0, 0.0, 0.0, 0)])
    nn = 2 * N
    x = torch.ones(nn, dtype=torch.float64, device=o.dev)
    z = torch.ones(nn, dtype=torch.float64, device=o.dev)
    y = o.zeros(o.ld)
    b = device.to_device_vec(b_host, o.ld, o.dev)
    u = o.zeros(N)
    Ax = o.zeros(o.ld)
    Aty = o.zeros(N)
    rp = o.zeros(o.ld)
    rd = o.zeros(nn)
    rc, w, dx, dz = o.zeros(nn), o.zeros(nn), o.zeros(nn), o.zeros(nn)
    wsum, vd = o.zeros(N), o.zeros(N)
    rhs = o.zeros(o.ld)
    M = o.zeros(d * d)
    sc = o.zeros(8)
    mu = 1.0                                               # x'z / 2N at x = z = 1
    b_scale = max(1.0, float(np.linalg.norm(b_host)))
    c_scale = 1.0 + math.sqrt(nn)
    gap_tol = min(config.tol, _GAP_TOL)
    pws = device.ptr(o.pws)
    trace, notes = [], []
    converged = False
    it = 0
    while it < config.max_iter:
        # residuals, objective, gap, support of x+ - x- (pdipa.py:136-146)
        _lib.check(L.ell1_pd_split(N, 1, device.ptr(x), device.ptr(u), device.ptr(sc[4:]), pws, st),
                   "ell1_pd_split")
        o.apply(u, Ax)
        o.adjoint(y, Aty)
        _lib.check(L.ell1_pd_resid(d, N, 1, device.ptr(Ax), device.ptr(b), device.ptr(y), device.ptr(Aty),
                                   device.ptr(x), device.ptr(z), None, device.ptr(rp), device.ptr(rd),
                                   device.ptr(sc), pws, st), "ell1_pd_resid")
        h = sc.cpu().numpy()
        cut = 1e-10 * max(float(h[4]), 1.0)                # model.py:227-233
        k8 = o.zeros(8)
        _lib.check(L.ell1_shard_kkt(N, device.ptr(u), device.ptr(u), 0.0, cut, device.ptr(k8), pws, st),
                   "ell1_shard_kkt")
        rpn, rdn, obj = math.sqrt(h[0]), math.sqrt(h[2]), float(h[3])
        gap = obj - float(h[1])
        trace.append(TraceEntry(it, obj, rpn, int(round(float(k8[4].item())))))
        if rpn <= _FEAS_TOL * b_scale and rdn <= _FEAS_TOL * c_scale and gap <= gap_tol * (1.0 + abs(obj)):
            converged = True
            break
        it += 1
        # Newton step by elimination (pdipa.py:147-160, 55-62)
        _lib.check(L.ell1_pd_prep(N, 1, device.ptr(x), device.ptr(z), device.ptr(rd), _SIGMA * mu,
                                  device.ptr(rc), device.ptr(w), device.ptr(wsum), device.ptr(vd), st),
                   "ell1_pd_prep")
        tr = o.gram(wsum, M)
        o.apply(vd, rhs)
        _lib.check(L.ell1_axpby(d, 1.0, device.ptr(rp), -1.0, device.ptr(rhs), device.ptr(rhs), st),
                   "ell1_axpby")
        try:
            dy = o.factor_solve(M, rhs, tr)
        except IllConditionedError:
            notes.append("stopped on ill-conditioned normal matrix")
            break
        dyp = o.zeros(o.ld)
        dyp[:d] = dy
        o.adjoint(dyp, Aty)
        _lib.check(L.ell1_pd_direction(N, 1, d, device.ptr(Aty), device.ptr(dyp), device.ptr(rd), device.ptr(rc),
                                       device.ptr(x), device.ptr(z), device.ptr(w), device.ptr(dx),
                                       device.ptr(dz), device.ptr(sc), pws, st), "ell1_pd_direction")
        h = sc.cpu().numpy()
        if h[2] != 0.0:
            notes.append("stopped on non-finite step")
            break
        ap = 1.0 if not np.isfinite(h[0]) else min(1.0, _BOUNDARY * float(h[0]))   # pdipa.py:35-40
        ad = 1.0 if not np.isfinite(h[1]) else min(1.0, _BOUNDARY * float(h[1]))
        ok = False
        for _ in range(40):                                 # pdipa.py:165-174
            _lib.check(L.ell1_pd_mu(nn, device.ptr(x), device.ptr(dx), ap, device.ptr(z), device.ptr(dz), ad,
                                    device.ptr(sc), pws, st), "ell1_pd_mu")
            mu_new = float(sc[0].item()) / nn
            if mu_new < mu:
                ok = True
                break
            ap *= 0.5
            ad *= 0.5
        if not ok:
            notes.append("stopped on stalled duality measure")
            break
        _lib.check(L.ell1_pd_update(nn, d, device.ptr(x), device.ptr(dx), ap, device.ptr(z), device.ptr(dz), ad,
                                    device.ptr(y), device.ptr(dyp), st), "ell1_pd_update")
        mu = mu_new
        if observer is not None:
            observer(PdipaState(x.cpu().numpy().copy(), y[:d].cpu().numpy().copy(), z.cpu().numpy().copy(), mu))
    xv = x.cpu().numpy()
    return SolverResult(xv[:N] - xv[N:], it, time.perf_counter() - t0, converged, trace, notes=tuple(notes))


def newton_kkt_step(state, A_ext, b, mu_hat, c=None):
    """Newton direction on the perturbed optimality system of an explicit
    A_ext with the 1e-8 residual contract (pdipa.py:65-94); returns host
    (dx, dy, dz) or raises IllConditionedError."""
    torch = device._torch()
    A_ext = np.asarray(A_ext, dtype=np.float64)
    o = _Ops(A_ext, None)
    L, st = o.L, o.st
    d, N = o.d, o.N
    x = device.to_device_vec(state.x, N, o.dev)
    z = device.to_device_vec(state.z, N, o.dev)
    y = device.to_device_vec(state.y, o.ld, o.dev)
    bd = device.to_device_vec(np.asarray(b, np.float64), o.ld, o.dev)
    cd = device.to_device_vec(np.ones(N) if c is None else np.asarray(c, np.float64), N, o.dev)
    Ax, Aty = o.zeros(o.ld), o.zeros(N)
    rp, rd, rc, w, wsum, vd, dx, dz = (o.zeros(o.ld), o.zeros(N), o.zeros(N), o.zeros(N), o.zeros(N),
                                       o.zeros(N), o.zeros(N), o.zeros(N))
    sc = o.zeros(8)
    pws = device.ptr(o.pws)
    o.apply(x, Ax)
    o.adjoint(y, Aty)
    _lib.check(L.ell1_pd_resid(d, N, 0, device.ptr(Ax), device.ptr(bd), device.ptr(y), device.ptr(Aty),
                               device.ptr(x), device.ptr(z), device.ptr(cd), device.ptr(rp), device.ptr(rd),
                               device.ptr(sc), pws, st), "ell1_pd_resid")
    h = sc.cpu().numpy().copy()
    _lib.check(L.ell1_pd_prep(N, 0, device.ptr(x), device.ptr(z), device.ptr(rd), float(mu_hat), device.ptr(rc),
                              device.ptr(w), device.ptr(wsum), device.ptr(vd), st), "ell1_pd_prep")
    M = o.zeros(d * d)
    tr = o.gram(wsum, M)
    rhs = o.zeros(o.ld)
    o.apply(vd, rhs)
    _lib.check(L.ell1_axpby(d, 1.0, device.ptr(rp), -1.0, device.ptr(rhs), device.ptr(rhs), st), "ell1_axpby")
    dy = o.factor_solve(M, rhs, tr)
    dyp = o.zeros(o.ld)
    dyp[:d] = dy
    o.adjoint(dyp, Aty)
    _lib.check(L.ell1_pd_direction(N, 0, d, device.ptr(Aty), device.ptr(dyp), device.ptr(rd), device.ptr(rc),
                                   device.ptr(x), device.ptr(z), device.ptr(w), device.ptr(dx), device.ptr(dz),
                                   device.ptr(sc), pws, st), "ell1_pd_direction")
    hd = sc.cpu().numpy().copy()
    # residual contract: ||A dx - rp||, ||A^T dy + dz - rd||, ||z dx + x dz - rc|| <= 1e-8 scale
    rcn = o.zeros(1)
    _lib.check(L.ell1_sumsq(N, device.ptr(rc), device.ptr(rcn), st), "ell1_sumsq")
    Adx = o.zeros(o.ld)
    o.apply(dx, Adx)
    t8 = o.zeros(8)
    tmp = o.zeros(max(o.ld, N))
    _lib.check(L.ell1_shard_resid(d, device.ptr(Adx), device.ptr(rp), device.ptr(rp), 0.0, device.ptr(tmp),
                                  device.ptr(t8), pws, st), "ell1_shard_resid")
    e1 = float(t8[0].item())
    _lib.check(L.ell1_axpby(N, 1.0, device.ptr(Aty), 1.0, device.ptr(dz), device.ptr(Aty), st), "ell1_axpby")
    _lib.check(L.ell1_shard_resid(N, device.ptr(Aty), device.ptr(rd), device.ptr(rd), 0.0, device.ptr(tmp),
                                  device.ptr(t8), pws, st), "ell1_shard_resid")
    e2 = float(t8[0].item())
    scale = max(1.0, math.sqrt(h[0]), math.sqrt(h[2]), math.sqrt(float(rcn.item())))
    ok = (math.sqrt(e1) <= 1e-8 * scale and math.sqrt(e2) <= 1e-8 * scale and math.sqrt(hd[3]) <= 1e-8 * scale)
    if not ok or hd[2] != 0.0:
        raise IllConditionedError("Newton system residual did not close")
    return dx.cpu().numpy(), dy.cpu().numpy(), dz.cpu().numpy()
