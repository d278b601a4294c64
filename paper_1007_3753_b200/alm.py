"""Augmented-Lagrangian solvers on the B200 — drop-in for ell1.alm.

dalm_solve runs as one persistent kernel (csrc/dalm.cu); palm_solve as one
persistent kernel (csrc/palm.cu).  The row-Gram factor of the dual solver is
computed once per device dictionary (DeviceDictionary.gram_factor) and
reused across solves.
"""

from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.exceptions import IllConditionedError
from paper_1007_3753_b200.model import SolverResult, TraceEntry
from paper_1007_3753_b200.numerics import CholFactor  # noqa: F401  (alm.CholFactor in the reference)

_INNER_CAP = 200        # alm.py:23
_Y_REFINE_TOL = 1e-10   # alm.py:24
_Y_REFINE_TOL_F32 = 1e-5  # documented fp32-storage scaling of the certificate


@dataclass
class AlmState:
    """Primal multiplier-loop state (alm.py:27-46)."""

    x: np.ndarray
    y: np.ndarray
    mu: float
    rho: float
    tau: float

    def __post_init__(self):
        if not self.mu > 0 or not self.tau > 0:
            raise ValueError("mu and tau must be positive")
        if not self.rho > 1:
            raise ValueError("rho must exceed 1")


@dataclass
class DalmState:
    """Dual three-step iteration state (alm.py:49-68)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    beta: float
    gram_chol: object

    def __post_init__(self):
        if not self.beta > 0:
            raise ValueError("beta must be positive")
        if float(np.max(np.abs(self.z))) > 1.0:
            raise ValueError("z must lie in the unit l-inf ball")


def _dict_and_ext(prep):
    return prep.D, prep.ext, prep.scale


def dalm_solve(P, config, observer=None):
    """Dual three-step iteration: project, least-squares, multiplier.

    Same contract as ell1.alm.dalm_solve (alm.py:206-272): option beta (1),
    y_cg_step (False); converges when ||b - Ax|| <= tol ||b|| and the
    box-scaled duality gap is within tol; observer receives (DalmState,
    x_prev) after every iteration; stopping-rule kkt slot = relative primal
    residual.  Extra options: dtype, device.
    """
    prep = Prepared(P, config)
    beta = float(config.opt("beta", 1.0))
    if not beta > 0:
        raise ValueError("beta must be positive")
    cg_mode = bool(config.opt("y_cg_step", False))
    D = prep.D
    try:
        MT, Gcm, Lfac, _ = D.gram_factor(prep.ext, prep.scale)
    except IllConditionedError:
        if not np.any(np.asarray(P.b)):       # alm.py:223-226: zero data exits first
            return SolverResult(np.zeros(prep.n), 0, prep.elapsed(), True, [TraceEntry(0, 0.0, 0.0, 0)])
        raise
    torch = device._torch()
    O = _lib.DalmOpts()
    O.beta = beta
    O.y_tol = _Y_REFINE_TOL if D.dtype == _lib.F64 else _Y_REFINE_TOL_F32
    O.y_cg_step = 1 if cg_mode else 0
    O.M = MT.data_ptr()
    O.Ginv = Gcm.data_ptr()
    L = _lib.lib()
    wsb = L.ell1_dalm_workspace(byref(prep.view), 0)
    observed = observer is not None
    bufs = Buffers(prep, wsb, config.max_iter + 2, want_prev=observed)
    yb = zb = None
    if observed:
        yb = torch.zeros(prep.ld, dtype=torch.float64, device=prep.dev)
        zb = torch.zeros(prep.n, dtype=torch.float64, device=prep.dev)
        O.y_out = yb.data_ptr()
        O.z_out = zb.data_ptr()

    def launch(io):
        return L.ell1_dalm(byref(prep.view), device.ptr(prep.b), byref(prep.ctrl), byref(O),
                           byref(io), prep.stream)

    step = None
    if observed:
        chol = CholFactor(Lfac.T.contiguous().cpu().numpy())

        def step(st):
            x = bufs.x_host()
            xp = host_vec(bufs.x_prev)
            observer(DalmState(x, host_vec(yb, prep.d), host_vec(zb), beta, chol), xp)
    st = drive(launch, bufs, step)
    raise_for(st.status, {_lib.ILL_CONDITIONED: "dual least-squares step failed its residual "
                                                 "contract" if not cg_mode else
                          "row Gram lost positive definiteness"})
    x = bufs.x_host()
    trace = bufs.read_trace(st.ntrace)
    notes = ()
    if not st.converged and st.iterations >= config.max_iter:
        notes = ("iteration budget exhausted",)
    return SolverResult(x, int(st.iterations), prep.elapsed(), bool(st.converged), trace, notes)


def palm_solve(P, config, observer=None):
    """Primal multiplier loop with inexact accelerated-shrinkage inner solves
    (alm.py:96-159)."""
    from paper_1007_3753_b200._palm import palm_solve_device
    return palm_solve_device(P, config, observer)


def dual_y_solve(state, A, z_next, b):
    """Least-squares multiplier step of the dual iteration (alm.py:172-189):
    solve beta A A^T y = beta A z_next - (A x - b) through state.gram_chol,
    certify ||rhs - A A^T y|| <= 1e-10 max(1, ||rhs||), refine once, else
    IllConditionedError.  Products, solves and norms run on the device."""
    import ctypes
    from paper_1007_3753_b200.operators import DenseDictionary
    torch = device._torch()
    op = A if isinstance(A, DenseDictionary) else DenseDictionary(A)
    D = op.device_dictionary()
    dev, d, n = D.device, D.d, D.n
    L = _lib.lib()
    st = device.stream_ptr(dev)
    R = np.ascontiguousarray(state.gram_chol.R, dtype=np.float64)
    if R.shape != (d, d):
        raise ValueError("gram factor must be d x d")
    Rd = torch.from_numpy(R).to(dev)
    zd = device.to_device_vec(np.asarray(z_next, np.float64), n, dev)
    xd = device.to_device_vec(np.asarray(state.x, np.float64), n, dev)
    bd = device.to_device_vec(np.asarray(b, np.float64), D.ld, dev)
    Az = op._apply_dev(zd)
    Ax = op._apply_dev(xd)
    t = torch.empty_like(Ax)
    _lib.check(L.ell1_axpby(d, 1.0, device.ptr(Ax), -1.0, device.ptr(bd), device.ptr(t), st), "ell1_axpby")
    rhs = torch.zeros_like(Ax)
    _lib.check(L.ell1_axpby(d, 1.0, device.ptr(Az), -1.0 / float(state.beta), device.ptr(t), device.ptr(rhs), st),
               "ell1_axpby")
    s2 = torch.zeros(2, dtype=torch.float64, device=dev)

    def solve(v):
        out = torch.zeros_like(v)
        _lib.check(L.ell1_chol_solve(device.ptr(Rd), device.ptr(v), device.ptr(out), d, st), "ell1_chol_solve")
        return out

    def residual(y):
        AAy = op._apply_dev(op._adjoint_dev(y))
        res = torch.zeros_like(y)
        _lib.check(L.ell1_axpby(d, 1.0, device.ptr(rhs), -1.0, device.ptr(AAy), device.ptr(res), st),
                   "ell1_axpby")
        _lib.check(L.ell1_sumsq(d, device.ptr(res), device.ptr(s2[1:]), st), "ell1_sumsq")
        return res

    y = solve(rhs)
    _lib.check(L.ell1_sumsq(d, device.ptr(rhs), device.ptr(s2), st), "ell1_sumsq")
    res = residual(y)
    h = s2.cpu().numpy()
    scale = max(1.0, float(np.sqrt(h[0])))
    if float(np.sqrt(h[1])) > _Y_REFINE_TOL * scale:
        dy = solve(res)
        y2 = torch.zeros_like(y)
        _lib.check(L.ell1_axpby(d, 1.0, device.ptr(y), 1.0, device.ptr(dy), device.ptr(y2), st), "ell1_axpby")
        y = y2
        residual(y)
        if float(np.sqrt(s2.cpu().numpy()[1])) > _Y_REFINE_TOL * scale:
            raise IllConditionedError("dual least-squares step failed its residual contract")
    return y[:d].cpu().numpy()
