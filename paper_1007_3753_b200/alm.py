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

_INNER_CAP = 200        # alm.py:23
_Y_REFINE_TOL = 1e-10   # alm.py:24
_Y_REFINE_TOL_F32 = 1e-5  # documented fp32-storage scaling of the certificate


class CholFactor:
    """Upper factor R with R^T R = G (numerics.py:47-72), host copy."""

    __slots__ = ("R",)

    def __init__(self, R):
        R = np.ascontiguousarray(R, dtype=np.float64)
        if R.ndim != 2 or R.shape[0] != R.shape[1]:
            raise ValueError("factor must be square, got shape %r" % (R.shape,))
        self.R = R

    @property
    def dim(self):
        return self.R.shape[0]

    def matrix(self):
        return self.R.T @ self.R

    def copy(self):
        return CholFactor(self.R.copy())


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
        MT, Gcm, Lfac = D.gram_factor(prep.ext, prep.scale)
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
            x = host_vec(bufs.x)
            xp = host_vec(bufs.x_prev)
            observer(DalmState(x, host_vec(yb, prep.d), host_vec(zb), beta, chol), xp)
    st = drive(launch, bufs, step)
    raise_for(st.status, {_lib.ILL_CONDITIONED: "dual least-squares step failed its residual "
                                                 "contract" if not cg_mode else
                          "row Gram lost positive definiteness"})
    x = host_vec(bufs.x)
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
