"""Gradient-projection and log-barrier solvers on the B200 — drop-in for
ell1.gradient_projection (gradient_projection.py).

gpsr_solve runs as one persistent kernel (csrc/gpsr.cu); tnipm_solve as one
persistent kernel with the PCG inner solve on the device (csrc/tnipm.cu).
The small helpers (gpsr_direction, gpsr_step_size, SplitIterate,
BarrierIterate) keep the reference's host contracts.
"""

from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.model import SolverResult, TraceEntry

_ALPHA_CAP = 1e8
_CURV_FLOOR = 1e-14


@dataclass
class SplitIterate:
    """Nonnegative split z = [x_plus; x_minus] (gradient_projection.py:29-48)."""

    z: np.ndarray

    def __post_init__(self):
        self.z = np.ascontiguousarray(self.z, dtype=np.float64)
        if self.z.ndim != 1 or self.z.shape[0] % 2:
            raise ValueError("z must be a vector of even length 2n")
        if np.any(self.z < 0):
            raise ValueError("split iterate must be componentwise nonnegative")

    @property
    def n(self):
        return self.z.shape[0] // 2

    def recombined(self):
        return self.z[: self.n] - self.z[self.n:]


@dataclass
class BarrierIterate:
    """Interior point (x, u, t) with |x_i| < u_i and t > 0 (gradient_projection.py:51-67)."""

    x: np.ndarray
    u: np.ndarray
    t: float

    def __post_init__(self):
        self.x = np.ascontiguousarray(self.x, dtype=np.float64)
        self.u = np.ascontiguousarray(self.u, dtype=np.float64)
        if self.x.shape != self.u.shape or self.x.ndim != 1:
            raise ValueError("x and u must be vectors of equal length")
        if not np.all(np.abs(self.x) < self.u):
            raise ValueError("barrier iterate must satisfy |x_i| < u_i")
        if not self.t > 0:
            raise ValueError("t must be positive")


def _split_vector(z):
    if isinstance(z, SplitIterate):
        return z.z
    z = np.ascontiguousarray(z, dtype=np.float64)
    if z.ndim != 1 or z.shape[0] % 2:
        raise ValueError("z must be a vector of even length 2n")
    return z


def gpsr_direction(z, grad):
    """Masked gradient (gradient_projection.py:79-90)."""
    zv = _split_vector(z)
    g = np.ascontiguousarray(grad, dtype=np.float64)
    if g.shape != zv.shape:
        raise ValueError("z and grad must have equal length")
    return np.where((zv > 0.0) | (g < 0.0), g, 0.0)


def gpsr_step_size(g, A):
    """Exact 1-D step gg / ||A (g+ - g-)||^2, capped at 1e8 when flat
    (gradient_projection.py:93-111)."""
    g = np.ascontiguousarray(g, dtype=np.float64)
    if g.ndim != 1 or g.shape[0] % 2:
        raise ValueError("g must be a vector of even length 2n")
    gg = float(g @ g)
    if gg == 0.0:
        raise ValueError("g must be nonzero")
    n = g.shape[0] // 2
    from paper_1007_3753_b200.operators import apply_any
    Av = apply_any(A, g[:n] - g[n:])
    curvature = float(Av @ Av)
    if curvature <= _CURV_FLOOR * gg:
        return _ALPHA_CAP
    return gg / curvature


_GPSR_NOTES = {1: "zero projected gradient before kkt tolerance", 2: "projection backtracking stalled"}


def gpsr_solve(P, lam, config, observer=None):
    """Projected steepest descent on the nonnegative split
    (gradient_projection.py:114-192); lam=None resolves the default weight."""
    if lam is None:
        lam = config.resolved_lambda(P)
    if not lam > 0:
        raise ValueError("lambda must be positive")
    prep = Prepared(P, config)
    torch = device._torch()
    L = _lib.lib()
    wsb = L.ell1_gpsr_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, config.max_iter + 2)
    zb = torch.zeros(2 * prep.n, dtype=torch.float64, device=prep.dev) if observer is not None else None

    def launch(io):
        return L.ell1_gpsr(byref(prep.view), device.ptr(prep.b), byref(prep.ctrl), float(lam),
                           device.ptr(zb), byref(io), prep.stream)

    step = None
    if observer is not None:
        def step(st):
            observer(SplitIterate(host_vec(zb)))
    st = drive(launch, bufs, step)
    raise_for(st.status, {})
    notes = (_GPSR_NOTES[st.rot[2]],) if st.rot[2] in _GPSR_NOTES else ()
    return SolverResult(bufs.x_host(), int(st.iterations), prep.elapsed(), bool(st.converged),
                        bufs.read_trace(st.ntrace), notes)


def tnipm_solve(P, lam, config, observer=None):
    """Truncated-Newton log-barrier solver (gradient_projection.py:218-339)."""
    from paper_1007_3753_b200._tnipm import tnipm_solve_device
    return tnipm_solve_device(P, lam, config, observer)
