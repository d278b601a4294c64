"""LASSO solution path on the B200 — drop-in for ell1.homotopy.

solve_path / homotopy_solve run as one persistent kernel (csrc/homotopy.cu):
direction solves with the maintained Cholesky factor, support-sparse panel
GEMVs, grid-wide argmins for the breakpoint step lengths and the factor
append / delete (rank-1 update) all happen on the device.  The small host
helpers (update_direction, breakpoint_gammas) keep the reference's
contracts on host arrays for callers that use them directly.
"""

import csv
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.alm import CholFactor
from paper_1007_3753_b200.model import SolverResult, TraceEntry

_TIE = 1e-12
_MIN_STEP_REL = 1e-10


@dataclass
class PathState:
    """Snapshot of the path at one breakpoint (homotopy.py:26-34)."""

    x: np.ndarray
    support: list
    lam: float
    c: np.ndarray
    chol: object


def breakpoint_gammas(state, d, A):
    """Step lengths to the next add / remove event (homotopy.py:78-115); the
    products v = A_I d_I and w = A^T v run on the device."""
    from paper_1007_3753_b200.operators import adjoint_any, apply_any
    if hasattr(A, "A") and isinstance(getattr(A, "A"), np.ndarray) and not hasattr(A, "device_extension"):
        A = A.A
    sup = list(state.support)
    dfull = np.zeros(np.asarray(state.x).shape[0])
    dfull[sup] = np.asarray(d, dtype=np.float64)[sup]
    v = apply_any(A, dfull)
    w = adjoint_any(A, v)
    mask = np.zeros(state.c.shape[0], dtype=bool)
    mask[sup] = True
    return _gammas(state.lam, state.c, state.x, d, w, mask)


def _gammas(lam, c, x, d, w, support_mask):
    off = ~support_mask
    gamma_plus, i_plus = np.inf, -1
    if np.any(off):
        idx = np.nonzero(off)[0]
        co, wo = c[idx], w[idx]
        with np.errstate(divide="ignore", invalid="ignore"):
            r1 = (lam - co) / (1.0 - wo)
            r2 = (lam + co) / (1.0 + wo)
        floor = _MIN_STEP_REL * max(lam, 1e-30)
        for ratios in (r1, r2):
            ok = np.isfinite(ratios) & (ratios > floor)
            if np.any(ok):
                j = int(np.argmin(np.where(ok, ratios, np.inf)))
                if ratios[j] < gamma_plus:
                    gamma_plus, i_plus = float(ratios[j]), int(idx[j])
    gamma_minus, i_minus = np.inf, -1
    sup = np.nonzero(support_mask)[0]
    if sup.size:
        with np.errstate(divide="ignore", invalid="ignore"):
            r = -x[sup] / d[sup]
        ok = np.isfinite(r) & (r > 0)
        if np.any(ok):
            j = int(np.argmin(np.where(ok, r, np.inf)))
            gamma_minus, i_minus = float(r[j]), int(sup[j])
    return gamma_plus, i_plus, gamma_minus, i_minus


def update_direction(state, A):
    """Full-length path direction from the state's factor (homotopy.py:67-75,
    _solve_direction :40-64): the triangular solves and the Gram check
    (A_I^T A_I d_I against the signs) run on the device; a drifted factor is
    replaced by a fresh device Cholesky of the support Gram, and a Gram that
    stays singular raises DegenerateSupportError."""
    from paper_1007_3753_b200.exceptions import DegenerateSupportError, NotPositiveDefiniteError
    from paper_1007_3753_b200.numerics import CholFactor, chol_factor
    from paper_1007_3753_b200.operators import adjoint_any, apply_any
    if hasattr(A, "A") and isinstance(getattr(A, "A"), np.ndarray) and not hasattr(A, "device_extension"):
        A = A.A
    sup = list(state.support)
    n = np.asarray(state.x).shape[0]
    d = np.zeros(n)
    if not sup:
        return d
    sgn = np.sign(state.c[sup])

    def gram_times(dI):
        full = np.zeros(n)
        full[sup] = dI
        return adjoint_any(A, apply_any(A, full))[sup]

    d_I = CholFactor(state.chol.R).solve(sgn)
    tol = 1e-6 * max(1.0, float(np.linalg.norm(sgn)))
    if np.linalg.norm(gram_times(d_I) - sgn) > tol:
        G = np.empty((len(sup), len(sup)))
        for col in range(len(sup)):
            e = np.zeros(len(sup))
            e[col] = 1.0
            G[:, col] = gram_times(e)
        try:
            fresh = chol_factor(G)
        except NotPositiveDefiniteError as exc:
            raise DegenerateSupportError("active-set Gram is singular") from exc
        d_I = fresh.solve(sgn)
        if np.linalg.norm(gram_times(d_I) - sgn) > tol:
            raise DegenerateSupportError("active-set Gram solve failed")
    d[sup] = d_I
    return d


def _dump_path(path_csv, rows):
    if path_csv is None:
        return
    with open(path_csv, "w", newline="", encoding="utf-8") as fh:
        wr = csv.writer(fh, lineterminator="\n")
        wr.writerow(["lambda", "support_size", "objective"])
        for lam, size, obj in rows:
            wr.writerow(["%.17g" % lam, size, "%.17g" % obj])


class _DenseProblem:
    def __init__(self, A, b):
        self.A = A
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        self.ground_truth = None


def solve_path(D, b, target_lambda, config, path_csv=None, observer=None):
    """Run the path on a dictionary down to target_lambda (homotopy.py:128-244).

    D: numpy matrix, DenseDictionary-like (``.A``), DeviceDictionary or
    robust.ExtendedDictionary.  Returns (SolverResult, reached_lambda)."""
    if target_lambda < 0:
        raise ValueError("target lambda must be nonnegative")
    A = D
    if not isinstance(D, np.ndarray) and not hasattr(D, "device_extension") \
            and not isinstance(D, device.DeviceDictionary) and hasattr(D, "A"):
        A = D.A
    P = _DenseProblem(A, b)
    from paper_1007_3753_b200.model import SolverConfig
    cfg = SolverConfig(lam=None, tol=1.0, max_iter=config.max_iter, options=dict(config.options))
    prep = Prepared(P, cfg)
    torch = device._torch()
    L = _lib.lib()
    wsb = L.ell1_homotopy_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, config.max_iter + 2)
    cap = L.ell1_homotopy_capacity(byref(prep.view))
    out = _lib.HomOut()
    cbuf = torch.zeros(prep.n, dtype=torch.float64, device=prep.dev)
    lamp = torch.zeros(config.max_iter + 1, dtype=torch.float64, device=prep.dev)
    out.c = cbuf.data_ptr()
    out.lam_path = lamp.data_ptr()
    supb = Rb = None
    if observer is not None:
        supb = torch.zeros(cap, dtype=torch.int32, device=prep.dev)
        Rb = torch.zeros(cap * cap, dtype=torch.float64, device=prep.dev)
        out.support = supb.data_ptr()
        out.factor = Rb.data_ptr()

    def launch(io):
        return L.ell1_homotopy(byref(prep.view), device.ptr(prep.b), float(target_lambda),
                               int(config.max_iter), byref(out), byref(io), prep.stream)

    step = None
    if observer is not None:
        def step(st):
            m = int(st.rot[0])
            sup = [int(v) for v in supb[:m].cpu().numpy()]
            R = Rb[: m * m].cpu().numpy().reshape(m, m)
            observer(PathState(host_vec(bufs.x), sup, float(st.scal[0]), host_vec(cbuf),
                               CholFactor(R)))
    st = drive(launch, bufs, step)
    raise_for(st.status, {_lib.NOT_PD: "active-set Gram is singular",
                          _lib.DEGENERATE: "active-set Gram is singular"})
    trace = bufs.read_trace(st.ntrace)
    notes = ("ridge-regularized gram",) if st.rot[1] else ()
    x = bufs.x_host()
    lam = float(st.scal[0])
    if path_csv is not None:
        if st.status == _lib.ZERO_DATA:
            rows = [(lam, t.support_size, t.objective) for t in trace]
        else:
            lp = lamp[: len(trace)].cpu().numpy()
            rows = [(float(lp[i]), t.support_size, t.objective) for i, t in enumerate(trace)]
        _dump_path(path_csv, rows)
    res = SolverResult(x, int(st.iterations), prep.elapsed(), bool(st.converged), trace, notes)
    return res, lam


def homotopy_solve(P, target_lambda, config, path_csv=None, observer=None):
    """Path solver on a dense instance down to target_lambda (homotopy.py:257-261)."""
    res, _ = solve_path(P.A, P.b, target_lambda, config, path_csv=path_csv, observer=observer)
    return res
