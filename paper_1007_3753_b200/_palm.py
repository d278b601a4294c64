"""Host side of palm_solve (alm.py:96-159) — launches csrc/palm.cu."""

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.model import SolverResult


def palm_solve_device(P, config, observer=None):
    from paper_1007_3753_b200.alm import AlmState
    prep = Prepared(P, config)
    mu = float(config.opt("mu0", 1.0))
    rho = float(config.opt("rho", 2.0))
    if not mu > 0 or not rho > 1:
        raise ValueError("mu0 must be positive and rho must exceed 1")
    torch = device._torch()
    O = _lib.PalmOpts()
    O.mu0, O.rho = mu, rho
    import numpy as np
    if not np.any(np.asarray(P.b)):
        O.tau = 1.0              # zero data exits before tau is needed (alm.py:111-114)
    else:
        A = P.A
        O.tau = 1.01 * (A.norm_sq() if hasattr(A, "norm_sq") else prep.D.norm_sq())   # alm.py:119-122
    L = _lib.lib()
    wsb = L.ell1_palm_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, config.max_iter + 2)
    yb = None
    if observer is not None:
        yb = torch.zeros(prep.ld, dtype=torch.float64, device=prep.dev)
        O.y_out = yb.data_ptr()

    def launch(io):
        return L.ell1_palm(byref(prep.view), device.ptr(prep.b), byref(prep.ctrl), byref(O),
                           byref(io), prep.stream)

    step = None
    if observer is not None:
        def step(st):
            observer(AlmState(host_vec(bufs.x), host_vec(yb, prep.d), float(st.scal[4]), rho, O.tau))
    st = _drive_outer(launch, bufs, step)
    raise_for(st.status, {})
    x = bufs.x_host()
    trace = bufs.read_trace(st.ntrace)
    notes = ()
    if not st.converged and st.iterations >= config.max_iter:
        notes = ("inner-iteration budget exhausted",)
    return SolverResult(x, int(st.iterations), prep.elapsed(), bool(st.converged), trace, notes)


def _drive_outer(launch, bufs, step):
    """Like _runner.drive, but the observer granularity is an outer iteration
    (tracked by ntrace)."""
    if step is None:
        return drive(launch, bufs, None)
    while True:
        before = bufs.read_state().ntrace
        _lib.check(launch(bufs.io(1)), "solver launch")
        st = bufs.read_state()
        if st.status not in (_lib.OK, _lib.RUNNING, _lib.ZERO_DATA):
            return st
        if st.ntrace > max(before, 1) and st.status != _lib.ZERO_DATA:
            step(st)
        if st.status != _lib.RUNNING:
            return st
