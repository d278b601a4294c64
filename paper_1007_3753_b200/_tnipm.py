"""Host side of tnipm_solve (gradient_projection.py:218-339) — csrc/tnipm.cu."""

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.model import SolverResult


def tnipm_solve_device(P, lam, config, observer=None):
    from paper_1007_3753_b200.gradient_projection import BarrierIterate
    if lam is None:
        lam = config.resolved_lambda(P)
    if not lam > 0:
        raise ValueError("lambda must be positive")
    prep = Prepared(P, config)
    pcg_tol = float(config.opt("pcg_tol", 1e-4))
    cap = config.opt("pcg_max_iter", None)
    torch = device._torch()
    L = _lib.lib()
    wsb = L.ell1_tnipm_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, config.max_iter + 2)
    ub = torch.zeros(prep.n, dtype=torch.float64, device=prep.dev) if observer is not None else None

    def launch(io):
        return L.ell1_tnipm(byref(prep.view), device.ptr(prep.b), byref(prep.ctrl), float(lam),
                            pcg_tol, int(cap) if cap is not None else 0, device.ptr(ub), byref(io),
                            prep.stream)

    step = None
    if observer is not None:
        def step(st):
            observer(BarrierIterate(host_vec(bufs.x), host_vec(ub), float(st.scal[2])))
    st = drive(launch, bufs, step)
    raise_for(st.status, {_lib.BREAKDOWN: "barrier line search exhausted without an interior "
                                          "decrease"})
    notes = ()
    if st.rot[0]:
        notes = ("pcg hit its iteration cap %d times" % st.rot[0],)
    return SolverResult(bufs.x_host(), int(st.iterations), prep.elapsed(), bool(st.converged),
                        bufs.read_trace(st.ntrace), notes)
