"""Host side of ist_solve (shrinkage.py:105-181) — launches csrc/ist.cu."""

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import Buffers, Prepared, byref, drive, host_vec, raise_for
from paper_1007_3753_b200.model import SolverResult


def ist_solve_device(P, schedule, config, observer=None):
    from paper_1007_3753_b200.shrinkage import default_schedule
    prep = Prepared(P, config)
    if schedule is None:
        schedule = default_schedule(P, config.resolved_lambda(P))   # shrinkage.py:118-119
    stages = np.asarray(schedule.stages(), dtype=np.float64)
    sd = device.to_device_vec(stages, stages.shape[0], prep.dev)
    L = _lib.lib()
    wsb = L.ell1_ist_workspace(byref(prep.view), 0)
    bufs = Buffers(prep, wsb, config.max_iter + 2)

    def launch(io):
        return L.ell1_ist(byref(prep.view), device.ptr(prep.b), byref(prep.ctrl), device.ptr(sd),
                          int(stages.shape[0]), byref(io), prep.stream)

    step = None
    if observer is not None:
        def step(st):
            observer(host_vec(bufs.x), float(st.scal[1]), float(st.scal[4]))
    st = drive(launch, bufs, step)
    raise_for(st.status, {})
    return SolverResult(bufs.x_host(), int(st.iterations), prep.elapsed(), bool(st.converged),
                        bufs.read_trace(st.ntrace))
