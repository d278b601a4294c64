"""Host plumbing shared by the drop-in solver entry points.

A solve is: resolve the dictionary (upload or reuse a DeviceDictionary),
upload b (and the ground truth if a rule needs it), allocate the workspace /
state / trace, launch the persistent kernel (once, or one iteration per
launch when an observer is attached), then read back x, the trace and the
state and map the status onto the reference's return values / exceptions.
"""

import ctypes
import time

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200.exceptions import (DegenerateSupportError, DeviceError,
                                             IllConditionedError,
                                             NotPositiveDefiniteError,
                                             NumericalBreakdownError)
from paper_1007_3753_b200.model import TraceEntry


class Prepared:
    """Device-side inputs of one solve."""

    def __init__(self, P, config, ext=False, scale=0.0, need_gt=True):
        self.t0 = time.perf_counter()
        A = P.A
        op_ext = getattr(A, "device_extension", None)
        if op_ext is not None:             # robust.ExtendedDictionary
            D, scale = op_ext()
            ext = True
        else:
            D, _ = device.as_device_dictionary(A, config)
        self.D = D
        self.dev = D.device
        self.ext = ext
        self.scale = float(scale)
        self.view = D.view(ext=ext, scale=scale)
        self.d = D.d
        self.n = D.n + (D.d if ext else 0)       # columns of the operator
        self.ld = D.ld
        self.stream = device.stream_ptr(self.dev)
        self.b = device.to_device_vec(np.asarray(P.b, dtype=np.float64), D.ld, self.dev)
        self.config = config
        stop = config.stopping
        self.ctrl = _lib.Ctrl()
        lam = config.lam
        self.ctrl.lam = -1.0 if lam is None else float(lam)
        self.ctrl.tol = float(config.tol)
        self.ctrl.max_iter = int(config.max_iter)
        self.ctrl.stop_kind = _lib.STOP_CODES[stop.kind if stop is not None else None]
        self.ctrl.stop_thr = float(stop.threshold) if stop is not None else 0.0
        self.gt = None
        self.ctrl.ground_truth = None
        self.ctrl.gt_norm = 0.0
        if stop is not None and stop.kind == "ground-truth-distance" and need_gt:
            gt = getattr(P, "ground_truth", None)
            if gt is None:
                raise ValueError("ground-truth-distance rule needs a ground truth")
            gt = np.asarray(gt, dtype=np.float64)
            nrm = float(np.linalg.norm(gt))
            if nrm == 0.0:
                raise ValueError("ground truth must be nonzero")
            self.gt = device.to_device_vec(gt, self.n, self.dev)
            self.ctrl.ground_truth = self.gt.data_ptr()
            self.ctrl.gt_norm = nrm

    def elapsed(self):
        return time.perf_counter() - self.t0


class Buffers:
    """Workspace + state + trace + output vectors of one solve.

    state (256 bytes), x and the trace share one device allocation so a
    finished solve is read back with a single device->host copy
    (``read_all``) instead of one synchronising copy per field."""

    SNAP_ROWS = 512            # trace rows included in the single read-back (longer traces: one more copy)

    def __init__(self, prep, ws_bytes, trace_rows, want_prev=False, want_y=False):
        torch = device._torch()
        dev = prep.dev
        self.ws = device.alloc_bytes(ws_bytes, dev)
        self.ws_bytes = int(self.ws.numel())
        n = int(prep.n)
        rows = max(int(trace_rows), 1)
        self.n = n
        self.blob = torch.zeros(32 + n + rows * 4, dtype=torch.float64, device=dev)
        self.state = self.blob[:32].view(torch.uint8)
        self.x = self.blob[32:32 + n]
        self.trace = self.blob[32 + n:]
        self.x_prev = torch.zeros(n, dtype=torch.float64, device=dev) if want_prev else None
        self.y = torch.zeros(n, dtype=torch.float64, device=dev) if want_y else None
        self._snap = None

    def io(self, max_steps=0, blocks=0):
        self._snap = None
        io = _lib.IO()
        io.workspace = self.ws.data_ptr()
        io.workspace_bytes = self.ws_bytes
        io.state = self.state.data_ptr()
        io.trace = self.trace.data_ptr()
        io.x = self.x.data_ptr()
        io.x_prev = self.x_prev.data_ptr() if self.x_prev is not None else None
        io.y = self.y.data_ptr() if self.y is not None else None
        io.max_steps = int(max_steps)
        io.blocks = int(blocks)
        return io

    def read_all(self):
        """One copy of state + x + the leading trace rows; returns the state."""
        rows = min(self.trace.numel() // 4, self.SNAP_ROWS)
        self._snap = self.blob[: 32 + self.n + 4 * rows].cpu().numpy()
        return _lib.State.from_buffer_copy(self._snap[:32].tobytes())

    def read_state(self):
        raw = self.state.cpu().numpy().tobytes()
        return _lib.State.from_buffer_copy(raw)

    def x_host(self):
        if self._snap is not None:
            return self._snap[32:32 + self.n].copy()
        return host_vec(self.x)

    def read_trace(self, rows):
        if rows <= 0:
            return []
        if self._snap is not None and rows <= self.SNAP_ROWS:
            t = self._snap[32 + self.n: 32 + self.n + rows * 4].reshape(rows, 4)
        else:
            t = self.trace[: rows * 4].cpu().numpy().reshape(rows, 4)
        # one tolist() instead of numpy scalar indexing per field (~5x less host time per solve)
        return [TraceEntry(int(i), o, r, int(k)) for i, o, r, k in t.tolist()]


def raise_for(status, messages):
    """Map a terminal kernel status onto the reference's exception classes."""
    if status in (_lib.OK, _lib.ZERO_DATA, _lib.RUNNING):
        return
    if status == _lib.LAMBDA_NONPOS:
        raise ValueError(messages.get(status, "lambda must be positive"))
    cls = {_lib.BREAKDOWN: NumericalBreakdownError,
           _lib.ILL_CONDITIONED: IllConditionedError,
           _lib.NOT_PD: NotPositiveDefiniteError,
           _lib.DEGENERATE: DegenerateSupportError}.get(status)
    if cls is not None:
        raise cls(messages.get(status, "numerical failure"))
    raise DeviceError("solver kernel failed with status %d" % status)


def drive(launch, bufs, observer_step=None):
    """Run to completion.  launch(io) issues one kernel launch.

    Without an observer the whole solve is one launch.  With one, each
    launch advances exactly one iteration and observer_step(state) runs on
    the host in between (the reference's per-iteration callback)."""
    if observer_step is None:
        _lib.check(launch(bufs.io(0)), "solver launch")
        return bufs.read_all()
    while True:
        before = bufs.read_state().iterations
        _lib.check(launch(bufs.io(1)), "solver launch")
        st = bufs.read_state()
        if st.status not in (_lib.OK, _lib.RUNNING, _lib.ZERO_DATA):
            return st
        if st.iterations > before and st.status != _lib.ZERO_DATA:
            observer_step(st)
        if st.status != _lib.RUNNING:
            return st


def host_vec(t, n=None):
    a = t.cpu().numpy()
    return a[:n].copy() if n is not None else a.copy()


def byref(s):
    return ctypes.byref(s)
