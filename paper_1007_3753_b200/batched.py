"""Batched solvers: many right-hand sides sharing one dictionary (BASELINE
configs 3 and 5).  New entry points — the reference has no batched API —
whose element j equals the single-instance call on (A, b_j)
(SURVEY §8(b)).

The library runs the whole batch: dictionary products are GEMMs over the
active instances, the solver arithmetic runs in per-instance epilogue
kernels, converged instances are compacted out of the batch.
"""

import time
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import byref, raise_for
from paper_1007_3753_b200.model import SolverResult, TraceEntry


@dataclass
class BatchResult:
    """Arrays over the batch (column j = instance j)."""

    x: np.ndarray            # N x B
    iterations: np.ndarray
    converged: np.ndarray
    status: np.ndarray
    wall_time_seconds: float
    trace: np.ndarray = None  # B x rows x 4, or None
    kind: str = "fista"
    max_iter: int = 0
    lam: np.ndarray = None     # homotopy: lambda reached per instance
    notes: np.ndarray = None   # homotopy: ridge flag per instance

    def result(self, j):
        """SolverResult of instance j (reference record type)."""
        st = int(self.status[j])
        raise_for(st, {_lib.BREAKDOWN: "backtracking exceeded 100 growth steps",
                       _lib.ILL_CONDITIONED: "dual least-squares step failed its residual contract",
                       _lib.NOT_PD: "active-set Gram is singular",
                       _lib.DEGENERATE: "active-set Gram is singular"})
        it = int(self.iterations[j])
        tr = []
        if self.trace is not None:
            if st == _lib.ZERO_DATA:
                rows = 1
            else:
                rows = it + 1 if self.kind == "dalm" else it
            tr = [TraceEntry(int(r[0]), float(r[1]), float(r[2]), int(r[3]))
                  for r in self.trace[j, :rows]]
        notes = ()
        if self.kind == "dalm" and not self.converged[j] and it >= self.max_iter:
            notes = ("iteration budget exhausted",)
        if self.kind == "homotopy" and self.notes is not None and self.notes[j]:
            notes = ("ridge-regularized gram",)
        B = self.x.shape[1]
        return SolverResult(self.x[:, j].copy(), it, self.wall_time_seconds / B,
                            bool(self.converged[j]), tr, notes)

    def results(self):
        """Per-instance SolverResult records (reference record type)."""
        return [self.result(j) for j in range(self.x.shape[1])]


def _dict_view(A, config):
    if hasattr(A, "device_extension"):
        D, s = A.device_extension()
        return D, D.view(ext=True, scale=s), D.n + D.d
    D, _ = device.as_device_dictionary(A, config)
    return D, D.view(), D.n


def _ctrl(config, B, N, dev, ground_truth):
    C = _lib.Ctrl()
    C.lam = -1.0 if config.lam is None else float(config.lam)
    C.tol = float(config.tol)
    C.max_iter = int(config.max_iter)
    stop = config.stopping
    C.stop_kind = _lib.STOP_CODES[stop.kind if stop is not None else None]
    C.stop_thr = float(stop.threshold) if stop is not None else 0.0
    C.ground_truth = None
    C.gt_norm = 0.0
    keep = None
    if stop is not None and stop.kind == "ground-truth-distance":
        if ground_truth is None:
            raise ValueError("ground-truth-distance rule needs a ground truth")
        raise NotImplementedError("per-instance ground-truth rule in batch mode")
    return C, keep


def _upload_rhs(Bmat, D):
    torch = device._torch()
    dev = D.device
    if isinstance(Bmat, torch.Tensor):
        Bd = Bmat.to(device=dev, dtype=torch.float64)
    else:
        Bd = torch.from_numpy(np.ascontiguousarray(Bmat, dtype=np.float64)).to(dev)
    d, B = int(Bd.shape[0]), int(Bd.shape[1])
    if d != D.d:
        raise ValueError("Bmat must have d rows")
    Bpad = torch.zeros(B, D.ld, dtype=torch.float64, device=dev)
    Bpad[:, :d] = Bd.T
    return Bpad, B


def _outputs(B, N, rows, dev, with_trace):
    torch = device._torch()
    x = torch.zeros(B, N, dtype=torch.float64, device=dev)
    its = torch.zeros(B, dtype=torch.int32, device=dev)
    conv = torch.zeros(B, dtype=torch.int32, device=dev)
    stat = torch.zeros(B, dtype=torch.int32, device=dev)
    tr = torch.zeros(B, rows, 4, dtype=torch.float64, device=dev) if with_trace else None
    out = _lib.BatchOut()
    out.x, out.iterations, out.converged, out.status = (x.data_ptr(), its.data_ptr(), conv.data_ptr(),
                                                        stat.data_ptr())
    out.trace = tr.data_ptr() if tr is not None else None
    return out, (x, its, conv, stat, tr)


def _host(t):
    """Device tensor -> numpy.  Large results go through pinned host memory
    (torch's caching host allocator): a pageable 134 MB read-back of a B = 8192
    batch runs at ~2 GB/s (60 ms), the pinned one at the link rate (~6 ms)."""
    if t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    torch = device._torch()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _collect(bufs, t0, dev, trace_offset=0):
    torch = device._torch()
    x, its, conv, stat, tr = bufs
    torch.cuda.synchronize(dev)
    res = BatchResult(_host(x).T, its.cpu().numpy(), conv.cpu().numpy(), stat.cpu().numpy(),
                      time.perf_counter() - t0, _host(tr) if tr is not None else None)
    res._device_x = x          # B x N device copy (for on-device post-processing)
    return res


SMALL_B = 4     # below this, one persistent single-instance launch per column wins


def _empty(kind, A, Bmat, config):
    """The result of a batch with no instances (e.g. a rank's empty share)."""
    if hasattr(A, "device_extension"):
        D, _ = A.device_extension()
        N = D.n + D.d
    else:
        N = int(np.shape(A)[1]) if not hasattr(A, "n") else int(A.n)
    res = BatchResult(np.zeros((N, 0)), np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32),
                      0.0, None, kind, config.max_iter)
    if kind == "homotopy":
        res.lam = np.zeros(0)
        res.notes = np.zeros(0, np.int32)
    return res


def _status_of(exc):
    """Per-instance status code of a single-instance solver exception."""
    from paper_1007_3753_b200 import exceptions as ex
    for cls, code in ((ex.NumericalBreakdownError, _lib.BREAKDOWN), (ex.IllConditionedError, _lib.ILL_CONDITIONED),
                      (ex.NotPositiveDefiniteError, _lib.NOT_PD), (ex.DegenerateSupportError, _lib.DEGENERATE)):
        if isinstance(exc, cls):
            return code
    return None


def _ncols(Bmat):
    shape = getattr(Bmat, "shape", None)
    if shape is None:
        shape = np.shape(Bmat)
    return int(shape[1]) if len(shape) == 2 else None


def _small_batch(kind, A, Bmat, config, with_trace, target=None):
    """Batches of a few instances run as consecutive single-instance solves
    (each one persistent launch) — the batched round loop is launch-bound at
    tiny B.  Same semantics: element j is the single-instance call."""
    from paper_1007_3753_b200 import homotopy as hom
    from paper_1007_3753_b200.alm import dalm_solve
    from paper_1007_3753_b200.model import ProblemInstance
    from paper_1007_3753_b200.shrinkage import fista_solve
    t0 = time.perf_counter()
    if hasattr(Bmat, "detach"):
        Bmat = Bmat.detach().cpu().numpy()
    Bmat = np.asarray(Bmat, dtype=np.float64)
    B = Bmat.shape[1]
    D, view, N = _dict_view(A, config)
    xs, its, conv, stat, lams, notes, traces = [], [], [], [], [], [], []
    for j in range(B):
        P = ProblemInstance.__new__(ProblemInstance)
        P.A, P.b, P.ground_truth, P.noise_sigma = A if hasattr(A, "device_extension") else D, \
            np.ascontiguousarray(Bmat[:, j]), None, None
        try:
            if kind == "fista":
                r = fista_solve(P, config)
            elif kind == "dalm":
                r = dalm_solve(P, config)
            else:
                r, lam = hom.solve_path(P.A, P.b, target, config)
                lams.append(lam)
        except Exception as exc:  # noqa: BLE001 - numerical failures become per-instance status
            code = _status_of(exc)
            if code is None:
                raise
            # same as the batched path: status recorded, raised by BatchResult.result(j)
            xs.append(np.zeros(N))
            its.append(0)
            conv.append(0)
            stat.append(code)
            notes.append(0)
            traces.append(np.zeros((0, 4)))
            if kind == "homotopy":
                lams.append(float("nan"))
            continue
        xs.append(r.x_star)
        its.append(r.iterations)
        conv.append(int(r.converged))
        zero = len(r.trace) and r.iterations == 0 and r.converged
        stat.append(_lib.ZERO_DATA if zero else _lib.OK)
        notes.append(1 if r.notes and "ridge-regularized gram" in r.notes else 0)
        traces.append(np.array([tuple(t) for t in r.trace], dtype=np.float64).reshape(-1, 4))
    tr = None
    if with_trace:
        rows = max(int(config.max_iter), 1) + (1 if kind == "dalm" else 0)
        tr = np.zeros((B, rows, 4))
        for j, t in enumerate(traces):
            tr[j, : t.shape[0]] = t[:rows]
    res = BatchResult(np.stack(xs, axis=1), np.array(its, np.int32), np.array(conv, np.int32),
                      np.array(stat, np.int32), time.perf_counter() - t0, tr, kind, config.max_iter)
    if kind == "homotopy":
        res.lam = np.array(lams)
        res.notes = np.array(notes, np.int32)
    return res


def src_classify(A, class_labels, Bmat, config):
    """Cross-and-bouquet SRC (BASELINE config 3): solve every query on
    [A, I/e_weight] with the batched dual ALM (robust.cab_solve semantics,
    robust.py:181-220), then label_j = argmin_c ||b_j - e_j - A_c x_{j,c}||.
    class_labels: class id of each column of A (columns of a class contiguous).
    Returns (labels, class_residuals (B x C), BatchResult)."""
    torch = device._torch()
    from paper_1007_3753_b200.robust import ExtendedDictionary
    e_weight = float(config.opt("e_weight", 1.0))
    if not e_weight > 0:
        raise ValueError("e_weight must be positive")
    ext = A if hasattr(A, "device_extension") else ExtendedDictionary(
        A, 1.0 / e_weight, dtype=config.opt("dtype", "float64"), device_ordinal=config.opt("device", None))
    res = dalm_solve_batch(ext, Bmat, config)
    lab = np.asarray(class_labels)
    if res.x.shape[1] == 0:
        return np.zeros(0, np.int32), np.zeros((0, int(lab.max()) + 1)), res
    D, s = ext.device_extension()
    view = D.view(ext=True, scale=s)
    lab = np.asarray(class_labels)
    if np.any(np.diff(lab) < 0):
        raise ValueError("columns of a class must be contiguous (sorted class labels)")
    ncls = int(lab.max()) + 1
    offs = np.searchsorted(lab, np.arange(ncls + 1)).astype(np.int32)
    dev = D.device
    offd = torch.from_numpy(offs).to(dev)
    Bpad, B = _upload_rhs(Bmat, D)
    W = res._device_x.contiguous()                       # B x (n + d)
    labels = torch.zeros(B, dtype=torch.int32, device=dev)
    resid = torch.zeros(B, ncls, dtype=torch.float64, device=dev)
    rc = _lib.lib().ell1_src_classify(byref(view), device.ptr(Bpad), B, device.ptr(W), int(W.shape[1]),
                                      device.ptr(offd), ncls, device.ptr(labels), device.ptr(resid),
                                      device.stream_ptr(dev))
    _lib.check(rc, "ell1_src_classify")
    torch.cuda.synchronize(dev)
    return labels.cpu().numpy(), resid.cpu().numpy(), res


def dalm_solve_batch(A, Bmat, config, with_trace=False):
    """Dual ALM for every column of Bmat (d x B) against the shared A (or a
    robust.ExtendedDictionary for CAB batches).  Element j equals
    alm.dalm_solve on (A, b_j); option beta as in the reference."""
    if config.opt("y_cg_step", False):
        raise NotImplementedError("y_cg_step is single-instance only")
    if _ncols(Bmat) == 0:
        return _empty("dalm", A, Bmat, config)
    if (_ncols(Bmat) or SMALL_B) < SMALL_B:
        return _small_batch("dalm", A, Bmat, config, with_trace)
    t0 = time.perf_counter()
    D, view, N = _dict_view(A, config)
    ext = bool(view.ext)
    beta = float(config.opt("beta", 1.0))
    if not beta > 0:
        raise ValueError("beta must be positive")
    if config.opt("y_cg_step", False):
        raise NotImplementedError("y_cg_step is single-instance only")
    MT, Gcm, _, Gfull = D.gram_factor(ext, view.ext_scale)
    from paper_1007_3753_b200.alm import _Y_REFINE_TOL, _Y_REFINE_TOL_F32
    O = _lib.DalmOpts()
    O.beta = beta
    O.y_tol = _Y_REFINE_TOL if D.dtype == _lib.F64 else _Y_REFINE_TOL_F32
    O.y_cg_step = 0
    O.M = MT.data_ptr()
    O.Ginv = Gcm.data_ptr()
    # float64 storage: the y-step certificate as G y (d^2 per instance) instead
    # of A (A^T y) (d n); float32 keeps the single 2B-column tensor-core GEMM,
    # which measured faster than two B-column ones at config 3
    O.G = Gfull.data_ptr() if D.dtype == _lib.F64 else None
    Bpad, B = _upload_rhs(Bmat, D)
    C, _ = _ctrl(config, B, N, D.device, None)
    L = _lib.lib()
    wsb = L.ell1_batch_dalm_workspace(byref(view), B)
    ws = device.alloc_bytes(wsb, D.device)
    out, bufs = _outputs(B, N, config.max_iter + 1, D.device, with_trace)
    rc = L.ell1_batch_dalm(byref(view), device.ptr(Bpad), B, byref(C), byref(O), byref(out),
                           device.ptr(ws), int(ws.numel()), device.stream_ptr(D.device))
    _lib.check(rc, "ell1_batch_dalm")
    res = _collect(bufs, t0, D.device)
    res.kind = "dalm"
    res.max_iter = config.max_iter
    return res


def fista_solve_batch(A, Bmat, config, with_trace=False):
    """FISTA for every column of Bmat (d x B) against the shared A.
    Returns a BatchResult; ``.results()`` gives per-instance SolverResults."""
    if _ncols(Bmat) == 0:
        return _empty("fista", A, Bmat, config)
    if (_ncols(Bmat) or SMALL_B) < SMALL_B:
        return _small_batch("fista", A, Bmat, config, with_trace)
    torch = device._torch()
    t0 = time.perf_counter()
    D, view, N = _dict_view(A, config)
    dev = D.device
    if isinstance(Bmat, torch.Tensor):
        Bd = Bmat.to(device=dev, dtype=torch.float64)
    else:
        Bd = torch.from_numpy(np.ascontiguousarray(Bmat, dtype=np.float64)).to(dev)
    d, B = int(Bd.shape[0]), int(Bd.shape[1])
    if d != D.d:
        raise ValueError("Bmat must have d rows")
    Bpad = torch.zeros(B, D.ld, dtype=torch.float64, device=dev)
    Bpad[:, :d] = Bd.T
    from paper_1007_3753_b200.shrinkage import _fista_opts
    O = _fista_opts(config, None)
    if O.exact_L:
        sn = A.norm_sq() if hasattr(A, "norm_sq") else D.norm_sq()
        O.L_exact = sn * (1.0 + 1e-9)
    C, _keep = _ctrl(config, B, N, dev, None)
    L = _lib.lib()
    wsb = L.ell1_batch_fista_workspace(byref(view), B)
    ws = device.alloc_bytes(wsb, dev)
    x = torch.zeros(B, N, dtype=torch.float64, device=dev)
    its = torch.zeros(B, dtype=torch.int32, device=dev)
    conv = torch.zeros(B, dtype=torch.int32, device=dev)
    stat = torch.zeros(B, dtype=torch.int32, device=dev)
    tr = torch.zeros(B, config.max_iter, 4, dtype=torch.float64, device=dev) if with_trace else None
    out = _lib.BatchOut()
    out.x, out.iterations, out.converged, out.status = (x.data_ptr(), its.data_ptr(), conv.data_ptr(),
                                                        stat.data_ptr())
    out.trace = tr.data_ptr() if tr is not None else None
    rc = L.ell1_batch_fista(byref(view), device.ptr(Bpad), B, byref(C), byref(O), byref(out),
                            device.ptr(ws), int(ws.numel()), device.stream_ptr(dev))
    _lib.check(rc, "ell1_batch_fista")
    torch.cuda.synchronize(dev)
    return BatchResult(_host(x).T, its.cpu().numpy(), conv.cpu().numpy(), stat.cpu().numpy(),
                       time.perf_counter() - t0, _host(tr) if tr is not None else None)


def homotopy_solve_batch(A, Bmat, target_lambda, config, with_trace=False):
    """LASSO path to target_lambda for every column of Bmat (d x B) against the
    shared dictionary A (BASELINE config 5, batched Homotopy).  Element j
    equals homotopy.homotopy_solve on (A, b_j) (homotopy.py:128-261): same
    breakpoints, trace (one entry per breakpoint), notes and lambda reached
    (``.lam``).  Plain dictionaries only (no [A, sI] extension)."""
    torch = device._torch()
    if target_lambda < 0:
        raise ValueError("target lambda must be nonnegative")
    if hasattr(A, "device_extension"):
        raise NotImplementedError("batched Homotopy runs on plain dictionaries")
    if _ncols(Bmat) == 0:
        return _empty("homotopy", A, Bmat, config)
    if (_ncols(Bmat) or SMALL_B) < SMALL_B:
        return _small_batch("homotopy", A, Bmat, config, with_trace, target=float(target_lambda))
    t0 = time.perf_counter()
    D, view, N = _dict_view(A, config)
    dev = D.device
    Bpad, B = _upload_rhs(Bmat, D)
    L = _lib.lib()
    wsb = L.ell1_batch_homotopy_workspace(byref(view), B)
    if wsb == 0:
        raise ValueError("unsupported dictionary for batched Homotopy")
    ws = device.alloc_bytes(wsb, dev)
    rows = max(int(config.max_iter), 1)
    out, bufs = _outputs(B, N, rows, dev, with_trace)
    lam = torch.zeros(B, dtype=torch.float64, device=dev)
    notes = torch.zeros(B, dtype=torch.int32, device=dev)
    rc = L.ell1_batch_homotopy(byref(view), device.ptr(Bpad), B, float(target_lambda), int(config.max_iter),
                               byref(out), device.ptr(lam), device.ptr(notes), device.ptr(ws),
                               int(ws.numel()), device.stream_ptr(dev))
    _lib.check(rc, "ell1_batch_homotopy")
    res = _collect(bufs, t0, dev)
    res.kind = "homotopy"
    res.max_iter = config.max_iter
    res.lam = lam.cpu().numpy()
    res.notes = notes.cpu().numpy()
    return res
