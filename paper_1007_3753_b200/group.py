"""Group solves: many independent l1 problems, each with its OWN dictionary,
in one persistent launch per solver.

The reference's experiment harness fans its trials out over processes, one
solve per trial (bench.py:_run_tasks :145-151).  On the B200 a trial is a
small problem (n in the hundreds), far too small to fill 148 SMs; a group
launch instead runs the single-solve kernel bodies on teams of CTAs — each
team sized so its trial's dictionary panel stays resident in shared memory —
and walks the teams over all trials of the group (csrc/solvers_common.cuh
group_kernel, C-ABI ``ell1_<solver>_group``).  Every trial computes exactly
what the single-solve entry point computes for it (same kernel body, same
team-independent reduction order per team size).

``TrialGroup`` uploads the trials once (dictionaries stacked per shape) and
offers the per-trial helpers the harness needs (correlation max, spectral
norm) plus ``solve(name, config, lams)``.  Wall time per trial is the group's
device time divided by the trial count.
"""

import ctypes
import time

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200._runner import raise_for
from paper_1007_3753_b200.model import SolverResult, TraceEntry

GROUP_SOLVERS = ("homotopy", "gpsr", "tnipm", "ist", "fista", "palm", "dalm")
_CODES = {"fista": _lib.SOLVER_FISTA, "ist": _lib.SOLVER_IST, "palm": _lib.SOLVER_PALM,
          "dalm": _lib.SOLVER_DALM, "gpsr": _lib.SOLVER_GPSR, "tnipm": _lib.SOLVER_TNIPM,
          "homotopy": _lib.SOLVER_HOMOTOPY, "corr": _lib.SOLVER_CORR, "power": _lib.SOLVER_POWER}
_MAX_GROUP = 4096            # trials per launch (bounds the trace / workspace memory)


def _pad32(d):
    return (int(d) + 31) // 32 * 32


class TrialGroup:
    """Device copies of a list of problems (A_i, b_i), i = 0..count-1.

    ``ext=True`` runs every solve on the cross-and-bouquet operator [A_i, s I]
    (s = ``ext_scale``), as robust.cab_solve does for one problem.
    ``dtype`` "float64" (default) or "float32" dictionary storage."""

    def __init__(self, problems, dtype="float64", ext=False, ext_scale=1.0, device_ordinal=None):
        torch = device._torch()
        _lib.lib()
        self.dev = device.current_device(device_ordinal)
        self.stream = device.stream_ptr(self.dev)
        self.count = len(problems)
        self.ext = bool(ext)
        self.ext_scale = float(ext_scale)
        self.dtype = {"float64": _lib.F64, "float32": _lib.F32}[str(dtype)]
        tdt = torch.float64 if self.dtype == _lib.F64 else torch.float32
        self.dicts = (_lib.Dict * max(self.count, 1))()
        self.shapes = []
        self._keep = []
        by_shape = {}
        for i, P in enumerate(problems):
            A = np.asarray(P.A, dtype=np.float64)
            if A.ndim != 2:
                raise ValueError("dictionary must be a matrix")
            by_shape.setdefault(A.shape, []).append(i)
            self.shapes.append(A.shape)
        for (d, n), idx in by_shape.items():
            ld = _pad32(d)
            host = np.stack([np.asarray(problems[i].A, dtype=np.float64) for i in idx])
            src = torch.from_numpy(host).to(self.dev)
            st = torch.zeros((len(idx), n, ld), dtype=tdt, device=self.dev)
            st[:, :, :d] = src.transpose(1, 2).to(tdt)       # column-major, ld rows (layout plumbing)
            self._keep.append(st)
            for j, i in enumerate(idx):
                v = self.dicts[i]
                v.A = st[j].data_ptr()
                v.dtype = self.dtype
                v.ext = 1 if self.ext else 0
                v.d, v.n, v.ld = d, n, ld
                v.ext_scale = self.ext_scale
        self.ldmax = max((_pad32(d) for d, _ in self.shapes), default=32)
        B = np.zeros((max(self.count, 1), self.ldmax))
        for i, P in enumerate(problems):
            b = np.asarray(P.b, dtype=np.float64)
            if b.shape != (self.shapes[i][0],):
                raise ValueError("b must have length d")
            B[i, : b.shape[0]] = b
        self.bnorm_zero = [not np.any(np.asarray(P.b)) for P in problems]
        self.B = torch.from_numpy(B).to(self.dev)
        self.bptr = (ctypes.c_void_p * max(self.count, 1))(
            *[self.B[i].data_ptr() for i in range(max(self.count, 1))])
        self.ncols = [n + (d if self.ext else 0) for d, n in self.shapes]

    # ------------------------------------------------------------------ plumbing
    def _team(self, code, idx):
        L = _lib.lib()
        return max(int(L.ell1_group_team(code, ctypes.byref(self.dicts[i]))) for i in idx)

    def _chunks(self):
        for s in range(0, self.count, _MAX_GROUP):
            yield list(range(s, min(self.count, s + _MAX_GROUP)))

    def _group(self, code, idx, ctrls, trace_rows, xwidth=None):
        """Workspaces, states, traces, outputs and the ell1_group_t of trials idx."""
        torch = device._torch()
        L = _lib.lib()
        G = len(idx)
        team = self._team(code, idx)
        sizes = [int(L.ell1_group_workspace(code, ctypes.byref(self.dicts[i]), team)) for i in idx]
        offs = np.concatenate([[0], np.cumsum([(s + 255) // 256 * 256 for s in sizes])]).astype(np.int64)
        ws = device.alloc_bytes(int(offs[-1]), self.dev)
        N = xwidth or max(self.ncols[i] for i in idx)
        rows = max(int(trace_rows), 1)
        st = torch.zeros((G, 32), dtype=torch.float64, device=self.dev)
        x = torch.zeros((G, N), dtype=torch.float64, device=self.dev)
        tr = torch.empty((G, rows * 4), dtype=torch.float64, device=self.dev)
        dicts = (_lib.Dict * G)(*[self.dicts[i] for i in idx])
        bp = (ctypes.c_void_p * G)(*[self.bptr[i] for i in idx])
        cs = (_lib.Ctrl * G)(*ctrls) if ctrls is not None else (_lib.Ctrl * G)()
        ios = (_lib.IO * G)()
        base = ws.data_ptr()
        for j in range(G):
            io = ios[j]
            io.workspace = base + int(offs[j])
            io.workspace_bytes = sizes[j]
            io.state = st[j].data_ptr()
            io.trace = tr[j].data_ptr()
            io.x = x[j].data_ptr()
            io.max_steps = 0
            io.blocks = team
        aws_b = int(L.ell1_group_args_bytes(G))
        aws = device.alloc_bytes(aws_b, self.dev)
        g = _lib.Group()
        g.count, g.team = G, team
        g.dicts = ctypes.cast(dicts, ctypes.c_void_p)
        g.b = ctypes.cast(bp, ctypes.c_void_p)
        g.ctrl = ctypes.cast(cs, ctypes.c_void_p)
        g.io = ctypes.cast(ios, ctypes.c_void_p)
        g.args_ws = aws.data_ptr()
        g.args_ws_bytes = aws_b
        keep = (ws, st, x, tr, dicts, bp, cs, ios, aws)
        return g, keep, st, x, tr, team

    # ------------------------------------------------------------------ helpers
    def correlation_max(self):
        """max |A_i^T b_i| per trial (model.py:126-129 / bench.py:130-131), on the device."""
        torch = device._torch()
        L = _lib.lib()
        out = np.zeros(self.count)
        for idx in self._chunks():
            g, keep, *_ = self._group(_lib.SOLVER_CORR, idx, None, 1)
            o = torch.zeros(2 * len(idx), dtype=torch.float64, device=self.dev)
            _lib.check(L.ell1_correlation_max_group(ctypes.byref(g), device.ptr(o), self.stream),
                       "ell1_correlation_max_group")
            out[idx] = o.view(-1, 2)[:, 0].cpu().numpy()
        return out

    def norm_sq(self, tol=1e-6, max_iter=1000):
        """spectral_norm_sq(A_i) per trial (numerics.py:224-261), on the device,
        with the reference's seeded start vector for each shape."""
        torch = device._torch()
        L = _lib.lib()
        out = np.zeros(self.count)
        starts = {}
        for d, n in set(self.shapes):
            dim = d if d <= n else n
            rng = np.random.default_rng(device._POWER_SEED)
            draws = []
            for _ in range(4):
                v = rng.standard_normal(dim)
                draws.append(v / np.linalg.norm(v))
            starts[(d, n)] = torch.from_numpy(np.concatenate(draws)).to(self.dev)
        for idx in self._chunks():
            g, keep, *_ = self._group(_lib.SOLVER_POWER, idx, None, 1)
            g.team = 1
            v0 = (ctypes.c_void_p * len(idx))(*[starts[self.shapes[i]].data_ptr() for i in idx])
            o = torch.zeros(2 * len(idx), dtype=torch.float64, device=self.dev)
            _lib.check(L.ell1_spectral_norm_sq_group(ctypes.byref(g), v0, 3, float(tol), int(max_iter),
                                                     device.ptr(o), self.stream),
                       "ell1_spectral_norm_sq_group")
            out[idx] = o.view(-1, 2)[:, 0].cpu().numpy()
        return out

    # ------------------------------------------------------------------ solve
    def solve(self, name, config, lams=None, want_trace=False):
        """Solve every trial with solver `name` (bench.py:solve_named :41-62
        semantics: lambda = lams[i] if given, else config.lam, else the
        default 1e-2 ||A_i^T b_i||_inf).  Returns a list of SolverResult."""
        if name == "gp":
            name = "gpsr"
        if name not in GROUP_SOLVERS:
            raise ValueError("solver %r has no group form (choose from %s)" % (name, ", ".join(GROUP_SOLVERS)))
        if config.stopping is not None and config.stopping.kind == "ground-truth-distance":
            raise ValueError("group solves do not take per-trial ground truths")
        t0 = time.perf_counter()
        lam = self._lambdas(name, config, lams)
        results = [None] * self.count
        for idx in self._chunks():
            self._solve_chunk(name, config, lam, idx, results, want_trace)
        per = (time.perf_counter() - t0) / max(self.count, 1)
        for r in results:
            r.wall_time_seconds = per
        return results

    def _lambdas(self, name, config, lams):
        if lams is not None:
            lam = np.asarray(lams, dtype=np.float64)
            if lam.shape != (self.count,):
                raise ValueError("lams must hold one value per trial")
            return lam
        if config.lam is not None:
            return np.full(self.count, float(config.lam))
        if name in ("fista", "palm", "dalm"):
            return None                          # resolved on the device / unused
        return 1e-2 * self.correlation_max()     # model.py:126-129

    def _ctrls(self, config, lam, idx):
        stop = config.stopping
        out = []
        for i in idx:
            c = _lib.Ctrl()
            c.lam = -1.0 if lam is None else float(lam[i])
            c.tol = float(config.tol)
            c.max_iter = int(config.max_iter)
            c.stop_kind = _lib.STOP_CODES[stop.kind if stop is not None else None]
            c.stop_thr = float(stop.threshold) if stop is not None else 0.0
            c.ground_truth = None
            c.gt_norm = 0.0
            out.append(c)
        return out

    def _solve_chunk(self, name, config, lam, idx, results, want_trace):
        torch = device._torch()
        L = _lib.lib()
        code = _CODES[name]
        G = len(idx)
        if lam is not None and name not in ("palm", "dalm"):
            for i in idx:
                if not lam[i] > 0 and not (name == "homotopy" and lam[i] >= 0):
                    raise ValueError("lambda must be positive")
        ctrls = self._ctrls(config, lam, idx)
        rows = config.max_iter + 2
        g, keep, st, x, tr, team = self._group(code, idx, ctrls, rows)
        extra = []
        notes_of = lambda s: ()
        messages = {}
        if name == "fista":
            O = (_lib.FistaOpts * G)()
            exact = bool(config.opt("exact_L", False))
            Lx = self.norm_sq()[idx] if exact else None
            for j in range(G):
                o = O[j]
                o.L0 = float(config.opt("L0", 1.0))
                o.eta = float(config.opt("eta", 1.5))
                o.beta = float(config.opt("beta", 0.5))
                o.continuation = 1 if config.opt("continuation", True) else 0
                o.exact_L = 1 if exact else 0
                o.L_exact = float(Lx[j]) * (1.0 + 1e-9) if exact else 0.0
            extra = [O]
            rc = L.ell1_fista_group(ctypes.byref(g), O, self.stream)
            messages = {_lib.BREAKDOWN: "backtracking exceeded 100 growth steps",
                        _lib.LAMBDA_NONPOS: "lambda must be positive"}
        elif name == "ist":
            from paper_1007_3753_b200.shrinkage import ContinuationSchedule
            c0 = self.correlation_max()[idx]
            stages = []
            for j, i in enumerate(idx):
                lt = float(lam[i])
                stages.append(np.asarray(ContinuationSchedule(max(0.9 * c0[j], lt), 0.5, lt).stages()))
            width = max(s.shape[0] for s in stages)
            S = np.zeros((G, width))
            for j, s in enumerate(stages):
                S[j, : s.shape[0]] = s
            Sd = torch.from_numpy(S).to(self.dev)
            sp = (ctypes.c_void_p * G)(*[Sd[j].data_ptr() for j in range(G)])
            ns = (ctypes.c_int32 * G)(*[s.shape[0] for s in stages])
            extra = [Sd, sp, ns]
            rc = L.ell1_ist_group(ctypes.byref(g), sp, ns, self.stream)
        elif name in ("gpsr", "tnipm"):
            la = (ctypes.c_double * G)(*[float(lam[i]) for i in idx])
            extra = [la]
            if name == "gpsr":
                from paper_1007_3753_b200.gradient_projection import _GPSR_NOTES
                rc = L.ell1_gpsr_group(ctypes.byref(g), la, self.stream)
                notes_of = lambda s: (_GPSR_NOTES[s.rot[2]],) if s.rot[2] in _GPSR_NOTES else ()
            else:
                cap = config.opt("pcg_max_iter", None)
                rc = L.ell1_tnipm_group(ctypes.byref(g), la, float(config.opt("pcg_tol", 1e-4)),
                                        int(cap) if cap is not None else 0, self.stream)
                notes_of = lambda s: ("pcg hit its iteration cap %d times" % s.rot[0],) if s.rot[0] else ()
                messages = {_lib.BREAKDOWN: "barrier line search exhausted without an interior decrease"}
        elif name == "palm":
            mu, rho = float(config.opt("mu0", 1.0)), float(config.opt("rho", 2.0))
            if not mu > 0 or not rho > 1:
                raise ValueError("mu0 must be positive and rho must exceed 1")
            ns = self.norm_sq()[idx]
            O = (_lib.PalmOpts * G)()
            for j, i in enumerate(idx):
                O[j].mu0, O[j].rho = mu, rho
                O[j].tau = 1.0 if self.bnorm_zero[i] else 1.01 * float(ns[j])     # alm.py:111-122
            extra = [O]
            rc = L.ell1_palm_group(ctypes.byref(g), O, self.stream)
            notes_of = lambda s: (("inner-iteration budget exhausted",)
                                  if not s.converged and s.iterations >= config.max_iter else ())
        elif name == "dalm":
            O, extra = self._dalm_opts(config, idx)
            rc = L.ell1_dalm_group(ctypes.byref(g), O, self.stream)
            notes_of = lambda s: (("iteration budget exhausted",)
                                  if not s.converged and s.iterations >= config.max_iter else ())
            messages = {_lib.ILL_CONDITIONED: "dual least-squares step failed its residual contract"}
        else:                                    # homotopy
            tl = (ctypes.c_double * G)(*[float(lam[i]) for i in idx])
            C = torch.zeros((G, max(self.ncols[i] for i in idx)), dtype=torch.float64, device=self.dev)
            O = (_lib.HomOut * G)()
            for j in range(G):
                O[j].c = C[j].data_ptr()
            extra = [tl, C, O]
            rc = L.ell1_homotopy_group(ctypes.byref(g), tl, int(config.max_iter), O, self.stream)
            notes_of = lambda s: ("ridge-regularized gram",) if s.rot[1] else ()
            messages = {_lib.NOT_PD: "active-set Gram is singular",
                        _lib.DEGENERATE: "active-set Gram is singular"}
        _lib.check(rc, "ell1_%s_group" % name)
        states = st.cpu().numpy()
        xs = x.cpu().numpy()
        for j, i in enumerate(idx):
            s = _lib.State.from_buffer_copy(states[j].tobytes())
            raise_for(s.status, messages)
            trace = []
            if want_trace and s.ntrace > 0:
                t = tr[j, : s.ntrace * 4].cpu().numpy().reshape(-1, 4)
                trace = [TraceEntry(int(r[0]), float(r[1]), float(r[2]), int(r[3])) for r in t]
            results[i] = SolverResult(xs[j, : self.ncols[i]].copy(), int(s.iterations), 0.0,
                                      bool(s.converged), trace, notes_of(s))
        del keep, extra

    def _dalm_opts(self, config, idx):
        """Per-trial row-Gram factors (alm.py:162-169) for the dual ALM, batched
        per shape (cuBLAS / cuSOLVER setup, like DeviceDictionary.gram_factor)."""
        torch = device._torch()
        from paper_1007_3753_b200.alm import _Y_REFINE_TOL, _Y_REFINE_TOL_F32
        from paper_1007_3753_b200.exceptions import IllConditionedError
        beta = float(config.opt("beta", 1.0))
        if not beta > 0:
            raise ValueError("beta must be positive")
        cg = 1 if config.opt("y_cg_step", False) else 0
        G = len(idx)
        O = (_lib.DalmOpts * G)()
        keep = []
        by_shape = {}
        for j, i in enumerate(idx):
            by_shape.setdefault(self.shapes[i], []).append((j, i))
        for (d, n), members in by_shape.items():
            ld = _pad32(d)
            tdt = torch.float64 if self.dtype == _lib.F64 else torch.float32
            At = torch.stack([self._column_major(i)[:, :d] for _, i in members]).to(torch.float64)   # (k, n, d)
            Gm = At.transpose(1, 2) @ At
            if self.ext:
                Gm.diagonal(dim1=1, dim2=2).add_(self.ext_scale ** 2)
            Lf, info = torch.linalg.cholesky_ex(Gm)
            bad = info.cpu().numpy()
            Ginv = torch.cholesky_inverse(Lf)
            Gcm = torch.zeros((len(members), d, ld), dtype=torch.float64, device=self.dev)
            Gcm[:, :, :d] = Ginv
            MT = torch.zeros((len(members), n, ld), dtype=tdt, device=self.dev)
            MT[:, :, :d] = (At @ Ginv).to(tdt)      # row j of M^T == column j of M = G^-1 A
            keep += [Gcm, MT]
            for q, (j, i) in enumerate(members):
                if bad[q] != 0 and not self.bnorm_zero[i]:
                    raise IllConditionedError("row Gram A A^T is not positive definite; the dual "
                                              "solver needs full row rank")
                o = O[j]
                o.beta = beta
                o.y_tol = _Y_REFINE_TOL if self.dtype == _lib.F64 else _Y_REFINE_TOL_F32
                o.y_cg_step = cg
                o.M = MT[q].data_ptr()
                o.Ginv = Gcm[q].data_ptr()
        return O, [O] + keep

    def _column_major(self, i):
        """(n, ld) view of trial i's dictionary storage."""
        torch = device._torch()
        v = self.dicts[i]
        for st in self._keep:
            base = st.data_ptr()
            per = st.shape[1] * st.shape[2] * st.element_size()
            if base <= v.A < base + per * st.shape[0]:
                return st[(v.A - base) // per]
        raise KeyError(i)


def solve_group(name, problems, config, lams=None, dtype="float64", want_trace=False):
    """Solve independent problems (each its own dictionary) with one group
    launch: the GPU form of running bench.solve_named over trials."""
    if not problems:
        return []
    return TrialGroup(problems, dtype=dtype).solve(name, config, lams=lams, want_trace=want_trace)
