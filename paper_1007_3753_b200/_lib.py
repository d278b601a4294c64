"""ctypes binding of libell1b200.so (the C ABI declared in include/ell1_b200.h).

There is deliberately no fallback: if the library or a CUDA device is
missing, every solver call raises DeviceError.
"""

import ctypes
import os
import threading

from paper_1007_3753_b200.exceptions import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ELL1_LIB_PATH") or os.path.join(_HERE, "libell1b200.so")   # override: diagnostics

OK, ZERO_DATA, LAMBDA_NONPOS, BREAKDOWN, ILL_CONDITIONED, NOT_PD, DEGENERATE, RUNNING = range(8)
ERR_ARG, ERR_CUDA, ERR_TIMEOUT, ERR_NOCOOP = -1, -2, -3, -4
F64, F32 = 0, 1
STOP_CODES = {None: 0, "relative-objective": 1, "relative-estimate": 2,
              "ground-truth-distance": 3, "kkt-residual": 4}

_ERRTEXT = {ERR_ARG: "bad argument", ERR_CUDA: "CUDA runtime error",
            ERR_TIMEOUT: "grid barrier timed out", ERR_NOCOOP: "persistent grid does not fit the device"}


class Dict(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("ext", ctypes.c_int32),
                ("d", ctypes.c_int64), ("n", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("ext_scale", ctypes.c_double)]


class State(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("phase", ctypes.c_int32),
                ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("hist", ctypes.c_int32), ("ntrace", ctypes.c_int32),
                ("rot", ctypes.c_int32 * 10), ("scal", ctypes.c_double * 24)]


class Ctrl(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_iter", ctypes.c_int32), ("stop_kind", ctypes.c_int32),
                ("stop_thr", ctypes.c_double), ("ground_truth", ctypes.c_void_p),
                ("gt_norm", ctypes.c_double)]


class FistaOpts(ctypes.Structure):
    _fields_ = [("L0", ctypes.c_double), ("eta", ctypes.c_double), ("beta", ctypes.c_double),
                ("continuation", ctypes.c_int32), ("exact_L", ctypes.c_int32),
                ("L_exact", ctypes.c_double), ("x0", ctypes.c_void_p),
                ("probe", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class ShardCtl(ctypes.Structure):
    """ell1_shard_ctl_t: device-side control of the column-sharded FISTA."""
    _fields_ = ([(f, ctypes.c_double) for f in ("lam_bar", "tol", "stop_thr", "gt_norm", "eta", "beta")]
                + [("max_iter", ctypes.c_int64)]
                + [(f, ctypes.c_int32) for f in ("stop_kind", "exact", "world", "rank")]
                + [(f, ctypes.c_double) for f in ("L", "lam_k", "lam_used", "tp", "tc", "m", "mn", "f_y",
                                                   "F_prev", "cut")]
                + [(f, ctypes.c_int64) for f in ("it", "passes", "trials")]
                + [(f, ctypes.c_int32) for f in ("hist", "growths", "state", "converged", "status",
                                                  "run_trial", "adv", "pending")])


SF_RUNNING, SF_FINAL, SF_FINISHED = 0, 1, 2


class SfBufs(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("x", "xp", "xn", "g", "gp", "gn", "r", "rn", "gt", "b",
                                               "xchg", "trace")]


class DalmOpts(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_double), ("y_tol", ctypes.c_double),
                ("y_cg_step", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("M", ctypes.c_void_p), ("Ginv", ctypes.c_void_p), ("y_out", ctypes.c_void_p),
                ("z_out", ctypes.c_void_p), ("G", ctypes.c_void_p)]


class PalmOpts(ctypes.Structure):
    _fields_ = [("mu0", ctypes.c_double), ("rho", ctypes.c_double), ("tau", ctypes.c_double),
                ("y_out", ctypes.c_void_p)]


class HomOut(ctypes.Structure):
    _fields_ = [("c", ctypes.c_void_p), ("lam_path", ctypes.c_void_p), ("support", ctypes.c_void_p),
                ("factor", ctypes.c_void_p)]


class BatchOut(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("iterations", ctypes.c_void_p),
                ("converged", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("trace", ctypes.c_void_p)]


class IO(ctypes.Structure):
    _fields_ = [("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("state", ctypes.c_void_p), ("trace", ctypes.c_void_p),
                ("x", ctypes.c_void_p), ("x_prev", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("max_steps", ctypes.c_int32), ("blocks", ctypes.c_int32),
                ("phase_ns", ctypes.c_void_p)]


class Group(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int32), ("team", ctypes.c_int32),
                ("dicts", ctypes.c_void_p), ("b", ctypes.c_void_p), ("ctrl", ctypes.c_void_p),
                ("io", ctypes.c_void_p), ("args_ws", ctypes.c_void_p), ("args_ws_bytes", ctypes.c_size_t)]


SOLVER_CORR, SOLVER_FISTA, SOLVER_IST, SOLVER_PALM, SOLVER_DALM, SOLVER_GPSR, SOLVER_TNIPM, \
    SOLVER_HOMOTOPY, SOLVER_POWER = range(9)
GROUP_ARG_BYTES = 1024

assert ctypes.sizeof(State) == 256, ctypes.sizeof(State)

_lock = threading.Lock()
_lib = None
_load_error = None

class Align(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int32), ("d", ctypes.c_int32), ("m", ctypes.c_int32),
                ("max_iter", ctypes.c_int32), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
                ("b_stride", ctypes.c_int64), ("rhs", ctypes.c_void_p), ("ld_rhs", ctypes.c_int64),
                ("tol", ctypes.c_double), ("mu0", ctypes.c_double), ("rho", ctypes.c_double),
                ("lam", ctypes.c_double), ("v0", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("e", ctypes.c_void_p), ("status", ctypes.c_void_p), ("iterations", ctypes.c_void_p),
                ("Bstage", ctypes.c_void_p)]


P = ctypes.POINTER
_SIGS = {
    "ell1_dict_build": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_correlation_max": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_size_t, ctypes.c_void_p]),
    "ell1_correlation_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_spectral_norm_sq": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                             ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_size_t, ctypes.c_void_p]),
    "ell1_power_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_soft_threshold": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                           ctypes.c_int64, ctypes.c_void_p]),
    "ell1_project_box_linf": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_void_p]),
    "ell1_chol_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_chol_downdate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_chol_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "ell1_chol_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p]),
    "ell1_chol_append": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_column_norms_sq": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_gram_dd_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_gram_dd": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_void_p]),
    "ell1_pcg_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_pcg_dense": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int32,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.c_void_p]),
    "ell1_axpby": (ctypes.c_int, [ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_sumsq": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_fista_workspace": (ctypes.c_size_t, [P(Dict), P(Ctrl), ctypes.c_int32]),
    "ell1_fista": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), P(FistaOpts), P(IO),
                                  ctypes.c_void_p]),
    "ell1_dalm_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_dalm": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), P(DalmOpts), P(IO),
                                 ctypes.c_void_p]),
    "ell1_palm_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_palm": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), P(PalmOpts), P(IO),
                                 ctypes.c_void_p]),
    "ell1_ist_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_ist": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), ctypes.c_void_p, ctypes.c_int32,
                                P(IO), ctypes.c_void_p]),
    "ell1_gpsr_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_gpsr": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), ctypes.c_double, ctypes.c_void_p,
                                 P(IO), ctypes.c_void_p]),
    "ell1_tnipm_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_tnipm": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(Ctrl), ctypes.c_double, ctypes.c_double,
                                  ctypes.c_int32, ctypes.c_void_p, P(IO), ctypes.c_void_p]),
    "ell1_homotopy_capacity": (ctypes.c_int, [P(Dict)]),
    "ell1_homotopy_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_homotopy": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_double, ctypes.c_int32,
                                     P(HomOut), P(IO), ctypes.c_void_p]),
    "ell1_batch_fista_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_batch_fista": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_int32, P(Ctrl),
                                        P(FistaOpts), P(BatchOut), ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p]),
    "ell1_batch_dalm_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_batch_dalm": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_int32, P(Ctrl),
                                       P(DalmOpts), P(BatchOut), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "ell1_batch_homotopy_capacity": (ctypes.c_int, [P(Dict)]),
    "ell1_batch_homotopy_workspace": (ctypes.c_size_t, [P(Dict), ctypes.c_int32]),
    "ell1_batch_homotopy": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                           ctypes.c_int32, P(BatchOut), ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "ell1_src_classify": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_gemv_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_gemv": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_size_t, ctypes.c_void_p]),
    "ell1_gemv_t": (ctypes.c_int, [P(Dict), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_size_t, ctypes.c_void_p]),
    "ell1_sfista_workspace": (ctypes.c_size_t, [P(Dict)]),
    "ell1_sfista_pre": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(SfBufs), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "ell1_sfista_post": (ctypes.c_int, [P(Dict), ctypes.c_void_p, P(SfBufs), ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p]),
    "ell1_shard_kkt": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_shard_resid": (ctypes.c_int, [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_double] +
                         [ctypes.c_void_p] * 4),
    "ell1_hom_absmax": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_hom_gammas": (ctypes.c_int, [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_double] +
                        [ctypes.c_void_p] * 2),
    "ell1_hom_gamma_minus": (ctypes.c_int, [ctypes.c_int64] + [ctypes.c_void_p] * 5),
    "ell1_hom_xstats": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_chol_factor_dense": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                              ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_chol_solve_dense": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_chol_solve_dense_multi": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                                   ctypes.c_void_p]),
    "ell1_pd_workspace": (ctypes.c_size_t, []),
    "ell1_pd_split": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32] + [ctypes.c_void_p] * 5),
    "ell1_pd_resid": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32] + [ctypes.c_void_p] * 12),
    "ell1_pd_prep": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32] + [ctypes.c_void_p] * 3 + [ctypes.c_double]
                     + [ctypes.c_void_p] * 5),
    "ell1_pd_direction": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64] + [ctypes.c_void_p] * 12),
    "ell1_pd_mu": (ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_pd_update": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_pd_diag": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_group_args_bytes": (ctypes.c_size_t, [ctypes.c_int32]),
    "ell1_group_team": (ctypes.c_int32, [ctypes.c_int32, P(Dict)]),
    "ell1_group_workspace": (ctypes.c_size_t, [ctypes.c_int32, P(Dict), ctypes.c_int32]),
    "ell1_correlation_max_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_spectral_norm_sq_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                                   ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_fista_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_ist_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_palm_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_dalm_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_gpsr_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_void_p]),
    "ell1_tnipm_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_double, ctypes.c_int32,
                                        ctypes.c_void_p]),
    "ell1_homotopy_group": (ctypes.c_int, [P(Group), ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "ell1_align_ist_step": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64] +
                            [ctypes.c_void_p] * 3 + [ctypes.c_double] * 2 + [ctypes.c_void_p] * 3),
    "ell1_align_stage_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 4),
    "ell1_test_align_large_rows": (None, [ctypes.c_int32]),
    "ell1_align_palm_batch": (ctypes.c_int, [P(Align), ctypes.c_void_p]),
    "ell1_align_ist_batch": (ctypes.c_int, [P(Align), ctypes.c_void_p]),
    "ell1_align_homotopy_batch": (ctypes.c_int, [P(Align), ctypes.c_void_p]),
    "ell1_align_gp_batch": (ctypes.c_int, [P(Align), ctypes.c_void_p]),
    "ell1_gemm_f32_workspace": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64]),
    "ell1_gemm_f32": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_void_p]),
    "ell1_gemm_f64": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "ell1_gemm_f64_variant": (ctypes.c_int, [ctypes.c_int32] * 4 + [ctypes.c_int64] * 3 +
                              [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "ell1_device_sms": (ctypes.c_int, [ctypes.c_int32]),
    "ell1_version": (ctypes.c_char_p, []),
}

# every symbol include/ell1_b200.h declares (checked by tests/test_abi.py)
EXPORTS = tuple(_SIGS)


def _load():
    global _lib, _load_error
    with _lock:
        if _lib is not None or _load_error is not None:
            return _lib
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            _load_error = "cannot load %s: %s (run `python -m paper_1007_3753_b200.build`)" % (
                LIB_PATH, exc)
            return None
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return _lib


def available():
    return _load() is not None


def lib():
    """The loaded library; raises DeviceError (no fallback) when missing."""
    L = _load()
    if L is None:
        raise DeviceError(_load_error)
    return L


def check(rc, what):
    if rc < 0:
        raise DeviceError("%s failed: %s (status %d)" % (what, _ERRTEXT.get(rc, "error"), rc))
    return rc
