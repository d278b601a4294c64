"""Column-sharded FISTA for one huge instance over several GPUs (BASELINE config 4).

A = [A_0 | A_1 | ... | A_{G-1}] split by columns, one rank (process) per GPU,
x / gradient sharded the same way, the d-side vectors (b, residuals)
replicated.  Per iteration the only bulk exchange is ONE allreduce(sum) of the
d-length partial A_r x_r (NCCL over NVLink); the backtracking / stopping
scalars travel as an all_gather of 8 doubles per rank and are folded on the
host in rank order, so every rank takes identical control decisions.

The iteration is the reference FISTA (shrinkage.py:231-298, oracle/l1_oracle.py
``fista``) restated on shards:

    y      = x + m (x - x_prev)                        m = (t_prev - 1) / t
    r_y    = (1 + m) r_x - m r_xprev                   (linear combination, no pass)
    g_y    = (1 + m) g_x - m g_xprev
    repeat (shrinkage.py:199-213):
        x_n = soft(y - g_y / L, lam_k / L)             ell1_shard_prox   (local)
        A x_n = allreduce_r(A_r x_n,r)                 ell1_gemv + NCCL  (1 pass)
        r_n = A x_n - b, F_n, Q                        ell1_shard_resid  (replicated)
        accept if F_n <= Q + 1e-12 max(1, |Q|) else L *= eta
    g_n = A_r^T r_n                                    ell1_gemv_t       (local, 1 pass)
    KKT / support partials                             ell1_shard_kkt

so a non-backtracking iteration streams each shard twice.  The device work
is libell1b200.so (csrc/shard.cu); this module is the host control loop and
the collectives.  The same loop runs over any ``ops`` object with the
ShardOps interface, which is how the tests drive it with gloo on CPU.
"""

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200.exceptions import NumericalBreakdownError
from paper_1007_3753_b200.model import SolverResult, TraceEntry

_POWER_SEED = 218751   # numerics.py:224


def column_range(n, rank, world):
    """Balanced contiguous column split: rank r owns [c0, c1)."""
    base, extra = divmod(int(n), int(world))
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def _t_next(t):
    """shrinkage.py:184-196 (with the nextafter nudge)."""
    tn = 0.5 * (1.0 + math.sqrt(4.0 * t * t + 1.0))
    while tn * tn - tn > t * t:
        tn = float(np.nextafter(tn, 1.0))
    return tn


# ----------------------------------------------------------------------------
# the local shard of the dictionary
# ----------------------------------------------------------------------------

class ShardedDictionary:
    """This rank's column panel A[:, c0:c1] of a d x n dictionary.

    ``local`` is a DeviceDictionary holding the panel (column-major, ld rows).
    ``group`` is the torch.distributed process group the columns are spread
    over (None: the default group, or a single process when torch.distributed
    is not initialised)."""

    def __init__(self, local, c0, n_global, group=None):
        self.local = local
        self.d = int(local.d)
        self.c0 = int(c0)
        self.c1 = int(c0) + int(local.n)
        self.n = int(n_global)
        self.group = group

    @property
    def shape(self):
        return (self.d, self.n)

    @classmethod
    def from_dense(cls, A, rank=0, world=1, group=None, dtype="float64", device_ordinal=None):
        """Upload this rank's columns of a host matrix (tests / small cases)."""
        A = np.asarray(A)
        c0, c1 = column_range(A.shape[1], rank, world)
        local = device.DeviceDictionary(np.ascontiguousarray(A[:, c0:c1]), dtype=dtype,
                                        device=device_ordinal)
        return cls(local, c0, A.shape[1], group)


@dataclass
class ShardedInstance:
    """Problem handle of the sharded solve: A is a ShardedDictionary, b the
    full (replicated) right-hand side, ground_truth the full x0 or None."""

    A: object
    b: np.ndarray
    ground_truth: np.ndarray = None


# ----------------------------------------------------------------------------
# device ops (libell1b200.so + torch.distributed)
# ----------------------------------------------------------------------------

class DeviceShardOps:
    """ShardOps over libell1b200.so; collectives through torch.distributed
    (NCCL on GPUs).  Vectors are float64 torch tensors on the rank's GPU."""

    def __init__(self, shard):
        torch = device._torch()
        self.torch = torch
        self.L = _lib.lib()
        D = shard.local
        self.D = D
        self.view = D.view()
        self.dev = D.device
        self.stream = device.stream_ptr(self.dev)
        self.d, self.nl, self.ld = D.d, D.n, D.ld
        self.group = shard.group
        self.world, self.rank = _world(shard.group)
        self.gws_bytes = int(self.L.ell1_gemv_workspace(ctypes.byref(self.view)))
        self.gws = device.alloc_bytes(self.gws_bytes, self.dev)
        self.ews = device.alloc_bytes(296 * 8 * 8, self.dev)
        # [world x 8 prox partials | 8 replicated residual sums]
        self.scal = torch.zeros(self.world * 8 + 8, dtype=torch.float64, device=self.dev)
        self.kscal = torch.zeros(self.world * 8, dtype=torch.float64, device=self.dev)
        self.mine = torch.zeros(8, dtype=torch.float64, device=self.dev)

    # vectors
    def zeros_d(self):
        return self.torch.zeros(self.ld, dtype=self.torch.float64, device=self.dev)

    def zeros_n(self):
        return self.torch.zeros(max(self.nl, 1), dtype=self.torch.float64, device=self.dev)

    def from_host_d(self, v):
        return device.to_device_vec(v, self.ld, self.dev)

    def from_host_n(self, v):
        return device.to_device_vec(v, max(self.nl, 1), self.dev)

    def to_host_n(self, v):
        return v[: self.nl].cpu().numpy().copy()

    def to_host_d(self, v):
        return v[: self.d].cpu().numpy().copy()

    # kernels
    def gemv(self, x, out):
        _lib.check(self.L.ell1_gemv(ctypes.byref(self.view), device.ptr(x), device.ptr(out),
                                    device.ptr(self.gws), self.gws_bytes, self.stream), "ell1_gemv")

    def gemv_t(self, r, out):
        _lib.check(self.L.ell1_gemv_t(ctypes.byref(self.view), device.ptr(r), device.ptr(out),
                                      device.ptr(self.gws), self.gws_bytes, self.stream),
                   "ell1_gemv_t")

    def prox(self, x, xp, gx, gxp, xn, m, L, lam, gt):
        _lib.check(self.L.ell1_shard_prox(self.nl, device.ptr(x), device.ptr(xp), device.ptr(gx),
                                          device.ptr(gxp), device.ptr(xn), float(m), float(L),
                                          float(lam), device.ptr(gt), device.ptr(self.mine),
                                          device.ptr(self.ews), self.stream), "ell1_shard_prox")

    def resid(self, ax, b, rx, mn, rn):
        out = self.scal[self.world * 8:]
        _lib.check(self.L.ell1_shard_resid(self.d, device.ptr(ax), device.ptr(b), device.ptr(rx),
                                           float(mn), device.ptr(rn), device.ptr(out),
                                           device.ptr(self.ews), self.stream), "ell1_shard_resid")

    def kkt(self, x, g, lam, cut):
        _lib.check(self.L.ell1_shard_kkt(self.nl, device.ptr(x), device.ptr(g), float(lam),
                                         float(cut), device.ptr(self.mine), device.ptr(self.ews),
                                         self.stream), "ell1_shard_kkt")

    # collectives + read-back
    def allreduce_(self, v):
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=self.group)

    def _gather_mine(self, dst):
        if self.world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(dst, self.mine, group=self.group)
        else:
            dst.copy_(self.mine)

    def trial_scalars(self):
        """-> (prox partials (world x 8), residual sums (8,)) on the host."""
        self._gather_mine(self.scal[: self.world * 8])
        h = self.scal.cpu().numpy()
        return h[: self.world * 8].reshape(self.world, 8), h[self.world * 8:]

    def kkt_scalars(self):
        self._gather_mine(self.kscal)
        return self.kscal.cpu().numpy().reshape(self.world, 8)

    def gather_n(self, v, n_global):
        """Full-length x on every rank (result assembly)."""
        torch = self.torch
        if self.world == 1:
            return self.to_host_n(v)
        import torch.distributed as dist
        sizes = [column_range(n_global, r, self.world) for r in range(self.world)]
        cap = max(c1 - c0 for c0, c1 in sizes)
        buf = torch.zeros(cap, dtype=torch.float64, device=self.dev)
        buf[: self.nl] = v[: self.nl]
        out = torch.zeros(cap * self.world, dtype=torch.float64, device=self.dev)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        h = out.cpu().numpy().reshape(self.world, cap)
        return np.concatenate([h[r, : c1 - c0] for r, (c0, c1) in enumerate(sizes)])

    def sync(self):
        self.torch.cuda.synchronize(self.dev)


def _world(group):
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(group), dist.get_rank(group)
    except ImportError:
        pass
    return 1, 0


# ----------------------------------------------------------------------------
# host control loop (identical on every rank)
# ----------------------------------------------------------------------------

def _fold_prox(parts):
    """Rank-order fold of the per-rank prox partials
    {sum|xn|, g_y.dl, dl.dl, max|xn|, ||xn-x||^2, ||x||^2, ||xn-gt||^2}."""
    s = np.zeros(8)
    mx = -math.inf
    for r in range(parts.shape[0]):
        for k in (0, 1, 2, 4, 5, 6):
            s[k] = s[k] + parts[r, k]
        mx = max(mx, float(parts[r, 3]))
    s[3] = mx
    return s


def _fold_kkt(parts, lam):
    """model.py:160-173 from {max_on, max_off, any_on, any_off, count} partials."""
    max_on = max(float(p) for p in parts[:, 0])
    max_off = max(float(p) for p in parts[:, 1])
    any_on = bool(np.any(parts[:, 2] > 0))
    any_off = bool(np.any(parts[:, 3] > 0))
    count = int(round(float(np.sum(parts[:, 4]))))
    worst = 0.0
    if any_on:
        worst = max_on
    if any_off:
        worst = max(worst, max_off - lam, 0.0)
    return worst, count


def _stop_fires(kind, thr, hist, F, F_prev, dx2, xp2, gt2, gtn, kk):
    """model.py:176-224 on reduced quantities."""
    if kind is None:
        return False
    if kind == "relative-objective":
        return hist >= 2 and abs(F - F_prev) <= thr * abs(F_prev)
    if kind == "relative-estimate":
        return hist >= 2 and math.sqrt(dx2) <= thr * math.sqrt(xp2)
    if kind == "ground-truth-distance":
        return math.sqrt(gt2) <= thr * gtn
    return kk <= thr


def sharded_power_norm_sq(ops, tol=1e-6, max_iter=1000):
    """Largest eigenvalue of A^T A over the shards (numerics.py:227-261) for
    d <= n: v -> A (A^T v) with one allreduce per step; the d-length power
    vector is kept on the host so the start vector and redraws follow the
    reference generator exactly."""
    gen = np.random.default_rng(_POWER_SEED)
    d = ops.d
    v = gen.standard_normal(d)
    v /= np.linalg.norm(v)
    theta = 0.0
    g = ops.zeros_n()
    w_d = ops.zeros_d()
    for _ in range(max_iter):
        ops.gemv_t(ops.from_host_d(v), g)
        ops.gemv(g, w_d)
        ops.allreduce_(w_d)
        w = ops.to_host_d(w_d)
        theta = float(v @ w)
        if np.linalg.norm(w - theta * v) <= tol * max(theta, np.finfo(float).tiny):
            break
        nw = np.linalg.norm(w)
        if nw == 0.0:
            v = gen.standard_normal(d)
            v /= np.linalg.norm(v)
            continue
        v = w / nw
    return theta


class ShardedFista:
    """Host driver of the column-sharded FISTA.  ``ops`` implements the
    ShardOps interface (DeviceShardOps in production)."""

    def __init__(self, ops, b, n_global, config, gt_local=None, gt_norm=0.0):
        self.ops = ops
        self.config = config
        self.b_host = np.asarray(b, dtype=np.float64)
        self.n = int(n_global)
        o = ops
        self.b = o.from_host_d(self.b_host)
        self.gt = o.from_host_n(gt_local) if gt_local is not None else None
        self.gt_norm = float(gt_norm)
        self.passes = 0        # panel passes (A x or A^T r) of the last solve
        self.trials = 0
        self._reset()

    def _reset(self):
        o = self.ops
        # iterate buffers (swapped, never copied)
        self.x, self.xp, self.xn = o.zeros_n(), o.zeros_n(), o.zeros_n()
        self.gx, self.gxp, self.gn = o.zeros_n(), o.zeros_n(), o.zeros_n()
        self.rx, self.rn, self.ax = o.zeros_d(), o.zeros_d(), o.zeros_d()

    def _kkt(self, x, g, lam, cut):
        self.ops.kkt(x, g, lam, cut)
        return _fold_kkt(self.ops.kkt_scalars(), lam)

    def solve(self):
        cfg, o = self.config, self.ops
        t0 = time.perf_counter()
        stop = cfg.stopping
        kind = stop.kind if stop is not None else None
        thr = float(stop.threshold) if stop is not None else 0.0
        if kind == "ground-truth-distance" and self.gt is None:
            raise ValueError("ground-truth-distance rule needs a ground truth")
        eta = float(cfg.opt("eta", 1.5))
        L = float(cfg.opt("L0", 1.0))
        beta = float(cfg.opt("beta", 0.5))
        exact = bool(cfg.opt("exact_L", False))
        bn2 = float(self.b_host @ self.b_host)
        if self.passes:
            self._reset()
        self.passes = 0
        self.trials = 0
        # r_x = A 0 - b = -b ; g_x = A^T r_x = -A^T b ; c0 = max|A^T b|
        o.resid(self.ax, self.b, self.rx, 0.0, self.rx)          # ax == 0 -> rx = -b
        o.gemv_t(self.rx, self.gx)
        self.passes += 1
        o.kkt(self.x, self.gx, 0.0, 1.0)
        c0 = max(float(p) for p in o.kkt_scalars()[:, 1])
        lam_bar = float(cfg.lam) if cfg.lam is not None else 1e-2 * c0
        if c0 == 0.0:
            x = np.zeros(self.n)
            return SolverResult(x, 0, time.perf_counter() - t0, True,
                                [TraceEntry(0, 0.0, math.sqrt(bn2), 0)])
        if not lam_bar > 0:
            raise ValueError("lambda must be positive")
        if exact:
            L = sharded_power_norm_sq(o) * (1.0 + 1e-9)
        lam_k = max(0.9 * c0, lam_bar) if cfg.opt("continuation", True) else lam_bar
        tp = tc = 1.0
        trace = []
        hist = 0
        F_prev = 0.0
        f_y = 0.5 * bn2                 # r_y = r_x = -b at the first iteration
        done = False
        it = 0
        while it < cfg.max_iter:
            it += 1
            m = (tp - 1.0) / tc
            t_new = _t_next(tc)
            mn = (tc - 1.0) / t_new     # momentum of the NEXT iteration
            accepted = False
            for _ in range(1 if exact else 101):
                o.prox(self.x, self.xp, self.gx, self.gxp, self.xn, m, L, lam_k, self.gt)
                o.gemv(self.xn, self.ax)
                self.passes += 1
                self.trials += 1
                o.allreduce_(self.ax)
                o.resid(self.ax, self.b, self.rx, mn, self.rn)
                parts, rs = o.trial_scalars()
                s = _fold_prox(parts)
                l1 = s[0]
                Fn = 0.5 * float(rs[0]) + lam_k * l1
                if exact:
                    accepted = True
                    break
                Q = f_y + float(s[1]) + 0.5 * L * float(s[2]) + lam_k * l1
                if Fn <= Q + 1e-12 * max(1.0, abs(Q)):
                    accepted = True
                    break
                L *= eta
            if not accepted:
                raise NumericalBreakdownError("backtracking exceeded 100 growth steps")
            # rotate: x_prev <- x, x <- x_n ; r, g likewise
            self.xp, self.x, self.xn = self.x, self.xn, self.xp
            self.rx, self.rn = self.rn, self.rx
            self.gxp, self.gx, self.gn = self.gx, self.gn, self.gxp
            o.gemv_t(self.rx, self.gx)
            self.passes += 1
            tp, tc = tc, t_new
            f_next = 0.5 * float(rs[1])
            cut = 1e-10 * max(float(s[3]), 1.0)
            kk, count = self._kkt(self.x, self.gx, lam_k, cut)
            trace.append(TraceEntry(it, Fn, math.sqrt(float(rs[0])), count))
            hist = min(hist + 1, 2)
            fires = _stop_fires(kind, thr, hist, Fn, F_prev, float(s[4]), float(s[5]),
                                float(s[6]), self.gt_norm, kk)
            F_prev = Fn
            f_y = f_next
            if lam_k == lam_bar and kk <= cfg.tol * lam_bar:
                done = True
                break
            if fires:
                done = True
                break
            lam_k = max(beta * lam_k, lam_bar)
        self.L = L
        x = o.gather_n(self.x, self.n)
        return SolverResult(x, it, time.perf_counter() - t0, done, trace)


def sharded_fista_solve(P, config, ops=None):
    """FISTA (shrinkage.fista_solve contract, shrinkage.py:231-298) on a
    column-sharded dictionary.  Call collectively on every rank of
    ``P.A.group``; every rank returns the same SolverResult with the full x.
    Options: L0, eta, beta, continuation, exact_L (d <= n)."""
    shard = P.A
    if not all(hasattr(shard, a) for a in ("c0", "c1", "d", "n")):
        raise TypeError("sharded_fista_solve needs a ShardedDictionary")
    if ops is None:
        ops = DeviceShardOps(shard)
    if config.opt("exact_L", False) and shard.d > shard.n:
        raise ValueError("exact_L on a sharded dictionary needs d <= n")
    gt_local, gtn = None, 0.0
    stop = config.stopping
    if stop is not None and stop.kind == "ground-truth-distance":
        gt = getattr(P, "ground_truth", None)
        if gt is None:
            raise ValueError("ground-truth-distance rule needs a ground truth")
        gt = np.asarray(gt, dtype=np.float64)
        gtn = float(np.linalg.norm(gt))
        if gtn == 0.0:
            raise ValueError("ground truth must be nonzero")
        gt_local = gt[shard.c0: shard.c1]
    drv = ShardedFista(ops, P.b, shard.n, config, gt_local, gtn)
    return drv.solve()
