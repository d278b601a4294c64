"""Column-sharded FISTA for one huge instance over several GPUs (BASELINE config 4).

A = [A_0 | A_1 | ... | A_{G-1}] split by columns, one rank (process) per GPU,
x / gradient sharded the same way, the d-side vectors (b, residuals)
replicated.  The iteration is the reference FISTA (shrinkage.py:231-298,
oracle/l1_oracle.py ``fista``) restated on shards:

    y      = x + m (x - x_prev)                        m = (t_prev - 1) / t
    g_y    = (1 + m) g_x - m g_xprev                   (linear combination, no pass)
    repeat (shrinkage.py:199-213):                     one ROUND per trial
        x_n = soft(y - g_y / L, lam_k / L)             local
        A x_n = allreduce_r(A_r x_n,r)                 1 pass + THE collective
        r_n = A x_n - b, F_n, Q                        replicated
        accept if F_n <= Q + 1e-12 max(1, |Q|) else L *= eta
    g_n = A_r^T r_n                                    local, 1 pass
    KKT / support partials                             ride on the next round's allreduce

Control lives on the device (csrc/shard.cu ``ell1_sfista_pre`` /
``ell1_sfista_post``): the d-length partial A_r x_n and every rank's scalar
partials (8 prox sums + 8 KKT partials, one 16-double slot per rank, the
other ranks' slots zero) travel in ONE allreduce(sum) per round, so each
rank folds the slots in rank order and takes bit-identical decisions without
any host round trip.  The host only enqueues rounds and polls the device
state word every ``ROUNDS_PER_POLL`` rounds (asynchronously, one batch
behind, so the GPU queue never drains).  The trace row's support count and
the KKT exit test of iteration k are finalised in round k+1 (their partials
need the global max|x| first); a solve therefore ends with one extra round.

The driver runs over any ``ops`` object with this interface
(``setup / begin / round / poll_async / poll_wait / result`` plus the
``gemv / gemv_t / allreduce_`` primitives of the exact-L power iteration);
``DeviceShardOps`` is the product, tests/shard_numpy_ops.py restates it in
numpy for the gloo (CPU) tests.
"""

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from paper_1007_3753_b200 import _lib, device
from paper_1007_3753_b200.exceptions import DeviceError, NumericalBreakdownError
from paper_1007_3753_b200.model import SolverResult, TraceEntry

_POWER_SEED = 218751   # numerics.py:224
SLOT = 16              # doubles per rank in the exchange buffer


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
# collectives
# ----------------------------------------------------------------------------

class TorchCollective:
    """torch.distributed (NCCL on GPUs) over ``group``; a no-op at world 1."""

    def __init__(self, group=None):
        self.group = group
        self.world, self.rank = _world(group)

    def allreduce_(self, t):
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def all_gather(self, t):
        """-> tensor of world * len(t) (rank-major)."""
        if self.world == 1:
            return t.clone()
        import torch
        import torch.distributed as dist
        out = torch.empty(t.numel() * self.world, dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out


class SoloCollective:
    """One process, whatever torch.distributed says: a single-GPU solve of
    the whole dictionary (shrinkage.fista_solve's streaming route)."""
    world, rank = 1, 0

    def allreduce_(self, t):
        pass

    def all_gather(self, t):
        return t.clone()


def _world(group):
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(group), dist.get_rank(group)
    except ImportError:
        pass
    return 1, 0


# ----------------------------------------------------------------------------
# device ops (libell1b200.so + one collective per round)
# ----------------------------------------------------------------------------

class DeviceShardOps:
    """The rank's device state of a column-sharded FISTA solve.  Vectors are
    float64 torch tensors on the rank's GPU; the control block
    (ell1_shard_ctl_t) lives in device memory."""

    def __init__(self, shard, coll=None):
        torch = device._torch()
        self.torch = torch
        self.L = _lib.lib()
        D = shard.local
        self.D = D
        self.view = D.view()
        self.dev = D.device
        self.stream = device.stream_ptr(self.dev)
        self.d, self.nl, self.ld = D.d, D.n, D.ld
        self.n_global = shard.n
        self.coll = coll if coll is not None else TorchCollective(shard.group)
        self.world, self.rank = self.coll.world, self.coll.rank
        c0, c1 = column_range(shard.n, self.rank, self.world)
        if (shard.c0, shard.c1) != (c0, c1):
            raise ValueError("shard columns [%d, %d) differ from column_range(n, %d, %d) = [%d, %d)"
                             % (shard.c0, shard.c1, self.rank, self.world, c0, c1))
        self.gws_bytes = int(self.L.ell1_gemv_workspace(ctypes.byref(self.view)))
        self.ws_bytes = int(self.L.ell1_sfista_workspace(ctypes.byref(self.view)))
        self.ws = torch.zeros(self.ws_bytes, dtype=torch.uint8, device=self.dev)  # tickets start at 0
        self.ews = device.alloc_bytes(296 * 8 * 8, self.dev)
        f64 = dict(dtype=torch.float64, device=self.dev)
        nl = max(self.nl, 1)
        self.vec = torch.zeros(6 * nl, **f64)          # x, xp, xn, g, gp, gn
        self.x, self.xp, self.xn, self.g, self.gp, self.gn = self.vec.split(nl)
        self.dvec = torch.zeros(2 * self.ld, **f64)    # r, rn
        self.r, self.rn = self.dvec.split(self.ld)
        self.xchg = torch.zeros(self.ld + SLOT * self.world, **f64)
        self.out8 = torch.zeros(8, **f64)
        self.ctl = torch.zeros(ctypes.sizeof(_lib.ShardCtl), dtype=torch.uint8, device=self.dev)
        self._state_word = _lib.ShardCtl.state.offset // 4
        self._pin = torch.zeros(2, dtype=torch.int32).pin_memory()
        self._polls = 0
        self.b = None
        self.gt = None
        self.trace = None
        self.bufs = None
        self.timing = None      # list -> per-round events (pre | collective | post), bench only

    # -- primitives (set-up, power iteration) --------------------------------
    def zeros_d(self):
        return self.torch.zeros(self.ld, dtype=self.torch.float64, device=self.dev)

    def zeros_n(self):
        return self.torch.zeros(max(self.nl, 1), dtype=self.torch.float64, device=self.dev)

    def from_host_d(self, v):
        return device.to_device_vec(v, self.ld, self.dev)

    def to_host_d(self, v):
        return v[: self.d].cpu().numpy().copy()

    def gemv(self, x, out):
        _lib.check(self.L.ell1_gemv(ctypes.byref(self.view), device.ptr(x), device.ptr(out),
                                    device.ptr(self.ws), self.gws_bytes, self.stream), "ell1_gemv")

    def gemv_t(self, r, out):
        _lib.check(self.L.ell1_gemv_t(ctypes.byref(self.view), device.ptr(r), device.ptr(out),
                                      device.ptr(self.ws), self.gws_bytes, self.stream), "ell1_gemv_t")

    def allreduce_(self, v):
        self.coll.allreduce_(v)

    # -- the solve --------------------------------------------------------------
    def setup(self, b, gt_local=None):
        """r = -b, g = A_r^T r, and the global max|A^T b| (one slot allreduce).
        ``b`` is a host vector or a device tensor of ld entries (resident).
        Returns c0."""
        self.vec.zero_()
        self.dvec.zero_()
        self.b = b if isinstance(b, self.torch.Tensor) else self.from_host_d(b)
        self.gt = device.to_device_vec(gt_local, max(self.nl, 1), self.dev) if gt_local is not None else None
        _lib.check(self.L.ell1_shard_resid(self.d, device.ptr(self.rn), device.ptr(self.b), device.ptr(self.r),
                                           0.0, device.ptr(self.r), device.ptr(self.out8),
                                           device.ptr(self.ews), self.stream), "ell1_shard_resid")
        self.gemv_t(self.r, self.g)
        _lib.check(self.L.ell1_shard_kkt(self.nl, device.ptr(self.x), device.ptr(self.g), 0.0, 1.0,
                                         device.ptr(self.out8), device.ptr(self.ews), self.stream),
                   "ell1_shard_kkt")
        slots = self.xchg[self.ld:].view(self.world, SLOT)
        slots.zero_()
        slots[self.rank, 8:] = self.out8
        self.coll.allreduce_(self.xchg[self.ld:])
        return float(slots[:, 9].max().item())

    def begin(self, ctl):
        """Upload the control block (an _lib.ShardCtl) and size the trace."""
        torch = self.torch
        ctl.world, ctl.rank = self.world, self.rank
        self.trace = torch.zeros(max(int(ctl.max_iter), 1) * 4, dtype=torch.float64, device=self.dev)
        raw = torch.frombuffer(bytearray(bytes(ctl)), dtype=torch.uint8)
        self.ctl.copy_(raw)
        B = _lib.SfBufs()
        for f in ("x", "xp", "xn", "g", "gp", "gn", "r", "rn", "b", "xchg", "trace"):
            setattr(B, f, getattr(self, f).data_ptr())
        B.gt = self.gt.data_ptr() if self.gt is not None else None
        self.bufs = B
        self._polls = 0

    def round(self):
        """One backtracking trial: pre (prox, A_r x_n) -> allreduce -> post."""
        V = ctypes.byref(self.bufs)
        cp = ctypes.c_void_p(self.ctl.data_ptr())
        ev = None
        if self.timing is not None:
            ev = [self.torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
        _lib.check(self.L.ell1_sfista_pre(ctypes.byref(self.view), cp, V, device.ptr(self.ws), self.ws_bytes,
                                          self.stream), "ell1_sfista_pre")
        if ev:
            ev[1].record()
        self.coll.allreduce_(self.xchg)
        if ev:
            ev[2].record()
        _lib.check(self.L.ell1_sfista_post(ctypes.byref(self.view), cp, V, device.ptr(self.ws), self.ws_bytes,
                                           self.stream), "ell1_sfista_post")
        if ev:
            ev[3].record()
            self.timing.append(ev)

    def poll_async(self):
        """Queue a read of ctl->state into pinned memory; returns a handle."""
        k = self._polls & 1
        self._polls += 1
        self._pin[k:k + 1].copy_(self.ctl.view(self.torch.int32)[self._state_word:self._state_word + 1],
                                 non_blocking=True)
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream(self.dev))
        return (k, ev)

    def poll_wait(self, h):
        k, ev = h
        ev.synchronize()
        return int(self._pin[k])

    def result(self):
        """-> (ShardCtl, trace rows (it x 4), full x) on every rank."""
        ctl = _lib.ShardCtl.from_buffer_copy(bytes(self.ctl.cpu().numpy().tobytes()))
        it = int(ctl.it)
        tr = self.trace[: 4 * it].cpu().numpy().reshape(-1, 4) if it else np.zeros((0, 4))
        sizes = [column_range(self.n_global, r, self.world) for r in range(self.world)]
        cap = max(c1 - c0 for c0, c1 in sizes)
        buf = self.torch.zeros(cap, dtype=self.torch.float64, device=self.dev)
        buf[: self.nl] = self.x[: self.nl]
        h = self.coll.all_gather(buf).cpu().numpy().reshape(self.world, cap)
        x = np.concatenate([h[r, : c1 - c0] for r, (c0, c1) in enumerate(sizes)])
        return ctl, tr, x

    def sync(self):
        self.torch.cuda.synchronize(self.dev)


# ----------------------------------------------------------------------------
# host driver (identical on every rank)
# ----------------------------------------------------------------------------

def sharded_power_norm_sq(ops, tol=1e-6, max_iter=1000):
    """Largest eigenvalue of A^T A over the shards (numerics.py:227-261) for
    d <= n: v -> A (A^T v) with one allreduce per step; the d-length power
    vector is kept on the host so the start vector and redraws follow the
    reference generator exactly (exact_L option only)."""
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
    """Host driver of the column-sharded FISTA: set-up, then rounds until the
    device reports FINISHED.  ``ops`` implements the ShardOps interface."""

    ROUNDS_PER_POLL = 8

    def __init__(self, ops, b, n_global, config, gt_local=None, gt_norm=0.0, b_device=None):
        self.ops = ops
        self.config = config
        self.b_host = np.asarray(b, dtype=np.float64)
        self.b_device = b_device     # optional resident copy of b (skips the H2D)
        self.span_events = None      # optional (start, end) CUDA events around the device work
        self.n = int(n_global)
        self.gt_local = gt_local
        self.gt_norm = float(gt_norm)
        self.passes = 0        # panel passes (A x or A^T r) of the last solve
        self.trials = 0
        self.rounds = 0

    def solve(self):
        cfg, o = self.config, self.ops
        t0 = time.perf_counter()
        stop = cfg.stopping
        kind = stop.kind if stop is not None else None
        if kind == "ground-truth-distance" and self.gt_local is None:
            raise ValueError("ground-truth-distance rule needs a ground truth")
        bn2 = float(self.b_host @ self.b_host)
        if self.span_events:
            self.span_events[0].record()
        c0 = o.setup(self.b_host if self.b_device is None else self.b_device, self.gt_local)
        lam_bar = float(cfg.lam) if cfg.lam is not None else 1e-2 * c0
        if c0 == 0.0:                                   # shrinkage.py:245-247
            self.passes, self.trials, self.rounds = 1, 0, 0
            return SolverResult(np.zeros(self.n), 0, time.perf_counter() - t0, True,
                                [TraceEntry(0, 0.0, math.sqrt(bn2), 0)])
        if not lam_bar > 0:
            raise ValueError("lambda must be positive")
        exact = bool(cfg.opt("exact_L", False))
        L = float(cfg.opt("L0", 1.0))
        if exact:
            L = sharded_power_norm_sq(o) * (1.0 + 1e-9)
        C = _lib.ShardCtl()
        C.lam_bar, C.tol = lam_bar, float(cfg.tol)
        C.stop_kind = _lib.STOP_CODES[kind]
        C.stop_thr = float(stop.threshold) if stop is not None else 0.0
        C.gt_norm = self.gt_norm
        C.eta, C.beta = float(cfg.opt("eta", 1.5)), float(cfg.opt("beta", 0.5))
        C.max_iter, C.exact = int(cfg.max_iter), int(exact)
        C.L = L
        C.lam_k = max(0.9 * c0, lam_bar) if cfg.opt("continuation", True) else lam_bar
        C.tp = C.tc = 1.0
        C.m, C.mn = 0.0, 0.0               # (t_prev - 1) / t and (t - 1) / t_next at t = 1
        C.f_y = 0.5 * bn2                  # r_y = r_x = -b at the first iteration
        C.state, C.run_trial = _lib.SF_RUNNING, 1
        o.begin(C)
        # every trial is one round; each iteration adds <= 101 trials, the
        # solve one finalising round, the poll lag one batch
        limit = (int(cfg.max_iter) + 1) * 102 + 4 * self.ROUNDS_PER_POLL
        rounds, prev = 0, None
        while True:
            for _ in range(self.ROUNDS_PER_POLL):
                o.round()
            rounds += self.ROUNDS_PER_POLL
            h = o.poll_async()
            if prev is not None and o.poll_wait(prev) == _lib.SF_FINISHED:
                break
            prev = h
            if rounds > limit:
                raise DeviceError("sharded FISTA did not finish within %d rounds" % limit)
        if self.span_events:
            self.span_events[1].record()
        ctl, tr, x = o.result()
        self.rounds = rounds
        self.passes = 1 + int(ctl.passes)
        self.trials = int(ctl.trials)
        if ctl.status == _lib.BREAKDOWN:
            raise NumericalBreakdownError("backtracking exceeded 100 growth steps")
        trace = [TraceEntry(int(r[0]), float(r[1]), float(r[2]), int(r[3])) for r in tr]
        return SolverResult(x, int(ctl.it), time.perf_counter() - t0, bool(ctl.converged), trace)


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


# ----------------------------------------------------------------------------
# BASELINE config 4 on the device
# ----------------------------------------------------------------------------

CFG4 = dict(d=65536, n=262144, k=2048, chunk=2048, dict_seed=7000003, x_seed=44, noise_rel=1e-3)


def make_cfg4_shard(rank=0, world=1, dev=None, coll=None, d=CFG4["d"], n=CFG4["n"], k=CFG4["k"],
                    dtype="float32"):
    """This rank's column panel of the config-4 instance, generated on the
    device: A = unit-norm N(0,1) columns drawn per 2048-column global chunk
    from a seeded Philox stream (the same matrix for every world size), x0 =
    k N(0,1) values on a uniform support (numpy PCG64), b = A x0 + 1e-3
    relative Gaussian noise (one allreduce of the partial A_r x0_r).
    Returns (ShardedDictionary, b (host, d), x0 (host, n), ops)."""
    torch = device._torch()
    dev = dev if dev is not None else device.current_device()
    c0, c1 = column_range(n, rank, world)
    nl = c1 - c0
    ld = (d + 31) // 32 * 32
    tdt = torch.float32 if dtype == "float32" else torch.float64
    storage = torch.zeros(nl, ld, dtype=tdt, device=dev)
    CH = CFG4["chunk"]
    g = torch.Generator(device=dev)
    for j0 in range(c0 // CH * CH, c1, CH):
        g.manual_seed(CFG4["dict_seed"] + j0 // CH)
        blk = torch.randn(CH, d, generator=g, device=dev, dtype=torch.float32)
        blk /= torch.linalg.vector_norm(blk, dim=1, keepdim=True)
        a, e = max(j0, c0), min(j0 + CH, c1)
        storage[a - c0:e - c0, :d] = blk[a - j0:e - j0]
        del blk
    torch.cuda.empty_cache()
    D = device.DeviceDictionary.wrap(storage, d)
    shard = ShardedDictionary(D, c0, n, None if coll is None else getattr(coll, "group", None))
    ops = DeviceShardOps(shard, coll)
    rng = np.random.default_rng(CFG4["x_seed"])
    x0 = np.zeros(n)
    x0[rng.choice(n, k, replace=False)] = rng.standard_normal(k)
    xl = device.to_device_vec(x0[c0:c1], max(nl, 1), dev)
    bd = ops.zeros_d()
    ops.gemv(xl, bd)
    ops.allreduce_(bd)
    b = ops.to_host_d(bd)
    sigma = CFG4["noise_rel"] * float(np.linalg.norm(b)) / np.sqrt(d)
    b = b + sigma * rng.standard_normal(d)
    return shard, b, x0, ops


def kkt_certificate(ops, x_local, b, lam):
    """Independent fp64 optimality certificate of a sharded solution:
    c = A^T (b - A x) by fresh GEMV / GEMV^T passes (fp64 accumulation) and
    model.kkt_from_correlation (model.py:160-173) folded over the ranks.
    Returns (kkt, objective)."""
    torch = ops.torch
    xl = device.to_device_vec(x_local, max(ops.nl, 1), ops.dev)
    ax = ops.zeros_d()
    ops.gemv(xl, ax)
    ops.allreduce_(ax)
    r = ops.from_host_d(b) - ax
    r[ops.d:] = 0.0
    c = ops.zeros_n()
    ops.gemv_t(r, c)
    x = xl[: ops.nl]
    c = c[: ops.nl]
    on = x != 0
    part = torch.zeros(4, dtype=torch.float64, device=ops.dev)
    if bool(on.any()):
        part[0] = (c[on] - lam * torch.sign(x[on])).abs().max()
    if bool((~on).any()):
        part[1] = (c[~on].abs() - lam).clamp_min(0.0).max()
    part[2] = x.abs().sum()
    part[3] = 0.0
    g = ops.coll.all_gather(part).view(-1, 4)
    kk = float(torch.maximum(g[:, 0].max(), g[:, 1].max()).item())
    rr = float((r[: ops.d] ** 2).sum().item())
    return kk, 0.5 * rr + lam * float(g[:, 2].sum().item())
