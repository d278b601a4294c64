"""Host (numpy + gloo) restatement of the device rounds of the column-sharded
FISTA (csrc/shard.cu ell1_sfista_pre / ell1_sfista_post) — TEST
INFRASTRUCTURE ONLY.

It implements the ShardOps interface of paper_1007_3753_b200/sharded.py so
the CPU suite can drive the sharded solve at world size 1..3 over
torch.distributed/gloo with the product's one-allreduce-per-round protocol
(d-length partial + one 16-double slot per rank) and compare it with the
reference's golden outputs.  The product path (DeviceShardOps) never touches
this module.
"""

import math

import numpy as np

from oracle.l1_oracle import soft

SLOT = 16
RUNNING, FINAL, FINISHED = 0, 1, 2
STOP = {None: 0, "relative-objective": 1, "relative-estimate": 2, "ground-truth-distance": 3,
        "kkt-residual": 4}


def _t_next(t):
    tn = 0.5 * (1.0 + math.sqrt(4.0 * t * t + 1.0))
    while tn * tn - tn > t * t:
        tn = float(np.nextafter(tn, 1.0))
    return tn


def _stop_fires(kind, thr, hist, F, F_prev, dx2, xp2, gt2, gtn):
    if kind == 1:
        return hist >= 2 and abs(F - F_prev) <= thr * abs(F_prev)
    if kind == 2:
        return hist >= 2 and math.sqrt(dx2) <= thr * math.sqrt(xp2)
    if kind == 3:
        return math.sqrt(gt2) <= thr * gtn
    return False


def _kkt_partials(x, g, lam, cut):
    c = -g
    on = x != 0.0
    s = np.zeros(8)
    if np.any(on):
        s[0] = np.max(np.abs(c[on] - lam * np.sign(x[on])))
        s[2] = 1.0
    if np.any(~on):
        s[1] = np.max(np.abs(c[~on]))
        s[3] = 1.0
    s[4] = float(np.count_nonzero(np.abs(x) > cut))
    return s


class _Ctl:
    pass


class NumpyShardOps:
    def __init__(self, A_local, n_global=None, group=None):
        import torch.distributed as dist
        self.A = np.ascontiguousarray(A_local, dtype=np.float64)
        self.d, self.nl = self.A.shape
        self.ld = self.d
        self.n_global = n_global
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.xchg = np.zeros(self.d + SLOT * self.world)

    # primitives
    def zeros_d(self):
        return np.zeros(self.d)

    def zeros_n(self):
        return np.zeros(self.nl)

    def from_host_d(self, v):
        return np.array(v, dtype=np.float64)

    def to_host_d(self, v):
        return v.copy()

    def gemv(self, x, out):
        out[:] = self.A @ x

    def gemv_t(self, r, out):
        out[:] = self.A.T @ r

    def allreduce_(self, v):
        if self.world > 1:
            import torch
            import torch.distributed as dist
            dist.all_reduce(torch.from_numpy(v), op=dist.ReduceOp.SUM, group=self.group)

    # the solve
    def setup(self, b, gt_local=None):
        z = np.zeros(self.nl)
        self.x, self.xp, self.xn = z.copy(), z.copy(), z.copy()
        self.b = np.array(b, dtype=np.float64)
        self.gt = None if gt_local is None else np.array(gt_local, dtype=np.float64)
        self.r = -self.b
        self.rn = np.zeros(self.d)
        self.g = self.A.T @ self.r
        self.gp, self.gn = z.copy(), z.copy()
        slots = self.xchg[self.d:].reshape(self.world, SLOT)
        slots[:] = 0.0
        slots[self.rank, 8:] = _kkt_partials(self.x, self.g, 0.0, 1.0)
        self.allreduce_(self.xchg[self.d:])
        return float(np.max(slots[:, 9]))

    def begin(self, ctl):
        C = _Ctl()
        for name, _ in ctl._fields_:
            setattr(C, name, getattr(ctl, name))
        C.world, C.rank = self.world, self.rank
        self.C = C
        self.trace = np.zeros((max(int(C.max_iter), 1), 4))

    def round(self):
        self._pre()
        self.allreduce_(self.xchg)
        self._post()

    def _pre(self):                                  # sf_prox_kernel + gemv
        C = self.C
        slots = self.xchg[self.d:].reshape(self.world, SLOT)
        for r in range(self.world):
            if r != self.rank:
                slots[r] = 0.0
        if C.state != RUNNING:
            return
        m, L = C.m, C.L
        y = self.x + m * (self.x - self.xp)
        g = (1.0 + m) * self.g - m * self.gp
        u = soft(y - g / L, C.lam_k / L)
        dl = u - y
        s = np.zeros(8)
        s[0] = np.sum(np.abs(u))
        s[1] = g @ dl
        s[2] = dl @ dl
        s[3] = np.max(np.abs(u)) if u.size else 0.0
        s[4] = (u - self.x) @ (u - self.x)
        s[5] = self.x @ self.x
        if self.gt is not None:
            s[6] = (u - self.gt) @ (u - self.gt)
        self.xn = u
        slots[self.rank, :8] = s
        if C.run_trial:
            self.xchg[: self.d] = self.A @ u

    def _post(self):                                 # sf_decide_kernel + gemv_t + sf_advance_kernel
        C = self.C
        if C.state == FINISHED:
            return
        slots = self.xchg[self.d:].reshape(self.world, SLOT)
        rs0 = rs1 = 0.0
        if C.run_trial:
            rn = self.xchg[: self.d] - self.b
            self.rn = rn
            ry = (1.0 + C.mn) * rn - C.mn * self.r
            rs0, rs1 = float(rn @ rn), float(ry @ ry)
        C.adv = 0
        if C.pending:
            q = slots[:, 8:]
            kk = 0.0
            if np.any(q[:, 2] > 0):
                kk = float(np.max(q[:, 0]))
            if np.any(q[:, 3] > 0):
                kk = max(kk, float(np.max(q[:, 1])) - C.lam_used, 0.0)
            self.trace[C.it - 1, 3] = round(float(np.sum(q[:, 4])))
            C.pending = 0
            conv = C.lam_used == C.lam_bar and kk <= C.tol * C.lam_bar
            kfire = C.stop_kind == 4 and kk <= C.stop_thr
            if conv or kfire:
                C.converged = 1
            if conv or kfire or C.state == FINAL:
                if C.run_trial:
                    C.passes += 1
                C.state, C.run_trial = FINISHED, 0
                return
        if C.state != RUNNING:
            C.state, C.run_trial = FINISHED, 0
            return
        p = np.zeros(8)
        for r in range(self.world):
            for k in (0, 1, 2, 4, 5, 6):
                p[k] = p[k] + slots[r, k]
        p[3] = float(np.max(slots[:, 3]))
        C.trials += 1
        C.passes += 1
        l1 = p[0]
        Fn = 0.5 * rs0 + C.lam_k * l1
        if not C.exact:
            Q = C.f_y + p[1] + 0.5 * C.L * p[2] + C.lam_k * l1
            if not Fn <= Q + 1e-12 * max(1.0, abs(Q)):
                C.L *= C.eta
                C.growths += 1
                if C.growths >= 101:
                    C.status, C.state, C.run_trial = 3, FINISHED, 0
                return
        C.growths = 0
        C.it += 1
        C.passes += 1
        C.adv = 1
        self.trace[C.it - 1] = (C.it, Fn, math.sqrt(rs0), 0.0)
        C.pending = 1
        C.lam_used = C.lam_k
        C.cut = 1e-10 * max(p[3], 1.0)
        C.hist = min(C.hist + 1, 2)
        fires = C.stop_kind != 4 and _stop_fires(C.stop_kind, C.stop_thr, C.hist, Fn, C.F_prev,
                                                  p[4], p[5], p[6], C.gt_norm)
        t_new = _t_next(C.tc)
        C.tp, C.tc = C.tc, t_new
        C.f_y = 0.5 * rs1
        C.F_prev = Fn
        if fires:
            C.converged = 1
        if fires or C.it >= C.max_iter:
            C.state, C.run_trial = FINAL, 0
        else:
            C.lam_k = max(C.beta * C.lam_k, C.lam_bar)
            C.m = (C.tp - 1.0) / C.tc
            C.mn = (C.tc - 1.0) / _t_next(C.tc)
        # A_r^T r_n, rotation, KKT partials of the accepted iterate
        self.gn = self.A.T @ self.rn
        self.xp, self.x = self.x, self.xn.copy()
        self.gp, self.g = self.g, self.gn.copy()
        self.r = self.rn.copy()
        slots[self.rank, 8:] = _kkt_partials(self.x, self.g, C.lam_used, C.cut)

    def poll_async(self):
        return self.C.state

    def poll_wait(self, h):
        return h

    def result(self):
        from types import SimpleNamespace
        C = self.C
        ctl = SimpleNamespace(it=C.it, passes=C.passes, trials=C.trials, status=C.status,
                              converged=C.converged)
        tr = self.trace[: C.it].copy()
        if self.world == 1:
            return ctl, tr, self.x.copy()
        import torch
        import torch.distributed as dist
        from paper_1007_3753_b200.sharded import column_range
        sizes = [column_range(self.n_global, r, self.world) for r in range(self.world)]
        cap = max(c1 - c0 for c0, c1 in sizes)
        buf = torch.zeros(cap, dtype=torch.float64)
        buf[: self.nl] = torch.from_numpy(self.x)
        outs = [torch.zeros(cap, dtype=torch.float64) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return ctl, tr, np.concatenate([outs[r].numpy()[: c1 - c0] for r, (c0, c1) in enumerate(sizes)])


# ---------------------------------------------------------------------------
# column-sharded Homotopy (paper_1007_3753_b200/sharded_homotopy.py ops)
# ---------------------------------------------------------------------------

class NumpyHomShardOps:
    """numpy + gloo restatement of DeviceHomShardOps (csrc/shard_hom.cu
    reductions, the chol_* factor kernels) — test infrastructure only."""

    SLOT = 4

    def __init__(self, A_local, n_global, group=None):
        import torch.distributed as dist
        from paper_1007_3753_b200.sharded import column_range
        self.A = np.ascontiguousarray(A_local, dtype=np.float64)
        self.d, self.nl = self.A.shape
        self.n = n_global
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.c0, _ = column_range(n_global, self.rank, self.world)
        self.S = np.zeros((0, self.d))
        self.mask = np.zeros(self.nl, dtype=bool)
        self.c = np.zeros(self.nl)
        self.w = np.zeros(self.nl)

    def _allreduce(self, v):
        if self.world > 1:
            import torch
            import torch.distributed as dist
            dist.all_reduce(torch.from_numpy(v), op=dist.ReduceOp.SUM, group=self.group)

    def vec_m(self, m):
        return np.zeros(max(m, 1))

    def set_b(self, b):
        self.b = np.array(b, dtype=np.float64)
        self.bnorm = float(np.linalg.norm(b))

    def corr(self, r):
        self.c = self.A.T @ r

    def corr_exchange(self, sup):
        m = len(sup)
        buf = np.zeros(m + self.SLOT * self.world)
        for p, j in enumerate(sup):
            if self.c0 <= j < self.c0 + self.nl:
                buf[p] = self.c[j - self.c0]
        s = buf[m + self.SLOT * self.rank:]
        if self.nl:
            k = int(np.argmax(np.abs(self.c)))
            s[0], s[1] = abs(self.c[k]), k + self.c0
        else:
            s[0], s[1] = -1.0, -1.0
        self._allreduce(buf)
        sl = buf[m:].reshape(self.world, self.SLOT)
        best, arg = -1.0, -1
        for r in range(self.world):
            if sl[r, 1] >= 0 and sl[r, 0] > best:
                best, arg = float(sl[r, 0]), int(sl[r, 1])
        return buf[:m].copy(), max(best, 0.0), arg

    def wpass(self, v):
        self.w = self.A.T @ v

    def gammas(self, lam):
        import math
        from paper_1007_3753_b200.sharded import column_range
        mask = self.mask
        gp_loc = np.full(4, np.inf)
        gp_loc[1] = gp_loc[3] = -1
        off = np.nonzero(~mask)[0]
        if off.size:
            co, wo = self.c[off], self.w[off]
            with np.errstate(divide="ignore", invalid="ignore"):
                ra = (lam - co) / (1.0 - wo)
                rb = (lam + co) / (1.0 + wo)
            floor = 1e-10 * max(lam, 1e-30)
            for q, rr in ((0, ra), (2, rb)):
                ok = np.isfinite(rr) & (rr > floor)
                if np.any(ok):
                    j = int(np.argmin(np.where(ok, rr, np.inf)))
                    gp_loc[q], gp_loc[q + 1] = rr[j], off[j]
        buf = np.zeros(self.SLOT * self.world)
        buf[self.SLOT * self.rank: self.SLOT * (self.rank + 1)] = gp_loc
        self._allreduce(buf)
        sl = buf.reshape(self.world, self.SLOT)
        ga, ia, gb, ib = math.inf, -1, math.inf, -1
        for r in range(self.world):
            c0 = column_range(self.n, r, self.world)[0]
            if sl[r, 1] >= 0 and sl[r, 0] < ga:
                ga, ia = float(sl[r, 0]), int(sl[r, 1]) + c0
            if sl[r, 3] >= 0 and sl[r, 2] < gb:
                gb, ib = float(sl[r, 2]), int(sl[r, 3]) + c0
        return (gb, ib) if gb < ga else (ga, ia)

    def fetch_column(self, j):
        col = np.zeros(self.d)
        if self.c0 <= j < self.c0 + self.nl:
            col[:] = self.A[:, j - self.c0]
        self._allreduce(col)
        return col

    def set_mask(self, j, on):
        if self.c0 <= j < self.c0 + self.nl:
            self.mask[j - self.c0] = on

    def store_put(self, m, col):
        self.S = np.vstack([self.S[:m], col[None, :]])

    def store_drop(self, pos, m):
        self.S = np.delete(self.S[:m], pos, axis=0)

    def S_times(self, m, xI):
        return self.S[:m].T @ xI[:m] if m else np.zeros(self.d)

    def St_times(self, m, v):
        return self.S[:m] @ v

    def resid(self, m, xI):
        return self.b - self.S_times(m, xI)

    def sumsq(self, v, n):
        return float(np.asarray(v)[:n] @ np.asarray(v)[:n])

    def norm(self, v, n):
        return float(np.linalg.norm(np.asarray(v)[:n]))

    def matvec(self, G, m, x):
        return G.reshape(m, m) @ x[:m]

    def gram(self, m):
        return (self.S[:m] @ self.S[:m].T).reshape(-1)

    def gram_ridge(self, m):
        G = self.S[:m] @ self.S[:m].T
        G[np.diag_indices_from(G)] += 1e-12 * max(float(np.trace(G)), 1.0)
        return G.reshape(-1)

    def remove_entry(self, x, pos, m):
        return np.delete(np.asarray(x)[:m], pos)

    def append_zero(self, x, m):
        return np.concatenate([np.asarray(x)[:m], [0.0]])

    def chol(self, G, m):
        from oracle.l1_oracle import NotPD, chol_upper
        from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError
        try:
            return chol_upper(G.reshape(m, m)).reshape(-1)
        except NotPD as exc:
            raise NotPositiveDefiniteError(str(exc)) from exc

    def solve(self, R, m, rhs):
        from oracle.l1_oracle import chol_solve
        return chol_solve(R.reshape(m, m), rhs[:m])

    def grow(self, R, m, g, diag):
        from oracle.l1_oracle import NotPD, chol_grow
        from paper_1007_3753_b200.exceptions import NotPositiveDefiniteError
        Rm = R.reshape(m, m) if m else np.zeros((0, 0))
        try:
            return chol_grow(Rm, g[:m] if m else np.zeros(0), diag).reshape(-1)
        except NotPD as exc:
            raise NotPositiveDefiniteError(str(exc)) from exc

    def drop(self, R, m, k):
        from oracle.l1_oracle import chol_drop
        return chol_drop(R.reshape(m, m), k).reshape(-1)

    def gamma_minus(self, m, xI, dI, sup):
        best, pos = np.inf, -1
        for k in np.argsort(sup, kind="stable"):
            with np.errstate(divide="ignore", invalid="ignore"):
                r = -xI[k] / dI[k]
            if np.isfinite(r) and r > 0 and r < best:
                best, pos = float(r), int(k)
        return best, pos

    def xstats(self, m, xI):
        x = np.asarray(xI[:m])
        cut = 1e-10 * max(float(np.max(np.abs(x))) if m else 0.0, 1.0)
        return float(np.sum(np.abs(x))), int(np.count_nonzero(np.abs(x) > cut))

    def axpy(self, a, x, y):
        y[: len(x)] += a * x

    def sign(self, v):
        return np.sign(v)

    def to_host(self, v):
        return np.array(v, dtype=np.float64)
