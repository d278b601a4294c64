"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference solvers.

This module restates, in its own structure, the algorithms of the
reference package ``ell1`` (``/root/reference/pkg/src/ell1``).  Every routine
cites the reference lines it follows.  It is the parity checker for the
B200 path and the CPU baseline timed by ``bench.py``; the product package
never imports it.  Pinned against the real reference via committed golden
fixtures (see ``oracle/__init__.py``).

Semantics notes
  * soft-threshold follows the compiled reference kernel
    (``_accel/_fastkernels.pyx:14-27``): u>a -> u-a, u<-a -> u+a, else +0.
  * all arithmetic is float64, operation order kept as in the reference so
    that the restatement reproduces the reference bit-for-bit on the same
    BLAS.
"""

from collections import namedtuple

import numpy as np
from scipy.linalg import solve_triangular

Outcome = namedtuple("Outcome", "x iterations converged trace notes")


class OracleError(RuntimeError):
    kind = "numerical"


class Breakdown(OracleError):
    kind = "breakdown"


class IllConditioned(OracleError):
    kind = "ill-conditioned"


class NotPD(OracleError):
    kind = "not-positive-definite"


class Degenerate(OracleError):
    kind = "degenerate-support"


# ----------------------------------------------------------------------------
# operators: dense A and the implicit [A, sI] stack (robust.py:57-155)
# ----------------------------------------------------------------------------

class Dense:
    """Dense dictionary (operators.py:13-58)."""

    def __init__(self, A):
        self.M = np.ascontiguousarray(A, dtype=np.float64)
        self._nsq = None

    @property
    def shape(self):
        return self.M.shape

    def mv(self, w):
        return self.M @ w

    def rmv(self, r):
        return self.M.T @ r

    def cols_mv(self, idx, coef):            # operators.py:32-33
        return self.M[:, idx] @ coef

    def cols_dot(self, idx, v):               # operators.py:35-36
        return self.M[:, idx].T @ v

    def gram_col(self, idx, j):               # operators.py:41-42
        return self.M[:, idx].T @ self.M[:, j]

    def col_sq(self):
        return np.sum(self.M * self.M, axis=0)

    def row_gram(self):                       # alm.py:164 (A @ A.T)
        return self.M @ self.M.T

    def wgram(self, w):                       # operators.py:53-55
        return (self.M * w) @ self.M.T

    def norm_sq(self):
        if self._nsq is None:
            self._nsq = power_norm_sq(self.M)
        return self._nsq


class Stacked:
    """[A, s I] never materialised (robust.py:57-155)."""

    def __init__(self, A, s):
        self.M = np.ascontiguousarray(A, dtype=np.float64)
        self.s = float(s)
        self._nsq = None

    @property
    def shape(self):
        d, n = self.M.shape
        return (d, n + d)

    def mv(self, w):                          # robust.py:91-93
        n = self.M.shape[1]
        return self.M @ w[:n] + self.s * w[n:]

    def rmv(self, r):                         # robust.py:95-96
        return np.concatenate([self.M.T @ r, self.s * r])

    def _col(self, j):                        # robust.py:98-104
        d, n = self.M.shape
        if j < n:
            return self.M[:, j].copy()
        e = np.zeros(d)
        e[j - n] = self.s
        return e

    def cols_mv(self, idx, coef):             # robust.py:106-117
        d, n = self.M.shape
        idx = np.asarray(idx, dtype=np.intp)
        coef = np.asarray(coef, dtype=np.float64)
        acc = np.zeros(d)
        lo = idx < n
        if np.any(lo):
            acc += self.M[:, idx[lo]] @ coef[lo]
        hi = ~lo
        if np.any(hi):
            acc[idx[hi] - n] += self.s * coef[hi]
        return acc

    def cols_dot(self, idx, v):               # robust.py:119-129
        n = self.M.shape[1]
        idx = np.asarray(idx, dtype=np.intp)
        res = np.empty(idx.shape[0])
        lo = idx < n
        if np.any(lo):
            res[lo] = self.M[:, idx[lo]].T @ v
        hi = ~lo
        if np.any(hi):
            res[hi] = self.s * v[idx[hi] - n]
        return res

    def gram_col(self, idx, j):               # robust.py:131-132
        return self.cols_dot(idx, self._col(j))

    def col_sq(self):                         # robust.py:134-137
        d = self.M.shape[0]
        return np.concatenate([np.sum(self.M * self.M, axis=0),
                               np.full(d, self.s ** 2)])

    def row_gram(self):                       # robust.py:151-155
        d = self.M.shape[0]
        G = self.M @ self.M.T
        G[np.diag_indices(d)] += self.s ** 2
        return G

    def norm_sq(self):                        # robust.py:139-143
        if self._nsq is None:
            self._nsq = power_norm_sq(self.M) + self.s ** 2
        return self._nsq

    def wgram(self, w):                       # robust.py:145-149
        d, n = self.M.shape
        G = (self.M * w[:n]) @ self.M.T
        G[np.diag_indices(d)] += self.s ** 2 * w[n:]
        return G


def as_op(A):
    if isinstance(A, (Dense, Stacked)):
        return A
    return Dense(A)


# ----------------------------------------------------------------------------
# elementwise kernels and small helpers
# ----------------------------------------------------------------------------

def soft(u, a):
    """Compiled shrinkage semantics (_fastkernels.pyx:14-27)."""
    u = np.asarray(u, dtype=np.float64)
    out = np.zeros(u.shape)
    hi = u > a
    lo = u < -a
    out[hi] = u[hi] - a
    out[lo] = u[lo] + a
    return out


def clamp1(z):
    """Box projection onto [-1, 1] (_fastkernels.pyx:30-43)."""
    return np.clip(np.asarray(z, dtype=np.float64), -1.0, 1.0)


def l1(x):
    return float(np.sum(np.abs(x)))


def count_support(x, rel=1e-10):
    """model.py:227-233."""
    x = np.asarray(x)
    if x.size == 0:
        return 0
    cut = rel * max(float(np.max(np.abs(x))), 1.0)
    return int(np.count_nonzero(np.abs(x) > cut))


def kkt_of(x, c, lam):
    """Worst first-order violation given c = A^T(b - Ax) (model.py:160-173)."""
    nz = x != 0.0
    worst = 0.0
    if np.any(nz):
        worst = float(np.max(np.abs(c[nz] - lam * np.sign(x[nz]))))
    if np.any(~nz):
        worst = max(worst, float(np.max(np.abs(c[~nz])) - lam), 0.0)
    return worst


class StopTracker:
    """User stopping rules over the last two snapshots (model.py:176-224)."""

    def __init__(self, rule, gt=None):
        self.rule = rule          # None or (kind, threshold)
        self.gt = gt
        self.hist = []

    def push(self, x, obj, kkt):
        self.hist.append((x.copy(), obj, kkt))
        self.hist = self.hist[-2:]

    def fire(self):
        if self.rule is None or not self.hist:
            return False
        kind, thr = self.rule
        if kind in ("relative-objective", "relative-estimate"):
            if len(self.hist) < 2:
                return False
            (xp, fp, _), (xc, fc, _) = self.hist
            if kind == "relative-objective":
                return abs(fc - fp) <= thr * abs(fp)
            return float(np.linalg.norm(xc - xp)) <= thr * float(np.linalg.norm(xp))
        if kind == "ground-truth-distance":
            if self.gt is None:
                raise ValueError("ground-truth-distance rule needs a ground truth")
            g = np.asarray(self.gt, dtype=np.float64)
            nrm = float(np.linalg.norm(g))
            if nrm == 0.0:
                raise ValueError("ground truth must be nonzero")
            return float(np.linalg.norm(self.hist[-1][0] - g)) <= thr * nrm
        kk = self.hist[-1][2]
        if kk is None:
            raise ValueError("kkt-residual rule needs records carrying kkt values")
        return kk <= thr


# ----------------------------------------------------------------------------
# numerics: power iteration, PCG, Cholesky machinery (numerics.py)
# ----------------------------------------------------------------------------

POWER_SEED = 218751


def power_norm_sq(M, tol=1e-6, max_iter=1000):
    """Largest eig of M^T M via the smaller Gram side (numerics.py:227-261)."""
    M = np.asarray(M, dtype=np.float64)
    if not np.any(M):
        raise ValueError("zero matrix")
    d, n = M.shape
    if d <= n:
        gram = lambda v: M @ (M.T @ v)
        dim = d
    else:
        gram = lambda v: M.T @ (M @ v)
        dim = n
    gen = np.random.default_rng(POWER_SEED)
    v = gen.standard_normal(dim)
    v /= np.linalg.norm(v)
    theta = 0.0
    for _ in range(max_iter):
        w = gram(v)
        theta = float(v @ w)
        if np.linalg.norm(w - theta * v) <= tol * max(theta, np.finfo(float).tiny):
            break
        nw = np.linalg.norm(w)
        if nw == 0.0:
            v = gen.standard_normal(dim)
            v /= np.linalg.norm(v)
            continue
        v = w / nw
    return theta


def pcg(matvec, rhs, diag=None, tol=1e-8, max_iter=None):
    """Jacobi-preconditioned CG; best iterate on breakdown (numerics.py:164-221).

    Returns (x, converged, iterations, rel_residual)."""
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    n = rhs.shape[0]
    prec = (lambda r: r) if diag is None else (lambda r, _d=np.asarray(diag): r / _d)
    if max_iter is None:
        max_iter = n
    bn = float(np.linalg.norm(rhs))
    x = np.zeros(n)
    if bn == 0.0:
        return x, True, 0, 0.0
    r = rhs.copy()
    z = prec(r)
    p = z.copy()
    rz = float(r @ z)
    best, best_res = x.copy(), bn
    for k in range(1, max_iter + 1):
        Ap = matvec(p)
        curv = float(p @ Ap)
        if not np.isfinite(curv):
            raise Breakdown("non-finite curvature in PCG")
        if curv <= 0.0:
            return best, False, k, best_res / bn
        step = rz / curv
        x = x + step * p
        r = r - step * Ap
        res = float(np.linalg.norm(r))
        if not np.isfinite(res):
            raise Breakdown("non-finite residual in PCG")
        if res < best_res:
            best_res, best = res, x.copy()
        if res <= tol * bn:
            return x, True, k, res / bn
        z = prec(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return best, False, max_iter, best_res / bn


def chol_upper(G):
    """Upper factor R with R^T R = G (numerics.py:75-87)."""
    try:
        Lw = np.linalg.cholesky(np.asarray(G, dtype=np.float64))
    except np.linalg.LinAlgError as exc:
        raise NotPD(str(exc)) from exc
    return np.ascontiguousarray(Lw.T)


def chol_solve(R, rhs):
    """(R^T R) x = rhs (numerics.py:62-65)."""
    t = solve_triangular(R, rhs, trans="T", lower=False)
    return solve_triangular(R, t, trans="N", lower=False)


def rank1_update(R, v):
    """LINPACK rank-1 update in place, consumes v (_fastkernels.pyx:46-59)."""
    m = R.shape[0]
    for k in range(m):
        rkk = R[k, k]
        r = np.hypot(rkk, v[k])
        c = r / rkk
        s = v[k] / rkk
        R[k, k] = r
        for j in range(k + 1, m):
            row = (R[k, j] + s * v[j]) / c
            R[k, j] = row
            v[j] = c * v[j] - s * row
    return 0


def rank1_downdate(R, v):
    """Rank-1 downdate; 0 or failing pivot+1 (_fastkernels.pyx:62-78)."""
    m = R.shape[0]
    for k in range(m):
        rkk = R[k, k]
        d2 = (rkk - v[k]) * (rkk + v[k])
        if d2 <= 0.0:
            return k + 1
        r = np.sqrt(d2)
        c = r / rkk
        s = v[k] / rkk
        R[k, k] = r
        for j in range(k + 1, m):
            row = (R[k, j] - s * v[j]) / c
            R[k, j] = row
            v[j] = c * v[j] - s * row
    return 0


def chol_grow(R, g, diag):
    """Factor of [[G, g], [g^T, diag]] from the factor of G (numerics.py:115-137)."""
    m = R.shape[0]
    out = np.zeros((m + 1, m + 1))
    out[:m, :m] = R
    if m:
        u = solve_triangular(R, g, trans="T", lower=False)
        out[:m, m] = u
        d2 = float(diag) - float(u @ u)
    else:
        d2 = float(diag)
    if d2 <= 0.0:
        raise NotPD("appended column makes the matrix singular")
    out[m, m] = np.sqrt(d2)
    return out


def chol_drop(R, k):
    """Remove row/col k: block permutation + rank-1 update (numerics.py:140-158)."""
    m = R.shape[0]
    out = np.zeros((m - 1, m - 1))
    out[:k, :k] = R[:k, :k]
    out[:k, k:] = R[:k, k + 1:]
    if k < m - 1:
        tail = np.ascontiguousarray(R[k + 1:, k + 1:].copy())
        rank1_update(tail, R[k, k + 1:].copy())
        out[k:, k:] = tail
    return out


# ----------------------------------------------------------------------------
# FISTA (shrinkage.py:184-298)
# ----------------------------------------------------------------------------

def t_next(t):
    """shrinkage.py:184-196 with the nextafter nudge."""
    if not t >= 1.0:
        raise ValueError("t must be at least 1")
    tn = 0.5 * (1.0 + np.sqrt(4.0 * t * t + 1.0))
    while tn * tn - tn > t * t:
        tn = np.nextafter(tn, 1.0)
    return tn


def _majorize(op, b, y, g_y, f_y, L, eta, lam):
    """Backtracking on L (shrinkage.py:199-213)."""
    for _ in range(101):
        xn = soft(y - g_y / L, lam / L)
        rn = op.mv(xn) - b
        Fn = 0.5 * float(rn @ rn) + lam * l1(xn)
        dl = xn - y
        Q = f_y + float(g_y @ dl) + 0.5 * L * float(dl @ dl) + lam * l1(xn)
        if Fn <= Q + 1e-12 * max(1.0, abs(Q)):
            return L, xn, rn, Fn
        L *= eta
    raise Breakdown("backtracking exceeded 100 growth steps")


def backtrack(A, b, y, L_prev, eta, lam):
    """shrinkage.py:216-228 -> (L, x_next)."""
    if not L_prev > 0:
        raise ValueError("L_prev must be positive")
    if not eta > 1:
        raise ValueError("eta must exceed 1")
    op = as_op(A)
    y = np.asarray(y, dtype=np.float64)
    r_y = op.mv(y) - b
    g_y = op.rmv(r_y)
    L, xn, _, _ = _majorize(op, b, y, g_y, 0.5 * float(r_y @ r_y), L_prev, eta, lam)
    return L, xn


def fista(A, b, lam=None, tol=1e-6, max_iter=5000, stop=None, opts=None, gt=None,
          watch=None):
    """Accelerated proximal gradient with continuation (shrinkage.py:231-298).

    watch(x_prev, x, t_prev, t_cur, L, y, lam) mirrors the observer."""
    op = as_op(A)
    opts = opts or {}
    b = np.asarray(b, dtype=np.float64)
    n = op.shape[1]
    c0 = float(np.max(np.abs(op.rmv(b)))) if n else 0.0
    lam_bar = float(lam) if lam is not None else 1e-2 * c0
    x = np.zeros(n)
    if c0 == 0.0:
        return Outcome(x, 0, True, [(0, 0.0, float(np.linalg.norm(b)), 0)], ())
    if not lam_bar > 0:
        raise ValueError("lambda must be positive")
    eta = opts.get("eta", 1.5)
    L = opts.get("L0", 1.0)
    beta = opts.get("beta", 0.5)
    exact = opts.get("exact_L", False)
    if exact:
        L = op.norm_sq() * (1.0 + 1e-9)
    lam_k = max(0.9 * c0, lam_bar) if opts.get("continuation", True) else lam_bar
    xp = x.copy()
    tp = tc = 1.0
    trace = []
    stopper = StopTracker(stop, gt)
    done = False
    it = 0
    while it < max_iter:
        it += 1
        y = x + ((tp - 1.0) / tc) * (x - xp)
        r_y = op.mv(y) - b
        g_y = op.rmv(r_y)
        if exact:
            xn = soft(y - g_y / L, lam_k / L)
            rn = op.mv(xn) - b
            Fn = 0.5 * float(rn @ rn) + lam_k * l1(xn)
        else:
            L, xn, rn, Fn = _majorize(op, b, y, g_y, 0.5 * float(r_y @ r_y),
                                      L, eta, lam_k)
        xp, x = x, xn
        tp, tc = tc, t_next(tc)
        trace.append((it, Fn, float(np.linalg.norm(rn)), count_support(x)))
        kk = kkt_of(x, -(op.rmv(rn)), lam_k)
        if watch is not None:
            watch(xp.copy(), x.copy(), tp, tc, L, y, lam_k)
        stopper.push(x, Fn, kk)
        if lam_k == lam_bar and kk <= tol * lam_bar:
            done = True
            break
        if stopper.fire():
            done = True
            break
        lam_k = max(beta * lam_k, lam_bar)
    return Outcome(x, it, done, trace, ())


# ----------------------------------------------------------------------------
# IST with BB steps over a continuation schedule (shrinkage.py:27-181)
# ----------------------------------------------------------------------------

def schedule_stages(lam_start, beta, lam_target):
    """shrinkage.py:43-58."""
    if lam_start == lam_target:
        return [lam_target]
    vals = [lam_start]
    while vals[-1] > lam_target:
        vals.append(max(vals[-1] * beta, lam_target))
    if len(vals) < 5:
        q = (lam_target / lam_start) ** 0.25
        vals = [lam_start * q ** i for i in range(5)]
        vals[-1] = lam_target
    return vals


def bb(s, g):
    """shrinkage.py:72-82."""
    ss = float(s @ s)
    ratio = float(s @ g) / ss if ss > 0.0 else 0.0
    return min(max(ratio, 1e-30), 1e30)


def obj_delta(x, cand, Ax, Acand, g, lam):
    """shrinkage.py:91-102."""
    dl = cand - x
    dA = Acand - Ax
    return (float(g @ dl) + 0.5 * float(dA @ dA)
            + lam * float(np.sum(np.abs(cand) - np.abs(x))))


def ist(A, b, stages=None, lam=None, tol=1e-6, max_iter=5000, stop=None, gt=None,
        watch=None):
    """SpaRSA-style IST (shrinkage.py:105-181).  stages=None -> default schedule
    (shrinkage.py:85-88) to the resolved lambda."""
    op = as_op(A)
    b = np.asarray(b, dtype=np.float64)
    n = op.shape[1]
    if stages is None:
        c0 = float(np.max(np.abs(op.rmv(b)))) if n else 0.0
        lam_t = float(lam) if lam is not None else 1e-2 * c0
        start = 0.9 * float(np.max(np.abs(op.rmv(b))))
        if not lam_t > 0:
            raise ValueError("lambda_target must be positive")
        stages = schedule_stages(max(start, lam_t), 0.5, lam_t)
    lam_t = stages[-1]
    x = np.zeros(n)
    if float(np.max(np.abs(op.rmv(b)))) == 0.0:
        return Outcome(x, 0, True, [(0, 0.0, float(np.linalg.norm(b)), 0)], ())
    trace = []
    stopper = StopTracker(stop, gt)
    it = 0
    done = False
    alpha = 1.0
    Ax = op.mv(x)
    g = op.rmv(Ax - b)
    kk = 0.0
    for lam_s in stages:
        last = lam_s == lam_t
        kk = kkt_of(x, -g, lam_s)
        if kk <= tol * lam_s:
            if last:
                done = True
            continue
        stalled = False
        while it < max_iter:
            ok = False
            for _ in range(50):
                cand = soft(x - g / alpha, lam_s / alpha)
                Ac = op.mv(cand)
                dF = obj_delta(x, cand, Ax, Ac, g, lam_s)
                if dF < 0.0:
                    ok = True
                    break
                alpha = min(alpha * 2.0, 1e30)
            if not ok:
                stalled = True
                break
            it += 1
            g_new = op.rmv(Ac - b)
            alpha = bb(cand - x, g_new - g)
            x, Ax, g = cand, Ac, g_new
            res = b - Ax
            F = 0.5 * float(res @ res) + lam_s * l1(x)
            trace.append((it, F, float(np.linalg.norm(res)), count_support(x)))
            if watch is not None:
                watch(x.copy(), lam_s, dF)
            kk = kkt_of(x, -g, lam_s)
            stopper.push(x, F, kk)
            if kk <= tol * lam_s:
                if last:
                    done = True
                break
            if stopper.fire():
                return Outcome(x, it, True, trace, ())
        if stalled and last and kk <= tol * lam_s:
            done = True
        if stalled and not last:
            continue
        if it >= max_iter and not done:
            break
    return Outcome(x, it, done, trace, ())


# ----------------------------------------------------------------------------
# PALM / DALM (alm.py)
# ----------------------------------------------------------------------------

def _palm_inner(op, x, b_eff, shrink, tau, tol_rel, cap):
    """alm.py:71-93 (plain t recurrence, no nudge)."""
    tp = 1.0
    xp = x
    yv = x
    k = 0
    for _ in range(cap):
        grad = op.rmv(op.mv(yv) - b_eff)
        xn = soft(yv - grad / tau, shrink)
        k += 1
        tn = 0.5 * (1.0 + np.sqrt(4.0 * tp * tp + 1.0))
        yv = xn + ((tp - 1.0) / tn) * (xn - xp)
        chg = float(np.linalg.norm(xn - xp))
        xp, tp = xn, tn
        if chg <= tol_rel * max(1.0, float(np.linalg.norm(xn))):
            break
    return xp, k


def palm(A, b, tol=1e-6, max_iter=5000, stop=None, opts=None, gt=None, watch=None):
    """Primal ALM (alm.py:96-159)."""
    op = as_op(A)
    opts = opts or {}
    b = np.asarray(b, dtype=np.float64)
    d, n = op.shape
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return Outcome(np.zeros(n), 0, True, [(0, 0.0, 0.0, 0)], ())
    mu = float(opts.get("mu0", 1.0))
    rho = float(opts.get("rho", 2.0))
    if not mu > 0 or not rho > 1:
        raise ValueError("mu0 must be positive and rho must exceed 1")
    tau = 1.01 * op.norm_sq()
    x = np.zeros(n)
    yd = np.zeros(d)
    trace = [(0, 0.0, bn, 0)]
    notes = []
    stopper = StopTracker(stop, gt)
    it = 0
    done = False
    while it < max_iter:
        b_eff = b + yd / mu
        x, k = _palm_inner(op, x, b_eff, 1.0 / (mu * tau), tau, 1e-2 / mu,
                           min(200, max_iter - it))
        it += k
        r = b - op.mv(x)
        rn = float(np.linalg.norm(r))
        yd = yd + mu * r
        v1 = l1(x)
        trace.append((it, v1, rn, count_support(x)))
        if watch is not None:
            watch(x.copy(), yd.copy(), mu, rho, tau)
        rel = rn / bn
        if rel <= tol:
            done = True
            break
        if stop is not None:
            stopper.push(x, v1, rel)
            if stopper.fire():
                done = True
                break
        mu *= rho
    if not done and it >= max_iter:
        notes.append("inner-iteration budget exhausted")
    return Outcome(x, it, done, trace, tuple(notes))


def gram_factor(op):
    """alm.py:162-169."""
    try:
        return chol_upper(op.row_gram())
    except NotPD as exc:
        raise IllConditioned("row Gram A A^T is not positive definite; the dual "
                             "solver needs full row rank") from exc


def y_step(op, R, x, beta, z, b):
    """Certified least-squares multiplier step (alm.py:172-189)."""
    rhs = op.mv(z) - (op.mv(x) - b) / beta
    y = chol_solve(R, rhs)
    res = rhs - op.mv(op.rmv(y))
    sc = max(1.0, float(np.linalg.norm(rhs)))
    if float(np.linalg.norm(res)) > 1e-10 * sc:
        y = y + chol_solve(R, res)
        res = rhs - op.mv(op.rmv(y))
        if float(np.linalg.norm(res)) > 1e-10 * sc:
            raise IllConditioned("dual least-squares step failed its residual contract")
    return y


def y_cg(op, yprev, x, beta, z, b):
    """One warm-started CG step on the y system (alm.py:192-203)."""
    rhs = op.mv(z) - (op.mv(x) - b) / beta
    r = rhs - op.mv(op.rmv(yprev))
    rr = float(r @ r)
    if rr == 0.0:
        return yprev
    Ar = op.mv(op.rmv(r))
    curv = float(r @ Ar)
    if curv <= 0.0:
        raise IllConditioned("row Gram lost positive definiteness")
    return yprev + (rr / curv) * r


def dalm(A, b, tol=1e-6, max_iter=5000, stop=None, opts=None, gt=None, watch=None):
    """Dual ALM (alm.py:206-272)."""
    op = as_op(A)
    opts = opts or {}
    b = np.asarray(b, dtype=np.float64)
    d, n = op.shape
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return Outcome(np.zeros(n), 0, True, [(0, 0.0, 0.0, 0)], ())
    beta = float(opts.get("beta", 1.0))
    if not beta > 0:
        raise ValueError("beta must be positive")
    cg_mode = bool(opts.get("y_cg_step", False))
    R = gram_factor(op)
    x = np.zeros(n)
    yv = np.zeros(d)
    trace = [(0, 0.0, bn, 0)]
    notes = []
    stopper = StopTracker(stop, gt)
    it = 0
    done = False
    while it < max_iter:
        z = clamp1(op.rmv(yv) + x / beta)
        if cg_mode:
            yv = y_cg(op, yv, x, beta, z, b)
        else:
            yv = y_step(op, R, x, beta, z, b)
        xprev = x
        Aty = op.rmv(yv)
        x = xprev - beta * (z - Aty)
        it += 1
        r = b - op.mv(x)
        rn = float(np.linalg.norm(r))
        v1 = l1(x)
        trace.append((it, v1, rn, count_support(x)))
        if watch is not None:
            watch(x.copy(), yv.copy(), z.copy(), xprev.copy())
        rel = rn / bn
        scale = max(1.0, float(np.max(np.abs(Aty))))
        gap = v1 - float(b @ yv) / scale
        if rel <= tol and gap <= tol * max(1.0, v1):
            done = True
            break
        if stop is not None:
            stopper.push(x, v1, rel)
            if stopper.fire():
                done = True
                break
    if not done and it >= max_iter:
        notes.append("iteration budget exhausted")
    return Outcome(x, it, done, trace, tuple(notes))


# ----------------------------------------------------------------------------
# GPSR and TNIPM (gradient_projection.py)
# ----------------------------------------------------------------------------

def gpsr(A, b, lam=None, tol=1e-6, max_iter=5000, stop=None, gt=None, watch=None):
    """Projected gradient on the nonnegative split (gradient_projection.py:114-192)."""
    op = as_op(A)
    b = np.asarray(b, dtype=np.float64)
    n = op.shape[1]
    if lam is None:
        lam = 1e-2 * (float(np.max(np.abs(op.rmv(b)))) if n else 0.0)
    if not lam > 0:
        raise ValueError("lambda must be positive")
    if float(np.max(np.abs(op.rmv(b)))) == 0.0:
        return Outcome(np.zeros(n), 0, True, [(0, 0.0, float(np.linalg.norm(b)), 0)], ())
    z = np.zeros(2 * n)
    x = np.zeros(n)
    r = -b.copy()
    gx = op.rmv(r)
    trace = [(0, 0.5 * float(b @ b), float(np.linalg.norm(b)), 0)]
    notes = []
    stopper = StopTracker(stop, gt)
    it = 0
    done = False
    while it < max_iter:
        kk = kkt_of(x, -gx, lam)
        if kk <= tol * lam:
            done = True
            break
        grad = np.concatenate([gx + lam, lam - gx])
        g = np.where((z > 0.0) | (grad < 0.0), grad, 0.0)
        gg = float(g @ g)
        if gg == 0.0:
            notes.append("zero projected gradient before kkt tolerance")
            break
        Av = op.mv(g[:n] - g[n:])
        curv = float(Av @ Av)
        alpha = 1e8 if curv <= 1e-14 * gg else gg / curv
        ok = False
        for _ in range(51):
            cand = np.maximum(z - alpha * g, 0.0)
            xc = cand[:n] - cand[n:]
            Adx = op.mv(xc - x)
            dQ = float(grad @ (cand - z)) + 0.5 * float(Adx @ Adx)
            if dQ < 0.0:
                ok = True
                break
            alpha *= 0.5
        if not ok:
            notes.append("projection backtracking stalled")
            done = kk <= tol * lam
            break
        it += 1
        z, x = cand, xc
        if it % 64 == 0:
            r = op.mv(x) - b
        else:
            r = r + Adx
        gx = op.rmv(r)
        F = 0.5 * float(r @ r) + lam * l1(x)
        trace.append((it, F, float(np.linalg.norm(r)), count_support(x)))
        if watch is not None:
            watch(z.copy())
        if stop is not None:
            kk = kkt_of(x, -gx, lam)
            stopper.push(x, F, kk)
            if stopper.fire():
                return Outcome(x, it, True, trace, tuple(notes))
    if not done:
        done = kkt_of(x, -gx, lam) <= tol * lam
    return Outcome(x, it, done, trace, tuple(notes))


def _snap(x):
    """gradient_projection.py:195-206."""
    out = x.copy()
    top = float(np.max(np.abs(out))) if out.size else 0.0
    if top > 0.0:
        out[np.abs(out) <= 1e-7 * top] = 0.0
    return out


def _barrier(t, lam, r, x, u):
    """gradient_projection.py:209-215."""
    up = u + x
    um = u - x
    if float(np.min(up)) <= 0.0 or float(np.min(um)) <= 0.0:
        return np.inf
    return (t * (0.5 * float(r @ r) + lam * float(np.sum(u)))
            - float(np.sum(np.log(up))) - float(np.sum(np.log(um))))


def tnipm(A, b, lam=None, tol=1e-6, max_iter=5000, stop=None, opts=None, gt=None,
          watch=None, pcg_fn=None):
    """Truncated-Newton interior point (gradient_projection.py:218-339)."""
    op = as_op(A)
    opts = opts or {}
    b = np.asarray(b, dtype=np.float64)
    n = op.shape[1]
    if lam is None:
        lam = 1e-2 * (float(np.max(np.abs(op.rmv(b)))) if n else 0.0)
    if not lam > 0:
        raise ValueError("lambda must be positive")
    if float(np.max(np.abs(op.rmv(b)))) == 0.0:
        return Outcome(np.zeros(n), 0, True, [(0, 0.0, float(np.linalg.norm(b)), 0)], ())
    solve = pcg_fn or pcg
    ptol = opts.get("pcg_tol", 1e-4)
    pcap = opts.get("pcg_max_iter", None)
    csq = op.col_sq()
    x = np.zeros(n)
    u = np.ones(n)
    t = 1.0 / lam
    trace = []
    notes = []
    stopper = StopTracker(stop, gt)
    it = 0
    done = False
    capped = 0
    while it < max_iter:
        r = op.mv(x) - b
        Ar = op.rmv(r)
        F = 0.5 * float(r @ r) + lam * l1(x)
        trace.append((it, F, float(np.linalg.norm(r)), count_support(_snap(x))))
        if stop is not None:
            stopper.push(x, F, kkt_of(x, -Ar, lam))
            if stopper.fire():
                done = True
                x = _snap(x)
                break
        if 2.0 * n / t <= tol * (1.0 + F):
            xt = _snap(x)
            ct = op.rmv(b - op.mv(xt))
            if kkt_of(xt, ct, lam) <= tol * lam:
                done = True
                x = xt
                break
        up = u + x
        um = u - x
        p = 1.0 / up
        q = 1.0 / um
        g_x = t * Ar + (q - p)
        g_u = t * lam - p - q
        pp = p * p
        qq = q * q
        dsum = pp + qq
        ddif = pp - qq
        dred = 4.0 * pp * qq / dsum
        rhs = -g_x + ddif * (g_u / dsum)
        mv = lambda v: t * (op.rmv(op.mv(v))) + dred * v
        dx, conv, _, _ = solve(mv, rhs, t * csq + dred, ptol, pcap)
        if not conv:
            capped += 1
        du = -(g_u + ddif * dx) / dsum
        dec = -(float(g_x @ dx) + float(g_u @ du))
        s = 1.0
        dup = du + dx
        dum = du - dx
        m = dup < 0.0
        if np.any(m):
            s = min(s, 0.99 * float(np.min(up[m] / -dup[m])))
        m = dum < 0.0
        if np.any(m):
            s = min(s, 0.99 * float(np.min(um[m] / -dum[m])))
        Ft = _barrier(t, lam, r, x, u)
        Adx = op.mv(dx)
        ok = False
        for _ in range(51):
            Fnew = _barrier(t, lam, r + s * Adx, x + s * dx, u + s * du)
            if Fnew <= Ft - 0.01 * s * dec:
                ok = True
                break
            s *= 0.5
        if not ok:
            raise Breakdown("barrier line search exhausted without an interior decrease")
        x = x + s * dx
        u = u + s * du
        it += 1
        if watch is not None:
            watch(x.copy(), u.copy(), t)
        if dec <= 0.25:
            t *= 10.0
    x = _snap(x)
    if not done:
        rt = op.mv(x) - b
        Ft = 0.5 * float(rt @ rt) + lam * l1(x)
        if (2.0 * n / t <= tol * (1.0 + Ft)
                and kkt_of(x, op.rmv(-rt), lam) <= tol * lam):
            done = True
    if capped:
        notes.append("pcg hit its iteration cap %d times" % capped)
    return Outcome(x, it, done, trace, tuple(notes))


# ----------------------------------------------------------------------------
# Homotopy (homotopy.py)
# ----------------------------------------------------------------------------

def _direction(R, op, sup, sgn):
    """homotopy.py:41-64 -> (d_I, R)."""
    if not sup:
        return np.zeros(0), R
    dI = chol_solve(R, sgn)
    v = op.cols_mv(sup, dI)
    Gd = op.cols_dot(sup, v)
    tol = 1e-6 * max(1.0, float(np.linalg.norm(sgn)))
    if np.linalg.norm(Gd - sgn) <= tol:
        return dI, R
    G = np.empty((len(sup), len(sup)))
    for c, j in enumerate(sup):
        G[:, c] = op.gram_col(sup, j)
    try:
        Rf = chol_upper(G)
    except NotPD as exc:
        raise Degenerate("active-set Gram is singular") from exc
    dI = chol_solve(Rf, sgn)
    if np.linalg.norm(G @ dI - sgn) > tol:
        raise Degenerate("active-set Gram solve failed")
    return dI, Rf


def step_lengths(lam, c, x, dfull, w, mask):
    """Next add/remove events (homotopy.py:78-105)."""
    off = ~mask
    gp, ip = np.inf, -1
    if np.any(off):
        idx = np.nonzero(off)[0]
        co, wo = c[idx], w[idx]
        with np.errstate(divide="ignore", invalid="ignore"):
            ra = (lam - co) / (1.0 - wo)
            rb = (lam + co) / (1.0 + wo)
        floor = 1e-10 * max(lam, 1e-30)
        for rr in (ra, rb):
            ok = np.isfinite(rr) & (rr > floor)
            if np.any(ok):
                j = int(np.argmin(np.where(ok, rr, np.inf)))
                if rr[j] < gp:
                    gp, ip = float(rr[j]), int(idx[j])
    gm, im = np.inf, -1
    sp = np.nonzero(mask)[0]
    if sp.size:
        with np.errstate(divide="ignore", invalid="ignore"):
            rr = -x[sp] / dfull[sp]
        ok = np.isfinite(rr) & (rr > 0)
        if np.any(ok):
            j = int(np.argmin(np.where(ok, rr, np.inf)))
            gm, im = float(rr[j]), int(sp[j])
    return gp, ip, gm, im


def _ridge(op, sup, notes):
    """homotopy.py:118-125."""
    G = np.empty((len(sup), len(sup)))
    for c, j in enumerate(sup):
        G[:, c] = op.gram_col(sup, j)
    G[np.diag_indices_from(G)] += 1e-12 * max(np.trace(G), 1.0)
    if "ridge-regularized gram" not in notes:
        notes.append("ridge-regularized gram")
    return chol_upper(G)


def homotopy(A, b, target, max_iter=5000, watch=None):
    """LASSO path to `target` (homotopy.py:128-244) -> (Outcome, reached lambda)."""
    if target < 0:
        raise ValueError("target lambda must be nonnegative")
    op = as_op(A)
    n = op.shape[1]
    b = np.asarray(b, dtype=np.float64)
    notes = []
    x = np.zeros(n)
    c = op.rmv(b)
    lam0 = float(np.max(np.abs(c))) if n else 0.0
    trace = []

    def log(k, lam_k, rnorm):
        trace.append((k, 0.5 * rnorm ** 2 + lam_k * l1(x), rnorm, count_support(x)))

    if lam0 <= target or lam0 == 0.0:
        log(0, max(lam0, target), float(np.linalg.norm(b)))
        return Outcome(x, 0, True, trace, ()), max(lam0, target)
    lam = lam0
    j0 = int(np.argmax(np.abs(c)))
    sup = [j0]
    R = chol_grow(np.zeros((0, 0)), np.zeros(0), float(op.gram_col([j0], j0)[0]))
    mask = np.zeros(n, dtype=bool)
    mask[j0] = True
    done = False
    it = 0
    floor = max(target, 1e-12 * lam0)
    while it < max_iter:
        it += 1
        sgn = np.sign(c[sup])
        try:
            dI, R = _direction(R, op, sup, sgn)
        except Degenerate:
            R = _ridge(op, sup, notes)
            dI = chol_solve(R, sgn)
        v = op.cols_mv(sup, dI)
        w = op.rmv(v)
        dfull = np.zeros(n)
        dfull[sup] = dI
        gp, ip, gm, im = step_lengths(lam, c, x, dfull, w, mask)
        ge = min(gp, gm)
        cap = lam - target
        if cap <= ge:
            x[sup] += cap * dI
            lam = target
            r = b - op.cols_mv(sup, x[sup])
            c = op.rmv(r)
            log(it, lam, float(np.linalg.norm(r)))
            if watch is not None:
                watch(x.copy(), list(sup), lam, c.copy(), R.copy())
            done = True
            break
        remove = gm <= gp + 1e-12
        gam = gm if remove else gp
        x[sup] += gam * dI
        if remove:
            pos = sup.index(im)
            x[im] = 0.0
            sup.pop(pos)
            mask[im] = False
            R = chol_drop(R, pos)
        else:
            gcol = op.gram_col(sup, ip)
            dg = float(op.gram_col([ip], ip)[0])
            try:
                R = chol_grow(R, gcol, dg)
                sup.append(ip)
            except NotPD:
                sup.append(ip)
                R = _ridge(op, sup, notes)
            mask[ip] = True
        r = b - op.cols_mv(sup, x[sup])
        c = op.rmv(r)
        lam_step = lam - gam
        lam_emp = float(np.max(np.abs(c)))
        if abs(lam_emp - lam_step) <= 1e-9 * max(lam_step, 1e-30) or not sup:
            lam = lam_step
        else:
            lam = lam_emp
        log(it, lam, float(np.linalg.norm(r)))
        if watch is not None:
            watch(x.copy(), list(sup), lam, c.copy(), R.copy())
        if lam <= floor:
            done = True
            break
    return Outcome(x, it, done, trace, tuple(notes)), lam


# ----------------------------------------------------------------------------
# PDIPA: primal-dual interior point on the split LP (pdipa.py:1-185)
# ----------------------------------------------------------------------------

PD_BOUNDARY = 0.99      # pdipa.py:19
PD_SIGMA = 0.1          # pdipa.py:20
PD_FEAS = 1e-8          # pdipa.py:21
PD_GAP = 1e-6           # pdipa.py:22


def pd_boundary(v, dv):
    """Damped step to the boundary of v > 0 (pdipa.py:35-40)."""
    neg = dv < 0
    if not np.any(neg):
        return 1.0
    return min(1.0, PD_BOUNDARY * float(np.min(-v[neg] / dv[neg])))


def pd_factor(M):
    """Cholesky with one jitter retry (pdipa.py:43-52) -> upper factor."""
    try:
        return chol_upper(M)
    except NotPD:
        jit = 1e-12 * max(np.trace(M) / M.shape[0], 1.0)
        try:
            return chol_upper(M + jit * np.eye(M.shape[0]))
        except NotPD as exc:
            raise IllConditioned("weighted normal matrix is singular") from exc


def pd_eliminate(x, z, rp, rd, rc, ext_mv, ext_rmv, M):
    """Eliminate dz then dx (pdipa.py:55-62)."""
    w = x / z
    rhs = rp - ext_mv(rc / z - w * rd)
    dy = chol_solve(pd_factor(M), rhs)
    dz = rd - ext_rmv(dy)
    dx = rc / z - w * dz
    return dx, dy, dz


def pd_newton(x, y, z, A_ext, b, mu_hat, c=None):
    """Newton direction with the 1e-8 residual contract (pdipa.py:65-94)."""
    A_ext = np.asarray(A_ext, dtype=np.float64)
    if c is None:
        c = np.ones(x.shape[0])
    rp = b - A_ext @ x
    rd = c - A_ext.T @ y - z
    rc = mu_hat - x * z
    M = (A_ext * (x / z)) @ A_ext.T
    dx, dy, dz = pd_eliminate(x, z, rp, rd, rc, lambda u: A_ext @ u, lambda v: A_ext.T @ v, M)
    scale = max(1.0, np.linalg.norm(rp), np.linalg.norm(rd), np.linalg.norm(rc))
    ok = (np.linalg.norm(A_ext @ dx - rp) <= 1e-8 * scale
          and np.linalg.norm(A_ext.T @ dy + dz - rd) <= 1e-8 * scale
          and np.linalg.norm(z * dx + x * dz - rc) <= 1e-8 * scale)
    if not ok or not (np.all(np.isfinite(dx)) and np.all(np.isfinite(dy)) and np.all(np.isfinite(dz))):
        raise IllConditioned("Newton system residual did not close")
    return dx, dy, dz


def pdipa(A, b, tol=1e-6, max_iter=5000, stop=None, gt=None, watch=None):
    """min ||x||_1 s.t. A x = b as the LP min 1'v, [A, -A] v = b, v >= 0
    (pdipa.py:97-185).  Returns Outcome with x = v[:n] - v[n:]."""
    op = as_op(A)
    b = np.asarray(b, dtype=np.float64)
    d, n = op.shape
    if np.linalg.norm(b) == 0.0:
        return Outcome(np.zeros(n), 0, True, [(0, 0.0, 0.0, 0)], ())
    nn = 2 * n
    c = np.ones(nn)
    x = np.ones(nn)
    y = np.zeros(d)
    z = np.ones(nn)
    mu = float(x @ z) / nn
    b_scale = max(1.0, float(np.linalg.norm(b)))
    c_scale = 1.0 + np.sqrt(nn)
    gap_tol = min(tol, PD_GAP)
    ext_mv = lambda u: op.mv(u[:n] - u[n:])
    def ext_rmv(v):
        t = op.rmv(v)
        return np.concatenate([t, -t])
    trace, notes = [], []
    conv = False
    it = 0
    while it < max_iter:
        rp = b - ext_mv(x)
        rd = c - ext_rmv(y) - z
        obj = float(c @ x)
        gap = obj - float(b @ y)
        trace.append((it, obj, float(np.linalg.norm(rp)), count_support(x[:n] - x[n:])))
        if (np.linalg.norm(rp) <= PD_FEAS * b_scale and np.linalg.norm(rd) <= PD_FEAS * c_scale
                and gap <= gap_tol * (1.0 + abs(obj))):
            conv = True
            break
        it += 1
        rc = PD_SIGMA * mu - x * z
        w = x / z
        M = op.wgram(w[:n] + w[n:])
        try:
            dx, dy, dz = pd_eliminate(x, z, rp, rd, rc, ext_mv, ext_rmv, M)
        except IllConditioned:
            notes.append("stopped on ill-conditioned normal matrix")
            break
        if not (np.all(np.isfinite(dx)) and np.all(np.isfinite(dy)) and np.all(np.isfinite(dz))):
            notes.append("stopped on non-finite step")
            break
        ap = pd_boundary(x, dx)
        ad = pd_boundary(z, dz)
        for _ in range(40):
            xn = x + ap * dx
            zn = z + ad * dz
            mun = float(xn @ zn) / nn
            if mun < mu:
                break
            ap *= 0.5
            ad *= 0.5
        else:
            notes.append("stopped on stalled duality measure")
            break
        x, y, z, mu = xn, y + ad * dy, zn, mun
        if watch is not None:
            watch(x.copy(), y.copy(), z.copy(), mu)
    return Outcome(x[:n] - x[n:], it, conv, trace, tuple(notes))


# ----------------------------------------------------------------------------
# CAB router (robust.py:181-220) for the first-order backends
# ----------------------------------------------------------------------------

def cab(A, b, solver, lam=None, tol=1e-6, max_iter=5000, stop=None, opts=None):
    """Cross-and-bouquet solve on [A, sI] -> (x, e, Outcome)."""
    opts = opts or {}
    ew = float(opts.get("e_weight", 1.0))
    if not ew > 0:
        raise ValueError("e_weight must be positive")
    s = 1.0 / ew
    op = Stacked(A, s)
    n = op.M.shape[1]
    b = np.ascontiguousarray(b, dtype=np.float64)
    kw = dict(tol=tol, max_iter=max_iter, stop=stop)
    if lam is None:
        lam_r = 1e-2 * float(np.max(np.abs(op.rmv(b))))
    else:
        lam_r = float(lam)
    if solver == "dalm":
        res = dalm(op, b, opts=opts, **kw)
    elif solver == "palm":
        res = palm(op, b, opts=opts, **kw)
    elif solver == "fista":
        res = fista(op, b, lam=lam, opts=opts, **kw)
    elif solver == "ist":
        res = ist(op, b, lam=lam, **kw)
    elif solver == "gp":
        res = gpsr(op, b, lam=lam_r, **kw)
    elif solver == "homotopy":
        res, _ = homotopy(op, b, lam_r, max_iter=max_iter)
    elif solver == "pdipa":
        res = pdipa(op, b, **kw)
    else:
        raise ValueError("unknown cab backend %r" % (solver,))
    w = res.x
    return w[:n], s * w[n:], res


# ----------------------------------------------------------------------------
# seeded generators (synth.py:39-148) used to rebuild inputs from seeds
# ----------------------------------------------------------------------------

def _stream(seed, k):
    return np.random.default_rng(np.random.SeedSequence((int(seed), k)))


def gaussian_dict(d, n, seed):
    """Unit-column Gaussian dictionary (synth.py:44-53)."""
    A = _stream(seed, 0).standard_normal((d, n))
    nr = np.linalg.norm(A, axis=0)
    while np.any(nr == 0.0):
        A = _stream(seed, 0).standard_normal((d, n))
        nr = np.linalg.norm(A, axis=0)
    return A / nr


def sparse_signal(n, k, seed):
    """Unit-norm k-sparse signal (synth.py:56-67)."""
    g = _stream(seed, 1)
    where = g.choice(n, size=k, replace=False)
    vals = g.standard_normal(k)
    while np.any(vals == 0.0):
        vals[vals == 0.0] = g.standard_normal(int(np.sum(vals == 0.0)))
    x = np.zeros(n)
    x[where] = vals / np.linalg.norm(vals)
    return x


def with_noise(b, sigma, seed):
    """synth.py:70-77."""
    b = np.asarray(b, dtype=np.float64)
    if sigma == 0.0:
        return b.copy()
    return b + sigma * _stream(seed, 2).standard_normal(b.shape[0])


def corrupt(b, frac, lo, hi, seed):
    """synth.py:80-99 -> (vector, mask)."""
    b = np.asarray(b, dtype=np.float64)
    d = b.shape[0]
    m = int(np.floor(frac * d))
    mask = np.zeros(d, dtype=bool)
    out = b.copy()
    if m:
        g = _stream(seed, 3)
        idx = g.choice(d, size=m, replace=False)
        mask[idx] = True
        out[idx] = g.uniform(lo, hi, size=m)
    return out, mask


def trial_seed(base, *idx):
    """synth.py:145-148."""
    ss = np.random.SeedSequence((int(base),) + tuple(int(i) for i in idx))
    return int(ss.generate_state(1, np.uint64)[0])


# ---------------------------------------------------------------- alignment
def align_palm(B, b, tol=1e-8, max_iter=5000, mu0=1.0, rho=2.0):
    """robust.py:470-515 (align_palm_solve): exact-fit multiplier method for
    min ||e||_1 s.t. b = B w + e.  Returns (w, e)."""
    B = np.asarray(B, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    R = chol_upper(B.T @ B)
    mu = float(mu0)
    bn = float(np.linalg.norm(b))
    w = chol_solve(R, B.T @ b)
    e = np.zeros(B.shape[0])
    y = np.zeros(B.shape[0])
    if bn == 0.0:
        return w, e
    it = 0
    while it < max_iter:
        for _ in range(min(100, max_iter - it)):
            it += 1
            w = chol_solve(R, B.T @ (b - e + y / mu))
            e_new = soft(b - B @ w + y / mu, 1.0 / mu)
            change = float(np.linalg.norm(e_new - e))
            e = e_new
            if change <= 1e-2 / mu * max(1.0, float(np.linalg.norm(e))):
                break
        r = b - B @ w - e
        y = y + mu * r
        if float(np.linalg.norm(r)) <= tol * bn:
            break
        mu *= rho
    return w, e

