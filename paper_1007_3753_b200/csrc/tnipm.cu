// tnipm.cu — truncated-Newton log-barrier interior point
// (gradient_projection.tnipm_solve, gradient_projection.py:218-339) with the
// diagonally preconditioned CG inner solve (numerics.pcg_solve,
// numerics.py:164-221) on the device, as one persistent cooperative launch.
//
// PCG matvec op(p) = t A^T(A p) + d_red p: one panel-GEMV round for A p, a
// local panel GEMV^T, and p'op(p) = t ||A p||^2 + sum d_red p^2 folded into the
// replication barrier (3 grid barriers per CG step).
#include "solvers_common.cuh"

namespace ell1 {

struct TnipmArgs {
  DictRaw D;
  const double* b;
  ell1_ctrl_t C;
  double lam, pcg_tol;
  int pcg_cap;              // <= 0: dimension (numerics.py:185-186)
  GridBufs g;
  double* Xg[2];            // backing: x, u (resume)
  double* Rv;               // replicated r = A x - b (ld)
  double* APd;              // replicated A p / scratch (ld)
  double* ADX;              // slice-owned A dx (ld)
  ell1_state_t* st;
  double* trace;
  double* x_out; double* u_out;
  int max_steps;
  int rc;
  int wmax;
  unsigned long long* prof;
};

enum { T_T = 0, T_FPREV, T_TUSED, T_PASSES };
constexpr int TN_OV = 18;

struct TnV {
  double t, t_used, Fprev, passes, rr, l1, top, obj, bn;
  double rhsn, rz, best_res, alpha, pap, res, s, dec, Ft;
  double S[12];
  int it, hist, steps, conv, status, quit, phase, ntr, capped, cgk, cgconv, acc, tries, done, trunc, cgs;
};

#define T0 if (threadIdx.x == 0)

template <class TA>
__device__ __forceinline__ void tnipm_body(const TnipmArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ TnV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + TN_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.steps = 0; V.done = 0;
    V.it = 0; V.hist = 0; V.Fprev = 0; V.passes = 0; V.ntr = 0; V.capped = 0; V.t = 1.0 / a.lam;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist; V.ntr = st->ntrace; V.capped = st->rot[0];
      V.t = st->scal[T_T]; V.Fprev = st->scal[T_FPREV]; V.passes = st->scal[T_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, reinterpret_cast<TA*>(smem), a.rc);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const double* b = a.b;
  const double s_ext = D.s;
  const double lam = a.lam;
  const double nn = (double)(D.n + (D.ext ? D.d : 0));
  auto OV = [&](int r) { return ov + r * Wm; };
  double *X = OV(0), *U = OV(1), *AR = OV(2), *DX = OV(3), *DU = OV(4), *P = OV(5);
  double *RC = OV(6), *ZC = OV(7), *XC = OV(8), *BX = OV(9), *AP = OV(10), *DRED = OV(11);
  double *DSUM = OV(12), *DDIF = OV(13), *GX = OV(14), *GU = OV(15), *CSQ = OV(16), *XH = OV(17);
  const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;
  const int cgcap = a.pcg_cap > 0 ? a.pcg_cap : (int)nn;

  // column norms^2 (preconditioner, gradient_projection.py:246)
  for (int jl = wpx(); jl < E.w; jl += NWARP) {
    double s = 0.0;
    const TA* col = PN.gl + (int64_t)jl * D.ld;
    for (int64_t i = lnx(); i < D.ld; i += 32) { const double v = (double)col[i]; s += v * v; }
    s = warp_sum(s);
    if (lnx() == 0) CSQ[jl] = s;
  }
  for (int k = E.w + tix(); k < E.W; k += NTHR) CSQ[k] = s_ext * s_ext;

  if (V.phase == 0) {
    {
      const double* rs[1] = {b};
      double* os[1] = {AR};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    double v[2] = {0.0, 0.0};
    for_owned(E, [&](int k) {
      const double c = (k < E.w) ? AR[k] : s_ext * b[E.r0 + (k - E.w)];
      v[0] = nmax(v[0], fabs(c));
      X[k] = 0.0; U[k] = 1.0; XH[k] = 0.0;
    });
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) v[1] += b[i] * b[i];
    if (!allreduce<2>(E, v, 1u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    T0 {
      if (v[0] == 0.0) {                                    // gradient_projection.py:240-242
        if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = sqrt(v[1]); a.trace[3] = 0.0; a.st->ntrace = 1; }
        V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
      }
      V.phase = 1;
    }
    __syncthreads();
    if (V.quit) goto out;
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      X[k] = a.Xg[0][j]; U[k] = a.Xg[1][j]; XH[k] = X[k];
    });
    __syncthreads();
  }

  while (true) {
    T0 V.quit = V.it >= C.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps);
    __syncthreads();
    if (V.quit) break;
    // ---------------- r = A x - b, A^T r, objective, trace (gradient_projection.py:257-261)
    {
      double s2[2] = {0.0, 0.0};                           // l1, max|x|
      for_owned(E, [&](int k) { s2[0] += fabs(X[k]); s2[1] = nmax(s2[1], fabs(X[k])); });
      block_reduce<2>(E, s2, 0x2u);
      publish<2>(E, s2);
      const double* xs[1] = {X};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double S2[2];
      double q[1] = {0.0};
      const double* aux[1] = {b};
      gather_slice<2, 1, 1>(E, S2, 0x2u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
        double ax = sums[0];
        if (D.ext) ax = ax + s_ext * X[E.w + (int)(i - E.r0)];
        const double r = ax - au[0];
        a.Rv[i] = r;
        q[0] += r * r;
      });
      T0 { V.l1 = S2[0]; V.top = S2[1]; V.passes += 1; }
      if (!allreduce<1>(E, q, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 { V.rr = q[0]; V.obj = 0.5 * q[0] + lam * V.l1; }
    }
    {
      const double* rs[1] = {a.Rv};
      double* os[1] = {AR};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    {
      // support of the truncated x (gradient_projection.py:195-206, model.py:227-233),
      // KKT of x for the stopping rule, relative-estimate / ground-truth terms
      const double top = V.top;
      const double cut_t = 1e-7 * top;
      const double cut_s = 1e-10 * pymax(top, 1.0);
      double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for_owned(E, [&](int k) {
        if (k >= E.w) AR[k] = s_ext * a.Rv[E.r0 + (k - E.w)];
        const double xk = X[k];
        if ((top > 0.0 ? fabs(xk) > cut_t : true) && fabs(xk) > cut_s) s[0] += 1.0;
        const double c = -AR[k];
        if (xk != 0.0) { s[1] = nmax(s[1], fabs(c - lam * sgn(xk))); s[3] = 1.0; }
        else { s[2] = nmax(s[2], fabs(c)); s[4] = 1.0; }
        if (relest) { const double dd = xk - XH[k]; s[5] += dd * dd; s[6] += XH[k] * XH[k]; }
        if (gtr) { const double e = xk - C.ground_truth[gcol(E, D.n, k)]; s[7] += e * e; }
        XH[k] = xk;
      });
      if (!allreduce<8>(E, s, 0x1Eu)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 {
        if (E.b == 0) {
          double* tr = a.trace + (size_t)V.ntr * 4;
          tr[0] = (double)V.it; tr[1] = V.obj; tr[2] = sqrt(V.rr); tr[3] = s[0];
        }
        V.ntr++;
        V.trunc = 0;
        if (C.stop_kind != ELL1_STOP_NONE) {                 // gradient_projection.py:262-268
          double kkt = s[3] > 0.0 ? s[1] : 0.0;
          if (s[4] > 0.0) kkt = pymax(pymax(kkt, s[2] - lam), 0.0);
          V.hist = V.hist < 2 ? V.hist + 1 : 2;
          if (stop_fires(C.stop_kind, C.stop_thr, V.hist, V.obj, V.Fprev, s[5], s[6], s[7], C.gt_norm, kkt)) {
            V.conv = 1; V.done = 1; V.trunc = 1;
          }
          V.Fprev = V.obj;
        }
      }
      __syncthreads();
      if (V.done) break;
    }
    // ---------------- duality-gap exit (gradient_projection.py:269-275)
    if (2.0 * nn / V.t <= C.tol * (1.0 + V.obj)) {
      const double cut_t = 1e-7 * V.top;
      const double top = V.top;
      for_owned(E, [&](int k) { DX[k] = (top > 0.0 && fabs(X[k]) <= cut_t) ? 0.0 : X[k]; });
      {
        const double* xs[1] = {DX};
        panel_gemv<TA, 1>(E, D, PN, xs);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        const double* aux[1] = {b};
        gather_slice<0, 1, 1>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          double ax = sums[0];
          if (D.ext) ax = ax + s_ext * DX[E.w + (int)(i - E.r0)];
          a.APd[i] = au[0] - ax;                            // b - A xt
        });
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        const double* rs[1] = {a.APd};
        double* os[1] = {DU};
        panel_gemv_t<TA, 1>(E, D, PN, rs, os);
      }
      __syncthreads();
      double k4[4] = {0, 0, 0, 0};
      for_owned(E, [&](int k) {
        if (k >= E.w) DU[k] = s_ext * a.APd[E.r0 + (k - E.w)];
        const double xk = DX[k], c = DU[k];
        if (xk != 0.0) { k4[0] = nmax(k4[0], fabs(c - lam * sgn(xk))); k4[2] = 1.0; }
        else { k4[1] = nmax(k4[1], fabs(c)); k4[3] = 1.0; }
      });
      if (!allreduce<4>(E, k4, 0xFu)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 {
        V.passes += 2;
        double kkt = k4[2] > 0.0 ? k4[0] : 0.0;
        if (k4[3] > 0.0) kkt = pymax(pymax(kkt, k4[1] - lam), 0.0);
        if (kkt <= C.tol * lam) { V.conv = 1; V.done = 1; }
      }
      __syncthreads();
      if (V.done) {
        for_owned(E, [&](int k) { X[k] = DX[k]; });
        break;
      }
    }
    // ---------------- Newton system (gradient_projection.py:276-289)
    {
      const double t = V.t;
      double s2[2] = {0.0, 0.0};                           // ||rhs||^2, r.z
      for_owned(E, [&](int k) {
        const double up = U[k] + X[k], um = U[k] - X[k];
        const double p = 1.0 / up, q = 1.0 / um;
        const double gx = t * AR[k] + (q - p);
        const double gu = t * lam - p - q;
        const double pp = p * p, qq = q * q;
        const double dsum = pp + qq, ddif = pp - qq;
        const double dred = 4.0 * pp * qq / dsum;
        GX[k] = gx; GU[k] = gu; DSUM[k] = dsum; DDIF[k] = ddif; DRED[k] = dred;
        const double rhs = -gx + ddif * (gu / dsum);
        const double dg = t * CSQ[k] + dred;                 // preconditioner diagonal
        RC[k] = rhs;
        const double z = rhs / dg;
        ZC[k] = z; P[k] = z; XC[k] = 0.0; BX[k] = 0.0;
        s2[0] += rhs * rhs;
        s2[1] += rhs * z;
      });
      if (!allreduce<2>(E, s2, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 { V.rhsn = sqrt(s2[0]); V.rz = s2[1]; V.best_res = V.rhsn; V.cgk = 0; V.cgconv = 0; V.cgs = 0; }
      __syncthreads();
    }
    // ---------------- PCG (numerics.py:188-221)
    if (V.rhsn == 0.0) {
      T0 V.cgconv = 1;
    } else {
      while (true) {
        T0 { V.cgk++; }
        __syncthreads();
        if (V.cgk > cgcap) break;
        {
          double s1[1] = {0.0};
          for_owned(E, [&](int k) { s1[0] += DRED[k] * P[k] * P[k]; });
          block_reduce<1>(E, s1, 0u);
          publish<1>(E, s1);
          const double* xs[1] = {P};
          panel_gemv<TA, 1>(E, D, PN, xs);
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          double S1[1];
          double q[1] = {0.0};
          gather_slice<1, 1, 0>(E, S1, 0u, D.ld, {nullptr}, [&](int64_t i, const double* sums, const double*) {
            double ap = sums[0];
            if (D.ext) ap = ap + s_ext * P[E.w + (int)(i - E.r0)];
            a.APd[i] = ap;
            q[0] += ap * ap;
          });
          if (!allreduce<1>(E, q, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          T0 {
            V.passes += 1;
            V.pap = V.t * q[0] + S1[0];                      // p'(t A^T A + D) p
            if (!isfinite(V.pap)) { V.status = ELL1_BREAKDOWN; V.cgs = 1; }
            else if (V.pap <= 0.0) V.cgs = 2;                // indefinite: best iterate
            else V.alpha = V.rz / V.pap;
          }
          __syncthreads();
          if (V.cgs) break;
        }
        {
          const double* rs[1] = {a.APd};
          double* os[1] = {AP};
          panel_gemv_t<TA, 1>(E, D, PN, rs, os);
        }
        __syncthreads();
        {
          const double t = V.t, alpha = V.alpha;
          double s2[2] = {0.0, 0.0};                         // ||r||^2, r.z
          for_owned(E, [&](int k) {
            if (k >= E.w) AP[k] = s_ext * a.APd[E.r0 + (k - E.w)];
            const double apk = t * AP[k] + DRED[k] * P[k];
            XC[k] = XC[k] + alpha * P[k];
            const double r = RC[k] - alpha * apk;
            RC[k] = r;
            const double z = r / (t * CSQ[k] + DRED[k]);
            ZC[k] = z;
            s2[0] += r * r;
            s2[1] += r * z;
          });
          if (!allreduce<2>(E, s2, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          T0 {
            V.passes += 1;
            V.res = sqrt(s2[0]);
            if (!isfinite(V.res)) { V.status = ELL1_BREAKDOWN; V.cgs = 1; }
            else {
              V.S[0] = V.res < V.best_res ? 1.0 : 0.0;
              if (V.res < V.best_res) V.best_res = V.res;
              if (V.res <= a.pcg_tol * V.rhsn) { V.cgconv = 1; V.cgs = 3; }
              else { V.S[1] = s2[1] / V.rz; V.rz = s2[1]; }
            }
          }
          __syncthreads();
          if (V.status != ELL1_OK) goto out;
          const bool better = V.S[0] != 0.0;
          const double beta = V.S[1];
          const bool fin = V.cgs == 3;
          for_owned(E, [&](int k) {
            if (better) BX[k] = XC[k];
            if (!fin) P[k] = ZC[k] + beta * P[k];
          });
          if (fin) break;
        }
      }
      if (V.status != ELL1_OK) goto out;
    }
    {
      // dx = converged x, else best iterate
      const bool conv_cg = V.cgconv != 0;
      __syncthreads();
      T0 if (!conv_cg) V.capped++;
      for_owned(E, [&](int k) { DX[k] = conv_cg ? XC[k] : BX[k]; });
      if (V.rhsn == 0.0) for_owned(E, [&](int k) { DX[k] = 0.0; });
    }
    // ---------------- du, decrement, interior step bound, barrier value (:290-301)
    {
      const double t = V.t;
      double s[8] = {0, 0, -INFINITY, -INFINITY, 0, 0, 0, 0};   // dec, -, -min1, -min2, sum u, sum log up, sum log um, bad
      double mn[2] = {INFINITY, INFINITY};
      for_owned(E, [&](int k) {
        const double dx = DX[k];
        const double du = -(GU[k] + DDIF[k] * dx) / DSUM[k];
        DU[k] = du;
        s[0] += GX[k] * dx + GU[k] * du;
        const double up = U[k] + X[k], um = U[k] - X[k];
        const double dup = du + dx, dum = du - dx;
        if (dup < 0.0) s[2] = nmax(s[2], -(up / -dup));
        if (dum < 0.0) s[3] = nmax(s[3], -(um / -dum));
        s[4] += U[k];
        s[5] += log(up);
        s[6] += log(um);
        mn[0] = fmin(mn[0], up); mn[1] = fmin(mn[1], um);
      });
      s[1] = -mn[0];
      s[7] = -mn[1];
      (void)t;
      if (!allreduce<8>(E, s, 0x8Eu)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 {
        V.dec = -s[0];
        double st = 1.0;
        if (s[2] > -INFINITY) st = fmin(st, 0.99 * (-s[2]));
        if (s[3] > -INFINITY) st = fmin(st, 0.99 * (-s[3]));
        V.s = st;
        const bool inside = (-s[1]) > 0.0 && (-s[7]) > 0.0;
        V.Ft = inside ? V.t * (0.5 * V.rr + lam * s[4]) - s[5] - s[6] : INFINITY;
        V.tries = 0; V.acc = 0;
      }
      __syncthreads();
    }
    {
      const double* xs[1] = {DX};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    gather_slice<0, 1, 0>(E, nullptr, 0u, D.ld, {nullptr}, [&](int64_t i, const double* sums, const double*) {
      double adx = sums[0];
      if (D.ext) adx = adx + s_ext * DX[E.w + (int)(i - E.r0)];
      a.ADX[i] = adx;
    });
    // ---------------- Armijo backtracking on the barrier (:302-315)
    while (true) {
      {
        const double s = V.s;
        double v[6] = {0, 0, 0, 0, 0, 0};                  // ||r + s Adx||^2, sum u', sum log up', sum log um', -min up', -min um'
        double m0 = INFINITY, m1 = INFINITY;
        for_owned(E, [&](int k) {
          const double xn = X[k] + s * DX[k];
          const double un = U[k] + s * DU[k];
          const double up = un + xn, um = un - xn;
          v[1] += un;
          v[2] += log(up);
          v[3] += log(um);
          m0 = fmin(m0, up); m1 = fmin(m1, um);
        });
        for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
          const double r = a.Rv[i] + s * a.ADX[i];
          v[0] += r * r;
        }
        v[4] = -m0; v[5] = -m1;
        if (!allreduce<6>(E, v, 0x30u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        T0 {
          const bool inside = (-v[4]) > 0.0 && (-v[5]) > 0.0;
          const double Fn = inside ? V.t * (0.5 * v[0] + lam * v[1]) - v[2] - v[3] : INFINITY;
          if (Fn <= V.Ft - 0.01 * V.s * V.dec) V.acc = 1;
          else { V.s *= 0.5; V.tries++; }
          if (!V.acc && V.tries > 50) { V.status = ELL1_BREAKDOWN; }
          V.passes += 0;
        }
        __syncthreads();
        if (V.status != ELL1_OK) goto out;
        if (V.acc) break;
      }
    }
    {
      const double s = V.s;
      for_owned(E, [&](int k) { X[k] = X[k] + s * DX[k]; U[k] = U[k] + s * DU[k]; });
      T0 {
        V.it++; V.steps++;
        V.t_used = V.t;
        if (V.dec <= 0.25) V.t *= 10.0;                     // :326-327
        V.passes += 1;
      }
      __syncthreads();
    }
  }
  // ---------------- truncation and final certificate (:328-337)
  if (V.status == ELL1_OK && !(V.quit && a.max_steps > 0 && V.it < C.max_iter)) {
    if (!V.conv || V.trunc) {
      double m1[1] = {0.0};
      for_owned(E, [&](int k) { m1[0] = nmax(m1[0], fabs(X[k])); });
      if (!allreduce<1>(E, m1, 1u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      const double top = m1[0];
      for_owned(E, [&](int k) { if (top > 0.0 && fabs(X[k]) <= 1e-7 * top) X[k] = 0.0; });
    }
    if (!V.conv) {
      {
        const double* xs[1] = {X};
        panel_gemv<TA, 1>(E, D, PN, xs);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      double q[2] = {0.0, 0.0};
      {
        const double* aux[1] = {b};
        gather_slice<0, 1, 1>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          double ax = sums[0];
          if (D.ext) ax = ax + s_ext * X[E.w + (int)(i - E.r0)];
          const double r = ax - au[0];
          a.APd[i] = -r;                                    // -rt = b - A x
          q[0] += r * r;
        });
      }
      for_owned(E, [&](int k) { q[1] += fabs(X[k]); });
      if (!allreduce<2>(E, q, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        const double* rs[1] = {a.APd};
        double* os[1] = {DU};
        panel_gemv_t<TA, 1>(E, D, PN, rs, os);
      }
      __syncthreads();
      double k4[4] = {0, 0, 0, 0};
      for_owned(E, [&](int k) {
        if (k >= E.w) DU[k] = s_ext * a.APd[E.r0 + (k - E.w)];
        const double xk = X[k], c = DU[k];
        if (xk != 0.0) { k4[0] = nmax(k4[0], fabs(c - lam * sgn(xk))); k4[2] = 1.0; }
        else { k4[1] = nmax(k4[1], fabs(c)); k4[3] = 1.0; }
      });
      if (!allreduce<4>(E, k4, 0xFu)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 {
        const double objt = 0.5 * q[0] + lam * q[1];
        double kkt = k4[2] > 0.0 ? k4[0] : 0.0;
        if (k4[3] > 0.0) kkt = pymax(pymax(kkt, k4[1] - lam), 0.0);
        if (2.0 * nn / V.t <= C.tol * (1.0 + objt) && kkt <= C.tol * lam) V.conv = 1;
      }
      __syncthreads();
    }
  } else if (V.status == ELL1_OK) {
    T0 V.status = ELL1_RUNNING;
    __syncthreads();
  }

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    const bool save = V.status == ELL1_RUNNING;
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = X[k];
      if (a.u_out) a.u_out[j] = U[k];
      if (save) { a.Xg[0][j] = X[k]; a.Xg[1][j] = U[k]; }
    });
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    st->hist = V.hist;
    if (V.status != ELL1_ZERO_DATA) st->ntrace = V.ntr;
    st->rot[0] = V.capped;
    st->scal[T_T] = V.t; st->scal[T_FPREV] = V.Fprev; st->scal[T_TUSED] = V.t_used;
    st->scal[T_PASSES] = V.passes;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) tnipm_kernel(const __grid_constant__ TnipmArgs a) {
  tnipm_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_tnipm_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  return grid_bytes(nb, D->d, 1) + 2 * align_up(N * 8, 256) + 3 * align_up(D->ld * 8, 256) + 4096;
}

static int tnipm_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
                          double pcg_tol, int32_t pcg_max_iter, double* u_out, const ell1_io_t* io, int nb, TnipmArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (!(lam > 0) || C->max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.lam = lam;
  a.pcg_tol = pcg_tol;
  a.pcg_cap = pcg_max_iter;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  a.Xg[0] = cv.take<double>(N); a.Xg[1] = cv.take<double>(N);
  a.Rv = cv.take<double>(D->ld); a.APd = cv.take<double>(D->ld); a.ADX = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x;
  a.u_out = u_out;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, TN_OV, 8, io->max_steps <= 0);
  if (sp.bytes > (size_t)max_smem_optin()) return ELL1_ERR_ARG;   // owned vectors must fit
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_tnipm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
                          double pcg_tol, int32_t pcg_max_iter, double* u_out, const ell1_io_t* io,
                          void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  TnipmArgs a;
  SmemPlan sp;
  const int rc0 = tnipm_setup(D, b, C, lam, pcg_tol, pcg_max_iter, u_out, io, nb, a, sp);
  if (rc0 != ELL1_OK) return rc0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->ld > D->d)
    for (double* p : {a.Rv, a.APd, a.ADX})
      if (cudaMemsetAsync(p + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(tnipm_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(tnipm_kernel<float>, nb, sp.bytes, s, a, a.g.bar);

}

namespace ell1 {
template <class TA>
struct TnipmRun {
  static __device__ void run(const TnipmArgs& a) { tnipm_body<TA>(a); }
  static __device__ void reset(const TnipmArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    zero_pad_rows(a.Rv, a.D.d, a.D.ld, lane);
    zero_pad_rows(a.APd, a.D.d, a.D.ld, lane);
    zero_pad_rows(a.ADX, a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(TnipmArgs) <= ELL1_GROUP_ARG_BYTES, "TnipmArgs too large for the group scratch");
}  // namespace ell1

int32_t ell1_tnipm_group_team_impl(const ell1_dict_t* D) {
  return dict_ok(D) ? group_team(to_raw(D), TN_OV, 8, 0) : 0;
}

extern "C" int ell1_tnipm_group(const ell1_group_t* G, const double* lam, double pcg_tol, int32_t pcg_max_iter,
                                void* stream) {
  if (!G || (G->count > 0 && !lam)) return ELL1_ERR_ARG;
  return run_group<TnipmArgs, TnipmRun>(G, TN_OV, 8, 0, [&](int i, int nb, TnipmArgs& a, SmemPlan& sp) {
    const int rc = tnipm_setup(&G->dicts[i], G->b[i], &G->ctrl[i], lam[i], pcg_tol, pcg_max_iter, nullptr,
                               &G->io[i], nb, a, sp);
    if (rc == ELL1_OK && sp.bytes > (size_t)max_smem_optin()) return (int)ELL1_ERR_ARG;
    return rc;
  }, stream);
}
