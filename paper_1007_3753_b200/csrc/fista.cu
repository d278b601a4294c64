// fista.cu — FISTA (shrinkage.fista_solve, shrinkage.py:231-298) as ONE persistent
// cooperative launch, plus the power iteration (numerics.spectral_norm_sq,
// numerics.py:224-261) and the correlation max (model.py:128) it depends on.
//
// Per iteration (accepted on the first backtracking try) the dictionary is
// streamed twice — A x_next (panel GEMV, fused with soft-threshold + the
// backtracking reductions) and A^T r_next (panel GEMV^T, fused with the KKT /
// support reductions) — and the grid synchronises three times.  y, A y and
// A^T(A y - b) are exact linear combinations of cached products
// (SURVEY §8(d)): y = (1+m)x - m x_prev  =>  r_y = (1+m) r_x - m r_xp,
// g_y = (1+m) g_x - m g_xp.
#include "solvers_common.cuh"

namespace ell1 {

struct FistaArgs {
  DictRaw D;
  const double* b;          // ld entries, zero padded
  ell1_ctrl_t C;
  ell1_fista_opts_t O;
  GridBufs g;
  double* X[3];             // iterate ring: x, x_prev, x_next (N each)
  double* G[2];             // g_x, g_xprev
  double* Y;                // y
  double* GY;               // g_y
  double* R[3];             // r ring (ld each): r_x, r_xprev, r_next
  ell1_state_t* st;
  double* trace;
  double* x_out; double* xprev_out; double* y_out;
  int max_steps;
};

// state scalar slots
enum { S_L = 0, S_TP, S_TC, S_LAM, S_LAMBAR, S_FPREV, S_C0, S_BN, S_FY, S_LAMUSED, S_PASSES };
// rotation slots
enum { R_IX = 0, R_IXP, R_IXN, R_IGX, R_IGXP, R_IRX, R_IRXP, R_IRN };

template <class TA, bool SM>
__global__ void __launch_bounds__(NTHR, 1) fista_kernel(FistaArgs a) {
  extern __shared__ __align__(16) double smem[];
  Ctx E;
  const DictV<TA> D = dict_view<TA>(a.D);
  ctx_init(E, D.d, D.n);
  ctx_bind(E, a.g, smem);
  Src<TA, SM> PS;
  if constexpr (SM) {
    PS = load_panel<TA>(E, D, reinterpret_cast<TA*>(smem));
    E.sh = smem + a.g.panel_bytes / 8;
  } else {
    PS = global_panel<TA>(E, D);
  }
  const int64_t N = D.ncols();
  ell1_state_t* st = a.st;
  const double* b = a.b;
  const ell1_ctrl_t& C = a.C;
  const ell1_fista_opts_t& O = a.O;
  const double s_ext = D.s;

  // ---------------------------------------------------------------- state
  int phase = ((volatile ell1_state_t*)st)->phase;
  int it = 0, hist = 0;
  int ix = 0, ixp = 1, ixn = 2, igx = 0, igxp = 1, irx = 0, irxp = 1, irn = 2;
  double L = 0, tp = 1, tc = 1, lam = 0, lam_bar = 0, Fprev = 0, fy = 0, lam_used = 0;
  double passes = 0;   // dictionary panel passes (roofline accounting)
  bool done = false, conv = false;
  int status = ELL1_OK;

  auto run = [&]() {
  if (phase == 0 && O.probe) {
    // backtrack_L probe: y = x0, r_y = A y - b, g_y = A^T r_y (shrinkage.py:484-488)
    for_owned(E, D, [&](int64_t j) {
      const double v = O.x0[j];
      a.X[0][j] = v; a.X[1][j] = v; a.X[2][j] = v;
    });
    __syncthreads();
    {
      const double* xs[1] = {a.X[0]};
      panel_gemv<TA, SM, 1>(E, D, PS, xs);
    }
    if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
    double q[1] = {0.0};
    slice_reduce<1>(E, D.ld, [&](int64_t i, const double* sums) {
      double ax = sums[0];
      if (D.ext) ax = ax + s_ext * a.X[0][D.n + i];
      const double r = ax - b[i];
      a.R[0][i] = r; a.R[1][i] = r;
      q[0] += r * r;
    });
    block_reduce<1>(E, q, 0u);
    publish<1>(E, q);
    if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
    double fq[1];
    gather<1>(E, fq, 0u);
    {
      const double* rs[1] = {a.R[0]};
      double* os[1] = {a.G[0]};
      panel_gemv_t<TA, SM, 1>(E, D, PS, rs, os);
    }
    if (D.ext)
      for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) a.G[0][D.n + i] = s_ext * a.R[0][i];
    __syncthreads();
    for_owned(E, D, [&](int64_t j) { a.G[1][j] = a.G[0][j]; });
    lam_bar = lam = C.lam;
    L = O.L0;
    passes = 2;
    tp = tc = 1.0;
    fy = 0.5 * fq[0];
    phase = 1;
  } else if (phase == 0) {
    // prologue: c = D^T b, g_x = -c (gradient at x = 0), r_x = r_xp = -b
    {
      const double* rs[1] = {b};
      double* os[1] = {a.G[0]};
      panel_gemv_t<TA, SM, 1>(E, D, PS, rs, os);
    }
    double v[2] = {0.0, 0.0};   // max|c|, sum b^2 (slice)
    for_owned(E, D, [&](int64_t j) {
      const double c = (j < D.n) ? a.G[0][j] : s_ext * b[j - D.n];
      v[0] = nmax(v[0], fabs(c));
      a.G[0][j] = -c;
      a.G[1][j] = -c;
      a.X[0][j] = 0.0; a.X[1][j] = 0.0; a.X[2][j] = 0.0;
    });
    for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) {
      const double bi = b[i];
      a.R[0][i] = -bi; a.R[1][i] = -bi;
      v[1] += bi * bi;
    }
    block_reduce<2>(E, v, 1u);
    publish<2>(E, v);
    if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
    double gsum[2];
    gather<2>(E, gsum, 1u);
    const double c0 = gsum[0];
    const double bn = sqrt(gsum[1]);
    if (E.b == 0 && E.tid == 0) { st->scal[S_C0] = c0; st->scal[S_BN] = bn; }
    if (c0 == 0.0) {
      if (E.b == 0 && E.tid == 0) {
        a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = bn; a.trace[3] = 0.0;
        st->ntrace = 1;
      }
      status = ELL1_ZERO_DATA; conv = true; done = true;
      return;
    }
    passes = 1;
    lam_bar = (C.lam < 0.0) ? 1e-2 * c0 : C.lam;
    if (!(lam_bar > 0.0)) { status = ELL1_LAMBDA_NONPOS; done = true; return; }
    L = O.exact_L ? O.L_exact : O.L0;
    lam = O.continuation ? pymax(0.9 * c0, lam_bar) : lam_bar;
    tp = tc = 1.0;
    fy = 0.5 * gsum[1];
    phase = 1;
  } else {
    const volatile ell1_state_t* vs = st;
    it = vs->iterations; hist = vs->hist;
    ix = vs->rot[R_IX]; ixp = vs->rot[R_IXP]; ixn = vs->rot[R_IXN];
    igx = vs->rot[R_IGX]; igxp = vs->rot[R_IGXP];
    irx = vs->rot[R_IRX]; irxp = vs->rot[R_IRXP]; irn = vs->rot[R_IRN];
    L = vs->scal[S_L]; tp = vs->scal[S_TP]; tc = vs->scal[S_TC]; lam = vs->scal[S_LAM];
    lam_bar = vs->scal[S_LAMBAR]; Fprev = vs->scal[S_FPREV]; fy = vs->scal[S_FY];
    passes = vs->scal[S_PASSES];
  }

  {
    int steps = 0;
    const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
    const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;
    while (it < C.max_iter) {
      ++it; ++steps;
      lam_used = lam;
      const double m = (tp - 1.0) / tc;
      const double tn = fista_t_next(tc);
      const double mn = (tc - 1.0) / tn;             // momentum of the next iteration
      double* x = a.X[ix];
      double* xp = a.X[ixp];
      double* xn = a.X[ixn];
      const double* gx = a.G[igx];
      const double* gxp = a.G[igxp];
      for_owned(E, D, [&](int64_t j) {
        const double xj = x[j];
        a.Y[j] = xj + m * (xj - xp[j]);                 // shrinkage.py:270
        a.GY[j] = (1.0 + m) * gx[j] - m * gxp[j];       // = A^T(A y - b)
      });
      double S[7], Q2[2];
      double rr = 0.0, Fn = 0.0;
      for (int bt = 0;; ++bt) {
        if (bt > 100) { status = ELL1_BREAKDOWN; done = true; return; }   // shrinkage.py:203,213
        const double thr = lam / L;
        double s[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for_owned(E, D, [&](int64_t j) {
          const double yj = a.Y[j], gj = a.GY[j];
          const double u = soft1(yj - gj / L, thr);     // shrinkage.py:204
          xn[j] = u;
          const double dl = u - yj;
          s[0] += fabs(u);
          s[1] += gj * dl;
          s[2] += dl * dl;
          s[3] = nmax(s[3], fabs(u));
          if (relest) { const double xo = x[j]; const double dd = u - xo; s[4] += dd * dd; s[5] += xo * xo; }
          if (gtr) { const double e = u - C.ground_truth[j]; s[6] += e * e; }
        });
        block_reduce<7>(E, s, 1u << 3);
        publish<7>(E, s);
        {
          __syncthreads();
          const double* xs[1] = {xn};
          panel_gemv<TA, SM, 1>(E, D, PS, xs);
        }
        passes += 1;
        if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
        gather<7>(E, S, 1u << 3);
        double q[2] = {0.0, 0.0};
        const double* rx = a.R[irx];
        double* rn = a.R[irn];
        slice_reduce<1>(E, D.ld, [&](int64_t i, const double* sums) {
          double ax = sums[0];
          if (D.ext) ax = ax + s_ext * xn[D.n + i];      // robust.py:93
          const double r = ax - b[i];                     // shrinkage.py:205
          rn[i] = r;
          q[0] += r * r;
          const double ry = (1.0 + mn) * r - mn * rx[i];
          q[1] += ry * ry;
        });
        block_reduce<2>(E, q, 0u);
        publish<2>(E, q);
        if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
        gather<2>(E, Q2, 0u);
        rr = Q2[0];
        Fn = 0.5 * rr + lam * S[0];
        if (O.exact_L) break;                             // shrinkage.py:534-538
        const double Qm = fy + S[1] + 0.5 * L * S[2] + lam * S[0];
        if (Fn <= Qm + 1e-12 * pymax(1.0, fabs(Qm))) break;   // shrinkage.py:210
        L *= O.eta;
      }
      // accept: rotate rings (shrinkage.py:283-284)
      { int t = ixp; ixp = ix; ix = ixn; ixn = t; }
      { int t = irxp; irxp = irx; irx = irn; irn = t; }
      { int t = igxp; igxp = igx; igx = t; }
      tp = tc; tc = tn;
      {
        const double* rs[1] = {a.R[irx]};
        double* os[1] = {a.G[igx]};
        panel_gemv_t<TA, SM, 1>(E, D, PS, rs, os);            // g_x = A^T r_next  (shrinkage.py:285)
      }
      passes += 1;
      if (D.ext) {
        for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) a.G[igx][D.n + i] = s_ext * a.R[irx][i];
        __syncthreads();
      }
      double k5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};       // max_on, max_off, any_on, any_off, support
      {
        const double cut = 1e-10 * pymax(S[3], 1.0);   // model.py:232
        const double* xc = a.X[ix];
        const double* gc = a.G[igx];
        const double lamk = lam;
        for_owned(E, D, [&](int64_t j) {
          const double xj = xc[j];
          const double c = -gc[j];
          if (xj != 0.0) { k5[0] = nmax(k5[0], fabs(c - lamk * sgn(xj))); k5[2] = 1.0; }
          else { k5[1] = nmax(k5[1], fabs(c)); k5[3] = 1.0; }
          if (fabs(xj) > cut) k5[4] += 1.0;
        });
      }
      block_reduce<5>(E, k5, 0xFu);
      publish<5>(E, k5);
      if (!grid_sync(E)) { status = ELL1_ERR_TIMEOUT; return; }
      double K[5];
      gather<5>(E, K, 0xFu);
      double kkt = K[2] > 0.0 ? K[0] : 0.0;           // model.py:166-173
      if (K[3] > 0.0) kkt = pymax(pymax(kkt, K[1] - lam), 0.0);
      if (E.b == 0 && E.tid == 0) {
        double* tr = a.trace + (size_t)(it - 1) * 4;
        tr[0] = (double)it; tr[1] = Fn; tr[2] = sqrt(rr); tr[3] = K[4];
      }
      hist = hist < 2 ? hist + 1 : 2;
      if (lam == lam_bar && kkt <= C.tol * lam_bar) { conv = true; done = true; break; }
      const bool fire = stop_fires(C.stop_kind, C.stop_thr, hist, Fn, Fprev, S[4], S[5], S[6],
                                   C.gt_norm, kkt);
      Fprev = Fn;
      if (fire) { conv = true; done = true; break; }
      lam = pymax(O.beta * lam, lam_bar);              // shrinkage.py:297
      fy = 0.5 * Q2[1];
      if (a.max_steps > 0 && steps >= a.max_steps && it < C.max_iter) break;
    }
    if (it >= C.max_iter) done = true;
    if (!done) status = ELL1_RUNNING;
  }
  };
  run();

  // outputs (owned columns) and state (CTA 0)
  if (status != ELL1_ERR_TIMEOUT) {
    const double* x = a.X[ix];
    const double* xp = a.X[ixp];
    for_owned(E, D, [&](int64_t j) {
      a.x_out[j] = x[j];
      if (a.xprev_out) a.xprev_out[j] = xp[j];
      if (a.y_out) a.y_out[j] = a.Y[j];
    });
  }
  if (E.b == 0 && E.tid == 0) {
    st->status = status;
    st->phase = (status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = it;
    st->converged = conv ? 1 : 0;
    st->hist = hist;
    if (status != ELL1_ZERO_DATA) st->ntrace = it;
    st->rot[R_IX] = ix; st->rot[R_IXP] = ixp; st->rot[R_IXN] = ixn;
    st->rot[R_IGX] = igx; st->rot[R_IGXP] = igxp;
    st->rot[R_IRX] = irx; st->rot[R_IRXP] = irxp; st->rot[R_IRN] = irn;
    st->scal[S_L] = L; st->scal[S_TP] = tp; st->scal[S_TC] = tc; st->scal[S_LAM] = lam;
    st->scal[S_LAMBAR] = lam_bar; st->scal[S_FPREV] = Fprev; st->scal[S_FY] = fy;
    st->scal[S_LAMUSED] = lam_used;
    st->scal[S_PASSES] = passes;
  }
}

// ---------------------------------------------------------------------------
// correlation max: out = {max_j |(D^T b)_j|, ||b||}
struct CorrArgs {
  DictRaw D;
  const double* b;
  double* tmp;      // N
  double* out;
  GridBufs g;
};

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) corr_kernel(CorrArgs a) {
  extern __shared__ double smem[];
  Ctx E;
  const DictV<TA> D = dict_view<TA>(a.D);
  ctx_init(E, D.d, D.n);
  ctx_bind(E, a.g, smem);
  {
    const double* rs[1] = {a.b};
    double* os[1] = {a.tmp};
    panel_gemv_t<TA, false, 1>(E, D, global_panel<TA>(E, D), rs, os);
  }
  double v[2] = {0.0, 0.0};
  for_owned(E, D, [&](int64_t j) {
    const double c = (j < D.n) ? a.tmp[j] : D.s * a.b[j - D.n];
    v[0] = nmax(v[0], fabs(c));
  });
  for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) v[1] += a.b[i] * a.b[i];
  block_reduce<2>(E, v, 1u);
  publish<2>(E, v);
  if (!grid_sync(E)) return;
  double o[2];
  gather<2>(E, o, 1u);
  if (E.b == 0 && E.tid == 0) { a.out[0] = o[0]; a.out[1] = sqrt(o[1]); }
}

// ---------------------------------------------------------------------------
// power iteration on the smaller Gram side of the PLAIN dictionary A
struct PowerArgs {
  DictRaw D;            // ext ignored
  const double* v0;     // start vector(s), dim each, normalised
  int nredraw;
  double tol;
  int max_iter;
  double* V[2];         // ld (d-side) or n (n-side)
  double* W;            // d-side: w (ld); n-side: u = A v (ld)
  double* U;            // n-side scratch: A^T(.) (n) / d-side: A^T v (n)
  double* out;
  GridBufs g;
};

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) power_kernel(PowerArgs a) {
  extern __shared__ double smem[];
  Ctx E;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  ctx_init(E, D.d, D.n);
  ctx_bind(E, a.g, smem);
  const bool dside = D.d <= D.n;
  const int64_t dim = dside ? D.d : D.n;
  int iv = 0, redraw = 0, k = 0;
  double theta = 0.0;
  // load v0
  if (dside) {
    for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) a.V[0][i] = a.v0[i];
  } else {
    for (int64_t j = E.c0 + E.tid; j < E.c1; j += NTHR) a.V[0][j] = a.v0[j];
  }
  if (!grid_sync(E)) return;
  for (k = 0; k < a.max_iter; ++k) {
    double* v = a.V[iv];
    double* vn = a.V[1 - iv];
    double T[2], R2[1];
    if (dside) {
      {
        const double* rs[1] = {v};
        double* os[1] = {a.U};
        panel_gemv_t<TA, false, 1>(E, D, global_panel<TA>(E, D), rs, os);           // u = A^T v
        const double* xs[1] = {a.U};
        panel_gemv<TA, false, 1>(E, D, global_panel<TA>(E, D), xs);                 // partial A u
      }
      if (!grid_sync(E)) return;
      double q[2] = {0.0, 0.0};
      slice_reduce<1>(E, D.ld, [&](int64_t i, const double* sums) {
        const double w = sums[0];
        a.W[i] = w;
        q[0] += v[i] * w;
        q[1] += w * w;
      });
      block_reduce<2>(E, q, 0u);
      publish<2>(E, q);
      if (!grid_sync(E)) return;
      gather<2>(E, T, 0u);
      theta = T[0];
      const double nw = sqrt(T[1]);
      double e[1] = {0.0};
      for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) {
        const double w = a.W[i];
        const double r = w - theta * v[i];
        e[0] += r * r;
        vn[i] = w / nw;                                // speculative next iterate
      }
      block_reduce<1>(E, e, 0u);
      publish<1>(E, e);
      if (!grid_sync(E)) return;
      gather<1>(E, R2, 0u);
      if (sqrt(R2[0]) <= a.tol * pymax(theta, 2.2250738585072014e-308)) break;
      if (nw == 0.0) {
        if (redraw >= a.nredraw) break;
        ++redraw;
        for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) vn[i] = a.v0[redraw * dim + i];
        if (!grid_sync(E)) return;
      }
    } else {
      {
        const double* xs[1] = {v};
        panel_gemv<TA, false, 1>(E, D, global_panel<TA>(E, D), xs);                 // partial A v
      }
      if (!grid_sync(E)) return;
      slice_reduce<1>(E, D.ld, [&](int64_t i, const double* sums) { a.W[i] = sums[0]; });
      if (!grid_sync(E)) return;
      {
        const double* rs[1] = {a.W};
        double* os[1] = {a.U};
        panel_gemv_t<TA, false, 1>(E, D, global_panel<TA>(E, D), rs, os);           // w = A^T A v (panel)
      }
      double q[2] = {0.0, 0.0};
      for (int64_t j = E.c0 + E.tid; j < E.c1; j += NTHR) {
        const double w = a.U[j];
        q[0] += v[j] * w;
        q[1] += w * w;
      }
      block_reduce<2>(E, q, 0u);
      publish<2>(E, q);
      if (!grid_sync(E)) return;
      gather<2>(E, T, 0u);
      theta = T[0];
      const double nw = sqrt(T[1]);
      double e[1] = {0.0};
      for (int64_t j = E.c0 + E.tid; j < E.c1; j += NTHR) {
        const double w = a.U[j];
        const double r = w - theta * v[j];
        e[0] += r * r;
        vn[j] = w / nw;
      }
      block_reduce<1>(E, e, 0u);
      publish<1>(E, e);
      if (!grid_sync(E)) return;
      gather<1>(E, R2, 0u);
      if (sqrt(R2[0]) <= a.tol * pymax(theta, 2.2250738585072014e-308)) break;
      if (nw == 0.0) {
        if (redraw >= a.nredraw) break;
        ++redraw;
        for (int64_t j = E.c0 + E.tid; j < E.c1; j += NTHR) vn[j] = a.v0[redraw * dim + j];
      }
    }
    iv = 1 - iv;
  }
  if (E.b == 0 && E.tid == 0) { a.out[0] = theta; a.out[1] = (double)(k < a.max_iter ? k + 1 : k); }
}

}  // namespace ell1

// ============================================================================ host
using namespace ell1;

static DictRaw to_raw(const ell1_dict_t* D) {
  DictRaw r;
  r.A = D->A; r.dtype = D->dtype; r.ext = D->ext; r.d = D->d; r.n = D->n; r.ld = D->ld;
  r.s = D->ext_scale;
  return r;
}

static bool dict_ok(const ell1_dict_t* D) {
  return D && D->A && D->d >= 1 && D->n >= 1 && D->ld >= D->d && D->ld % 32 == 0 &&
         (D->dtype == ELL1_F64 || D->dtype == ELL1_F32);
}

static int64_t ncols_of(const ell1_dict_t* D) { return D->n + (D->ext ? D->d : 0); }

extern "C" size_t ell1_fista_workspace(const ell1_dict_t* D, const ell1_ctrl_t* C, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  (void)C;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  size_t b = grid_bytes(nb, D->ld);
  b += 7 * align_up(N * 8, 256) + 3 * align_up(D->ld * 8, 256) + 4096;
  return b;
}

extern "C" int ell1_fista(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                          const ell1_fista_opts_t* O, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !b || !C || !O || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (C->max_iter < 1) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  const int64_t N = ncols_of(D);
  FistaArgs a;
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.O = *O;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->ld)) return ELL1_ERR_ARG;
  for (int k = 0; k < 3; ++k) a.X[k] = cv.take<double>(N);
  for (int k = 0; k < 2; ++k) a.G[k] = cv.take<double>(N);
  a.Y = cv.take<double>(N);
  a.GY = cv.take<double>(N);
  for (int k = 0; k < 3; ++k) a.R[k] = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x; a.xprev_out = io->x_prev; a.y_out = io->y;
  a.max_steps = io->max_steps;
  cudaStream_t s = (cudaStream_t)stream;
  const SmemPlan sp = plan_smem(a.D, nb, 1, io->max_steps <= 0, 7);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  // padding rows of the residual ring must read as zero (never written by the kernel)
  if (D->ld > D->d)
    for (int k = 0; k < 3; ++k)
      if (cudaMemsetAsync(a.R[k] + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  int rc;
  if (D->dtype == ELL1_F64)
    rc = sp.resident ? coop_launch(fista_kernel<double, true>, nb, sp.bytes, s, a, a.g.bar)
                     : coop_launch(fista_kernel<double, false>, nb, sp.bytes, s, a, a.g.bar);
  else
    rc = sp.resident ? coop_launch(fista_kernel<float, true>, nb, sp.bytes, s, a, a.g.bar)
                     : coop_launch(fista_kernel<float, false>, nb, sp.bytes, s, a, a.g.bar);
  return rc;
}

extern "C" size_t ell1_correlation_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, 32) + align_up(ncols_of(D) * 8, 256) + 1024;
}

extern "C" int ell1_correlation_max(const ell1_dict_t* D, const double* b, double* out,
                                    void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !b || !out) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, 0);
  CorrArgs a;
  a.D = to_raw(D);
  a.b = b;
  a.out = out;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, 32)) return ELL1_ERR_ARG;
  a.tmp = cv.take<double>(ncols_of(D));
  if (!cv.ok) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 1, false);
  const size_t smem = sp.bytes;
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return (D->dtype == ELL1_F64) ? coop_launch(corr_kernel<double>, nb, smem, s, a, a.g.bar)
                                : coop_launch(corr_kernel<float>, nb, smem, s, a, a.g.bar);
}

extern "C" size_t ell1_power_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  const int64_t m = D->ld > D->n ? D->ld : D->n;
  return grid_bytes(nb, D->ld) + 3 * align_up(m * 8, 256) + align_up(D->n * 8, 256) + 2048;
}

extern "C" int ell1_spectral_norm_sq(const ell1_dict_t* D, const double* v0, int32_t nredraw,
                                     double tol, int32_t max_iter, double* out, void* ws,
                                     size_t wsb, void* stream) {
  if (!dict_ok(D) || !v0 || !out || max_iter < 0) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, 0);
  PowerArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.v0 = v0; a.nredraw = nredraw; a.tol = tol; a.max_iter = max_iter; a.out = out;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->ld)) return ELL1_ERR_ARG;
  const int64_t m = D->ld > D->n ? D->ld : D->n;
  a.V[0] = cv.take<double>(m);
  a.V[1] = cv.take<double>(m);
  a.W = cv.take<double>(m);
  a.U = cv.take<double>(D->n);
  if (!cv.ok) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(a.V[0], 0, m * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaMemsetAsync(a.V[1], 0, m * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaMemsetAsync(a.W, 0, m * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  const SmemPlan sp = plan_smem(a.D, nb, 1, false);
  const size_t smem = sp.bytes;
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  return (D->dtype == ELL1_F64) ? coop_launch(power_kernel<double>, nb, smem, s, a, a.g.bar)
                                : coop_launch(power_kernel<float>, nb, smem, s, a, a.g.bar);
}
