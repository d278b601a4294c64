// fista.cu — FISTA (shrinkage.fista_solve, shrinkage.py:231-298) as ONE persistent
// cooperative launch, plus the power iteration (numerics.spectral_norm_sq,
// numerics.py:224-261) and the correlation max (model.py:128) it depends on.
//
// Per iteration (accepted on the first backtracking try): the dictionary
// panel is swept twice — A x_next (panel GEMV; soft-threshold and the
// backtracking reductions fused in front of it) and A^T r_next (panel GEMV^T;
// KKT / support reductions fused behind it) — and the grid synchronises
// twice: the KKT/support reduction of iteration k rides on the first
// barrier of iteration k+1 (its convergence test is therefore applied one
// barrier late; if it fires, the speculative work of k+1 is discarded and
// iteration k is returned, exactly as the reference would).
// y, A y and A^T(A y - b) are exact linear combinations of cached products
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
  double* Xg[3];            // global backing of the owned iterate ring (resume / outputs)
  double* Gg[2];
  double* R[3];             // residual ring (ld each): r_x, r_xprev, r_next
  ell1_state_t* st;
  double* trace;
  double* x_out; double* xprev_out; double* y_out;
  int max_steps;
  int rc;                   // resident panel columns
  int wmax;                 // owned-vector stride in shared memory
  unsigned long long* prof;
};

// state scalar slots
enum { S_L = 0, S_TP, S_TC, S_LAM, S_LAMBAR, S_FPREV, S_C0, S_BN, S_FY, S_LAMUSED, S_PASSES };
// rotation slots
enum { R_IX = 0, R_IXP, R_IXN, R_IGX, R_IGXP, R_IRX, R_IRXP, R_IRN };
constexpr int FISTA_OV = 7;      // owned vectors: x ring (3), g ring (2), y, g_y

// Control state: one copy per CTA in shared memory, written by thread 0
// only (every CTA computes the same values), read by all threads after a
// block barrier.  Keeping it out of registers avoids spills, whose reloads
// would miss in L1 after every grid barrier.
struct FistaV {
  double L, tp, tc, lam, lam_bar, Fprev, fy, lam_used, passes;
  double m, tn, mn, thr, tn2, mn2, lam2, thr2;
  double f_F, f_rr, f_lam, f_s4, f_s5, f_s6;
  double cut;
  double S[12];
  double Q2[2];
  double rr, Fn;
  int it, hist, steps, pend, f_it, conv, status, stop_prev, accept, bt, quit, phase, fin;
  int ix, ixp, ixn, igx, igxp, irx, irxp, irn;
};

// finalisation of the pending iteration (trace row, convergence, stop rule);
// thread 0 only.  Returns true when the solve stops at that iteration.
__device__ bool fista_finalize(FistaV& V, const ell1_ctrl_t& C, double* trace, bool write_trace,
                               const double* K) {
  double kkt = K[2] > 0.0 ? K[0] : 0.0;              // model.py:166-173
  if (K[3] > 0.0) kkt = pymax(pymax(kkt, K[1] - V.f_lam), 0.0);
  if (write_trace) {
    double* tr = trace + (size_t)(V.f_it - 1) * 4;
    tr[0] = (double)V.f_it; tr[1] = V.f_F; tr[2] = sqrt(V.f_rr); tr[3] = K[4];
  }
  V.hist = V.hist < 2 ? V.hist + 1 : 2;
  if (V.f_lam == V.lam_bar && kkt <= C.tol * V.lam_bar) return true;   // shrinkage.py:291-293
  const bool fire = stop_fires(C.stop_kind, C.stop_thr, V.hist, V.f_F, V.Fprev, V.f_s4, V.f_s5,
                               V.f_s6, C.gt_norm, kkt);                 // shrinkage.py:294-296
  V.Fprev = V.f_F;
  return fire;
}

#define T0 if (threadIdx.x == 0)

// PROF: phase timers (tools/phase_profile.py); the production variant has none.
#define MARK(k) do { if constexpr (PROF) mark(E, k); } while (0)

template <class TA, bool PROF>
__device__ __forceinline__ void fista_body(const FistaArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ FistaV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + FISTA_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.pend = 0; V.steps = 0; V.bt = 0;
    V.stop_prev = 0; V.accept = 0;
    V.it = 0; V.hist = 0; V.passes = 0; V.Fprev = 0; V.lam_used = 0;
    V.ix = 0; V.ixp = 1; V.ixn = 2; V.igx = 0; V.igxp = 1; V.irx = 0; V.irxp = 1; V.irn = 2;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist;
      V.ix = st->rot[R_IX]; V.ixp = st->rot[R_IXP]; V.ixn = st->rot[R_IXN];
      V.igx = st->rot[R_IGX]; V.igxp = st->rot[R_IGXP];
      V.irx = st->rot[R_IRX]; V.irxp = st->rot[R_IRXP]; V.irn = st->rot[R_IRN];
      V.L = st->scal[S_L]; V.tp = st->scal[S_TP]; V.tc = st->scal[S_TC]; V.lam = st->scal[S_LAM];
      V.lam_bar = st->scal[S_LAMBAR]; V.Fprev = st->scal[S_FPREV]; V.fy = st->scal[S_FY];
      V.passes = st->scal[S_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, reinterpret_cast<TA*>(smem), a.rc);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const ell1_fista_opts_t& O = a.O;
  const double* b = a.b;
  const double s_ext = D.s;
  auto Xp = [&](int r) { return ov + r * Wm; };          // x ring
  auto Gp = [&](int r) { return ov + (3 + r) * Wm; };    // g ring
  double* Y = ov + 5 * Wm;
  double* GY = ov + 6 * Wm;

  if (V.phase == 0 && O.probe) {
    // backtrack_L probe: y = x0, r_y = A y - b, g_y = A^T r_y (shrinkage.py:484-488)
    for_owned(E, [&](int k) {
      const double v = O.x0[gcol(E, D.n, k)];
      Xp(0)[k] = v; Xp(1)[k] = v; Xp(2)[k] = v;
    });
    {
      const double* xs[1] = {Xp(0)};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double q[1] = {0.0};
      const double* aux[1] = {b};
      gather_slice<0, 1, 1>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
        double ax = sums[0];
        if (D.ext) ax = ax + s_ext * Xp(0)[E.w + (int)(i - E.r0)];
        const double r = ax - au[0];
        a.R[0][i] = r; a.R[1][i] = r;
        q[0] += r * r;
      });
      block_reduce<1>(E, q, 0u);
      publish<1>(E, q);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double fq[1];
      gather<1>(E, fq, 0u);
      const double* rs[1] = {a.R[0]};
      double* os[1] = {Gp(0)};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
      __syncthreads();
      for_owned(E, [&](int k) {
        if (k >= E.w) Gp(0)[k] = s_ext * a.R[0][E.r0 + (k - E.w)];
        Gp(1)[k] = Gp(0)[k];
      });
      T0 {
        V.lam_bar = V.lam = C.lam;
        V.L = O.L0;
        V.tp = V.tc = 1.0;
        V.fy = 0.5 * fq[0];
        V.passes = 2;
        V.phase = 1;
      }
    }
  } else if (V.phase == 0) {
    // prologue: c = D^T b, g_x = -c (gradient at x = 0), r_x = r_xp = -b
    {
      const double* rs[1] = {b};
      double* os[1] = {Gp(0)};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    {
      double v[2] = {0.0, 0.0};   // max|c|, sum b^2 (slice)
      for_owned(E, [&](int k) {
        const double c = (k < E.w) ? Gp(0)[k] : s_ext * b[E.r0 + (k - E.w)];
        v[0] = nmax(v[0], fabs(c));
        Gp(0)[k] = -c;
        Gp(1)[k] = -c;
        Xp(0)[k] = 0.0; Xp(1)[k] = 0.0; Xp(2)[k] = 0.0;
      });
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
        const double bi = b[i];
        a.R[0][i] = -bi; a.R[1][i] = -bi;
        v[1] += bi * bi;
      }
      block_reduce<2>(E, v, 1u);
      publish<2>(E, v);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double gsum[2];
      gather<2>(E, gsum, 1u);
      T0 {
        const double c0 = gsum[0];
        const double bn = sqrt(gsum[1]);
        if (E.b == 0) { a.st->scal[S_C0] = c0; a.st->scal[S_BN] = bn; }
        if (c0 == 0.0) {                                 // shrinkage.py:245-247
          if (E.b == 0) {
            a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = bn; a.trace[3] = 0.0;
            a.st->ntrace = 1;
          }
          V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
        } else {
          V.passes = 1;
          V.lam_bar = (C.lam < 0.0) ? 1e-2 * c0 : C.lam;
          if (!(V.lam_bar > 0.0)) { V.status = ELL1_LAMBDA_NONPOS; V.quit = 1; }
          V.L = O.exact_L ? O.L_exact : O.L0;
          V.lam = O.continuation ? pymax(0.9 * c0, V.lam_bar) : V.lam_bar;   // shrinkage.py:259-260
          V.tp = V.tc = 1.0;
          V.fy = 0.5 * gsum[1];
          V.phase = 1;
        }
      }
      __syncthreads();
      if (V.quit) goto out;
    }
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      for (int r = 0; r < 3; ++r) Xp(r)[k] = a.Xg[r][j];
      for (int r = 0; r < 2; ++r) Gp(r)[k] = a.Gg[r][j];
    });
  }
  __syncthreads();

  {
    const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
    const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;
    const bool tw = E.b == 0;                             // CTA 0 writes the trace
    // Per-thread partials carried into the next reduction: [0..6] the prox /
    // backtracking sums of the current trial, [7..11] the KKT / support
    // partials of the previous accepted iterate (shrinkage.py:289-293, computed
    // right after its A^T r and reduced together with the next trial's sums).
    double s12[12];
    GtPre<TA, 1> gpre;
    // thread 0: start an iteration (shrinkage.py:269-270 momentum, t sequence)
    auto begin_iter = [&]() {
      V.quit = (V.it >= C.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps));
      if (!V.quit) {
        V.it++; V.steps++; V.bt = 0; V.stop_prev = 0;   // (accept is set by every decision)
        V.m = (V.tp - 1.0) / V.tc;
        V.tn = fista_t_next(V.tc);
        V.mn = (V.tc - 1.0) / V.tn;                       // momentum of the next iteration
        V.thr = V.lam / V.L;
      }
    };
    // prox trial over the owned columns (shrinkage.py:204-208), optionally
    // forming y and g_y first (linear combinations of cached products)
    auto prox = [&](bool form_y) {
      const double L = V.L, thr = V.thr, m = V.m;
      const double* x = Xp(V.ix);
      const double* xp = Xp(V.ixp);
      const double* gx = Gp(V.igx);
      const double* gxp = Gp(V.igxp);
      double* xn = Xp(V.ixn);
      for_owned(E, [&](int k) {
        double yj, gj;
        if (form_y) {
          const double xj = x[k];
          yj = xj + m * (xj - xp[k]);                       // shrinkage.py:270
          gj = (1.0 + m) * gx[k] - m * gxp[k];              // = A^T(A y - b)
          Y[k] = yj; GY[k] = gj;
        } else {
          yj = Y[k]; gj = GY[k];
        }
        const double u = soft1(yj - gj / L, thr);           // shrinkage.py:204
        xn[k] = u;
        const double dl = u - yj;
        s12[0] += fabs(u);
        s12[1] += gj * dl;
        s12[2] += dl * dl;
        s12[3] = nmax(s12[3], fabs(u));
        if (relest) { const double xo = x[k]; const double dd = u - xo; s12[4] += dd * dd; s12[5] += xo * xo; }
        if (gtr) { const double e = u - C.ground_truth[gcol(E, D.n, k)]; s12[6] += e * e; }
      });
    };
    auto zero12 = [&]() {
#pragma unroll
      for (int k = 0; k < 12; ++k) s12[k] = 0.0;
    };
    T0 begin_iter();
    __syncthreads();
    zero12();
    if (!V.quit) prox(true);
    while (!V.quit) {
      MARK(-1);
      block_reduce_w0<12>(E, s12, (1u << 3) | (0xFu << 7));   // panel_gemv syncs before E.sh reuse
      publish<12>(E, s12);
      MARK(0);
      {
        const double* xs[1] = {Xp(V.ixn)};
        panel_gemv<TA, 1>(E, D, PN, xs);
      }
      MARK(1);
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      MARK(2);
      {
        double q[2] = {0.0, 0.0};
        const double mn = V.mn;
        const double* xn = Xp(V.ixn);
        double* rnv = a.R[V.irn];
        const double* aux[2] = {b, a.R[V.irx]};
        gather_slice<12, 1, 2, true>(E, V.S, (1u << 3) | (0xFu << 7), D.ld, aux,
                               [&](int64_t i, const double* sums, const double* au) {
          double ax = sums[0];
          if (D.ext) ax = ax + s_ext * xn[E.w + (int)(i - E.r0)];   // robust.py:93
          const double r = ax - au[0];                  // shrinkage.py:205
          rnv[i] = r;
          q[0] += r * r;
          const double ry = (1.0 + mn) * r - mn * au[1];
          q[1] += ry * ry;
        });
        MARK(3);
        T0 {
          V.passes += 1;
          V.fin = V.pend && V.bt == 0;                  // iteration it-1 is finalised now
          if (V.fin) V.pend = 0;
        }
        block_reduce<2>(E, q, 0u);
        publish<2>(E, q);
      }
      MARK(4);
      grid_arrive(E);
      // hidden behind the barrier (three threads in parallel): the trace row /
      // convergence / stop rule of iteration it-1, and the scalars iteration
      // it+1 starts with should this trial be accepted (t sequence, momenta,
      // continuation, threshold) — identical expressions, computed early
      if (tix() == 0) {
        if (V.fin && fista_finalize(V, C, a.trace, tw, V.S + 7)) V.stop_prev = 1;
      } else if (tix() == 32) {
        V.tn2 = fista_t_next(V.tn);
        V.mn2 = (V.tn - 1.0) / V.tn2;
      } else if (tix() == 64) {
        V.lam2 = pymax(O.beta * V.lam, V.lam_bar);        // shrinkage.py:297
        V.thr2 = V.lam2 / V.L;
      }
      if (!grid_wait(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      MARK(5);
      if (V.stop_prev) {                                  // iteration it-1 was the answer
        T0 { V.it--; V.conv = 1; }
        __syncthreads();
        break;
      }
      {
        // r_next is complete: start the GEMV^T operand loads now so their L2
        // latency overlaps the decision round trip (used only on accept)
        {
          const double* rs[1] = {a.R[V.irn]};
          gemv_t_prefetch<TA, 1>(D, PN, rs, gpre);
        }
        double Q2[2];
        gather<2>(E, Q2, 0u);
        T0 {
          V.rr = Q2[0];
          V.Fn = 0.5 * V.rr + V.lam * V.S[0];
          if (O.exact_L) {
            V.accept = 1;                                   // shrinkage.py:534-538
          } else {
            const double Qm = V.fy + V.S[1] + 0.5 * V.L * V.S[2] + V.lam * V.S[0];
            V.accept = V.Fn <= Qm + 1e-12 * pymax(1.0, fabs(Qm));   // shrinkage.py:210
          }
          if (V.accept) {                                   // shrinkage.py:283-284, 297
            int t = V.ixp; V.ixp = V.ix; V.ix = V.ixn; V.ixn = t;
            t = V.irxp; V.irxp = V.irx; V.irx = V.irn; V.irn = t;
            t = V.igxp; V.igxp = V.igx; V.igx = t;
            V.tp = V.tc; V.tc = V.tn;
            V.lam_used = V.lam;
            V.passes += 1;
            V.pend = 1;
            V.f_it = V.it; V.f_F = V.Fn; V.f_rr = V.rr; V.f_lam = V.lam;
            V.f_s4 = V.S[4]; V.f_s5 = V.S[5]; V.f_s6 = V.S[6];
            V.cut = 1e-10 * pymax(V.S[3], 1.0);             // model.py:232
            V.lam = V.lam2;                                 // speculative continuation
            V.fy = 0.5 * Q2[1];
            // begin iteration it+1 with the scalars prepared behind the barrier
            V.quit = (V.it >= C.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps));
            if (!V.quit) {
              V.it++; V.steps++; V.bt = 0; V.stop_prev = 0;
              V.m = V.mn;                                   // (t_prev - 1) / t with t_prev, t rotated
              V.tn = V.tn2;
              V.mn = V.mn2;
              V.thr = V.thr2;
            }
          } else {
            V.L *= O.eta;
            V.bt++;
            if (V.bt > 100) { V.status = ELL1_BREAKDOWN; V.quit = 1; }   // shrinkage.py:203,213
            V.thr = V.lam / V.L;
          }
        }
        __syncthreads();
      }
      MARK(6);
      if (!V.accept) {
        if (V.quit) goto out;
        zero12();
        prox(false);
        MARK(9);
        continue;
      }
      {
        const double* rs[1] = {a.R[V.irx]};
        double* os[1] = {Gp(V.igx)};
        panel_gemv_t_pre<TA, 1>(E, D, PN, gpre, rs, os);   // g_x = A^T r_next  (shrinkage.py:285)
      }
      MARK(7);
      zero12();
      {
        // KKT / support partials of the accepted iterate (model.py:160-173, 227-233)
        const double cut = V.cut;
        const double lamk = V.lam_used;
        const double* xc = Xp(V.ix);
        double* gc = Gp(V.igx);
        const double* rnow = a.R[V.irx];
        for_owned(E, [&](int k) {
          if (k >= E.w) gc[k] = s_ext * rnow[E.r0 + (k - E.w)];
          const double xj = xc[k];
          const double c = -gc[k];
          if (xj != 0.0) { s12[7] = nmax(s12[7], fabs(c - lamk * sgn(xj))); s12[9] = 1.0; }
          else { s12[8] = nmax(s12[8], fabs(c)); s12[10] = 1.0; }
          if (fabs(xj) > cut) s12[11] += 1.0;
        });
      }
      if (V.quit) {                                       // budget reached: flush the pending KKT
        double k5[5] = {s12[7], s12[8], s12[9], s12[10], s12[11]};
        block_reduce<5>(E, k5, 0xFu);
        publish<5>(E, k5);
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        double K[5];
        gather<5>(E, K, 0xFu);
        T0 {
          if (fista_finalize(V, C, a.trace, tw, K)) V.conv = 1;
          V.pend = 0;
        }
        __syncthreads();
        break;
      }
      prox(true);                                         // next iteration's first trial (same thread per k)
      MARK(8);
    }
    T0 if (!V.conv && V.it < C.max_iter && a.max_steps > 0) V.status = ELL1_RUNNING;
    __syncthreads();
  }

out:
  __syncthreads();
  // outputs (owned columns) and resumable state (CTA 0)
  if (V.status != ELL1_ERR_TIMEOUT) {
    const double* x = Xp(V.ix);
    const double* xp = Xp(V.ixp);
    const bool save = V.status == ELL1_RUNNING;
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = x[k];
      if (a.xprev_out) a.xprev_out[j] = xp[k];
      if (a.y_out) a.y_out[j] = Y[k];
      if (save) {
        for (int r = 0; r < 3; ++r) a.Xg[r][j] = Xp(r)[k];
        for (int r = 0; r < 2; ++r) a.Gg[r][j] = Gp(r)[k];
      }
    });
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    st->hist = V.hist;
    if (V.status != ELL1_ZERO_DATA) st->ntrace = V.it;
    st->rot[R_IX] = V.ix; st->rot[R_IXP] = V.ixp; st->rot[R_IXN] = V.ixn;
    st->rot[R_IGX] = V.igx; st->rot[R_IGXP] = V.igxp;
    st->rot[R_IRX] = V.irx; st->rot[R_IRXP] = V.irxp; st->rot[R_IRN] = V.irn;
    st->scal[S_L] = V.L; st->scal[S_TP] = V.tp; st->scal[S_TC] = V.tc; st->scal[S_LAM] = V.lam;
    st->scal[S_LAMBAR] = V.lam_bar; st->scal[S_FPREV] = V.Fprev; st->scal[S_FY] = V.fy;
    st->scal[S_LAMUSED] = V.lam_used;
    st->scal[S_PASSES] = V.passes;
  }
}

template <class TA, bool PROF>
__global__ void __launch_bounds__(NTHR, 1) fista_kernel(const __grid_constant__ FistaArgs a) {
  fista_body<TA, PROF>(a);
}

// ---------------------------------------------------------------------------
// correlation max: out = {max_j |(D^T b)_j|, ||b||}
struct CorrArgs {
  DictRaw D;
  const double* b;
  double* out;
  GridBufs g;
  int wmax;
};

// a grid barrier timed out (the kernel aborts cleanly): tell the host through
// the output block — out[0] = NaN, out[1] = ELL1_ERR_TIMEOUT
__device__ __forceinline__ void timeout_out(const Ctx& E, double* out) {
  if (E.b == 0 && threadIdx.x == 0) { out[0] = NAN; out[1] = (double)ELL1_ERR_TIMEOUT; }
}

template <class TA>
__device__ __forceinline__ void corr_body(const CorrArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  const DictV<TA> D = dict_view<TA>(a.D);
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.sh = smem + a.wmax;
  }
  __syncthreads();
  double* c = smem;
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  {
    const double* rs[1] = {a.b};
    double* os[1] = {c};
    panel_gemv_t<TA, 1>(E, D, PN, rs, os);
  }
  __syncthreads();
  double v[2] = {0.0, 0.0};
  for_owned(E, [&](int k) {
    const double ck = (k < E.w) ? c[k] : D.s * a.b[E.r0 + (k - E.w)];
    v[0] = nmax(v[0], fabs(ck));
  });
  for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) v[1] += a.b[i] * a.b[i];
  block_reduce<2>(E, v, 1u);
  publish<2>(E, v);
  if (!grid_sync(E)) { timeout_out(E, a.out); return; }
  double o[2];
  gather<2>(E, o, 1u);
  if (E.b == 0 && threadIdx.x == 0) { a.out[0] = o[0]; a.out[1] = sqrt(o[1]); }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) corr_kernel(const __grid_constant__ CorrArgs a) {
  corr_body<TA>(a);
}

// ---------------------------------------------------------------------------
// power iteration on the smaller Gram side of the PLAIN dictionary A
struct PowerArgs {
  DictRaw D;            // ext ignored
  const double* v0;     // start vector(s), dim each, normalised
  int nredraw;
  double tol;
  int max_iter;
  double* V[2];         // d-side: replicated d-vectors (ld)
  double* W;            // d-side: w (ld); n-side: u = A v (ld)
  double* out;
  GridBufs g;
  int wmax;
};

template <class TA>
__device__ __forceinline__ void power_body(const PowerArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.sh = smem + 3 * a.wmax;
  }
  __syncthreads();
  double* U = smem;                 // owned: A^T v (d-side) / w (n-side)
  double* Vn[2] = {smem + a.wmax, smem + 2 * a.wmax};
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const bool dside = D.d <= D.n;
  const int64_t dim = dside ? D.d : D.n;
  int iv = 0, redraw = 0, k = 0;
  double theta = 0.0;
  if (dside) {
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) a.V[0][i] = a.v0[i];
  } else {
    for_owned(E, [&](int kk) { Vn[0][kk] = a.v0[E.c0 + kk]; });
  }
  if (!grid_sync(E)) { timeout_out(E, a.out); return; }
  for (k = 0; k < a.max_iter; ++k) {
    double T[2], R2[1];
    if (dside) {
      double* v = a.V[iv];
      double* vn = a.V[1 - iv];
      {
        const double* rs[1] = {v};
        double* os[1] = {U};
        panel_gemv_t<TA, 1>(E, D, PN, rs, os);           // u = A^T v
        __syncthreads();
        const double* xs[1] = {U};
        panel_gemv<TA, 1>(E, D, PN, xs);                 // partial A u
      }
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      double q[2] = {0.0, 0.0};
      double none[1];
      const double* aux[1] = {v};
      gather_slice<0, 1, 1>(E, none, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
        const double wv = sums[0];
        a.W[i] = wv;
        q[0] += au[0] * wv;
        q[1] += wv * wv;
      });
      block_reduce<2>(E, q, 0u);
      publish<2>(E, q);
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      gather<2>(E, T, 0u);
      theta = T[0];
      const double nw = sqrt(T[1]);
      double e[1] = {0.0};
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
        const double wv = a.W[i];
        const double r = wv - theta * v[i];
        e[0] += r * r;
        vn[i] = wv / nw;                                // speculative next iterate
      }
      block_reduce<1>(E, e, 0u);
      publish<1>(E, e);
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      gather<1>(E, R2, 0u);
      if (sqrt(R2[0]) <= a.tol * pymax(theta, 2.2250738585072014e-308)) break;
      if (nw == 0.0) {
        if (redraw >= a.nredraw) break;
        ++redraw;
        for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) vn[i] = a.v0[redraw * dim + i];
        if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      }
    } else {
      double* v = Vn[iv];
      double* vn = Vn[1 - iv];
      {
        const double* xs[1] = {v};
        panel_gemv<TA, 1>(E, D, PN, xs);                 // partial A v
      }
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      double none[1];
      const double* aux[1] = {nullptr};
      gather_slice<0, 1, 0>(E, none, 0u, D.ld, aux,
                            [&](int64_t i, const double* sums, const double*) { a.W[i] = sums[0]; });
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      {
        const double* rs[1] = {a.W};
        double* os[1] = {U};
        panel_gemv_t<TA, 1>(E, D, PN, rs, os);           // w = A^T A v (panel)
      }
      __syncthreads();
      double q[2] = {0.0, 0.0};
      for_owned(E, [&](int kk) {
        const double wv = U[kk];
        q[0] += v[kk] * wv;
        q[1] += wv * wv;
      });
      block_reduce<2>(E, q, 0u);
      publish<2>(E, q);
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      gather<2>(E, T, 0u);
      theta = T[0];
      const double nw = sqrt(T[1]);
      double e[1] = {0.0};
      for_owned(E, [&](int kk) {
        const double wv = U[kk];
        const double r = wv - theta * v[kk];
        e[0] += r * r;
        vn[kk] = wv / nw;
      });
      block_reduce<1>(E, e, 0u);
      publish<1>(E, e);
      if (!grid_sync(E)) { timeout_out(E, a.out); return; }
      gather<1>(E, R2, 0u);
      if (sqrt(R2[0]) <= a.tol * pymax(theta, 2.2250738585072014e-308)) break;
      if (nw == 0.0) {
        if (redraw >= a.nredraw) break;
        ++redraw;
        for_owned(E, [&](int kk) { vn[kk] = a.v0[redraw * dim + E.c0 + kk]; });
        __syncthreads();
      }
    }
    iv = 1 - iv;
  }
  if (E.b == 0 && threadIdx.x == 0) { a.out[0] = theta; a.out[1] = (double)(k < a.max_iter ? k + 1 : k); }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) power_kernel(const __grid_constant__ PowerArgs a) {
  power_body<TA>(a);
}

}  // namespace ell1

// ============================================================================ host
using namespace ell1;

extern "C" size_t ell1_fista_workspace(const ell1_dict_t* D, const ell1_ctrl_t* C, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  (void)C;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  size_t b = grid_bytes(nb, D->d, 1);
  b += 5 * align_up(N * 8, 256) + 3 * align_up(D->ld * 8, 256) + 4096;
  return b;
}

// Args of one FISTA solve on nb CTAs (shared by the single and group launches).
static int fista_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                       const ell1_fista_opts_t* O, const ell1_io_t* io, int nb, FistaArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !O || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (C->max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.O = *O;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  for (int k = 0; k < 3; ++k) a.Xg[k] = cv.take<double>(N);
  for (int k = 0; k < 2; ++k) a.Gg[k] = cv.take<double>(N);
  for (int k = 0; k < 3; ++k) a.R[k] = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x; a.xprev_out = io->x_prev; a.y_out = io->y;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, FISTA_OV, 12, io->max_steps <= 0);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_fista(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                          const ell1_fista_opts_t* O, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  FistaArgs a;
  SmemPlan sp;
  const int rc = fista_setup(D, b, C, O, io, nb, a, sp);
  if (rc != ELL1_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  // padding rows of the residual ring must read as zero (never written by the kernel)
  if (D->ld > D->d)
    for (int k = 0; k < 3; ++k)
      if (cudaMemsetAsync(a.R[k] + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (a.prof)
    return (D->dtype == ELL1_F64) ? coop_launch(fista_kernel<double, true>, nb, sp.bytes, s, a, a.g.bar)
                                  : coop_launch(fista_kernel<float, true>, nb, sp.bytes, s, a, a.g.bar);
  return (D->dtype == ELL1_F64) ? coop_launch(fista_kernel<double, false>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(fista_kernel<float, false>, nb, sp.bytes, s, a, a.g.bar);
}

namespace ell1 {
template <class TA>
struct FistaRun {
  static __device__ void run(const FistaArgs& a) { fista_body<TA, false>(a); }
  static __device__ void reset(const FistaArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    for (int k = 0; k < 3; ++k) zero_pad_rows(a.R[k], a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(FistaArgs) <= ELL1_GROUP_ARG_BYTES, "FistaArgs too large for the group scratch");
}  // namespace ell1


int32_t ell1_fista_group_team_impl(const ell1_dict_t* D) {
  return dict_ok(D) ? group_team(to_raw(D), FISTA_OV, 12, 0) : 0;
}

extern "C" int ell1_fista_group(const ell1_group_t* G, const ell1_fista_opts_t* O, void* stream) {
  if (!G || (G->count > 0 && !O)) return ELL1_ERR_ARG;
  return run_group<FistaArgs, FistaRun>(G, FISTA_OV, 12, 0, [&](int i, int nb, FistaArgs& a, SmemPlan& sp) {
    if (O[i].probe) return (int)ELL1_ERR_ARG;
    return fista_setup(&G->dicts[i], G->b[i], &G->ctrl[i], &O[i], &G->io[i], nb, a, sp);
  }, stream);
}

extern "C" size_t ell1_correlation_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, D->d, 0) + 1024;
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
  if (!carve_grid(cv, a.g, nb, D->d, 0)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 1, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  a.wmax = sp.wmax;
  cudaStream_t s = (cudaStream_t)stream;
  return (D->dtype == ELL1_F64) ? coop_launch(corr_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(corr_kernel<float>, nb, sp.bytes, s, a, a.g.bar);
}

extern "C" size_t ell1_power_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, D->d, 1) + 3 * align_up(D->ld * 8, 256) + 2048;
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
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  a.V[0] = cv.take<double>(D->ld);
  a.V[1] = cv.take<double>(D->ld);
  a.W = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  for (double* p : {a.V[0], a.V[1], a.W})
    if (cudaMemsetAsync(p, 0, D->ld * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  const SmemPlan sp = plan_smem(a.D, nb, 3, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  a.wmax = sp.wmax;
  return (D->dtype == ELL1_F64) ? coop_launch(power_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(power_kernel<float>, nb, sp.bytes, s, a, a.g.bar);
}

namespace ell1 {
template <class TA>
struct CorrRun {
  static __device__ void run(const CorrArgs& a) { corr_body<TA>(a); }
  static __device__ void reset(const CorrArgs& a, int lane) { reset_bar(a.g.bar, lane); }
};
template <class TA>
struct PowerRun {
  static __device__ void run(const PowerArgs& a) { power_body<TA>(a); }
  static __device__ void reset(const PowerArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    for (int64_t i = lane; i < a.D.ld; i += 32) { a.V[0][i] = 0.0; a.V[1][i] = 0.0; a.W[i] = 0.0; }
  }
};
static_assert(sizeof(CorrArgs) <= ELL1_GROUP_ARG_BYTES, "CorrArgs too large for the group scratch");
static_assert(sizeof(PowerArgs) <= ELL1_GROUP_ARG_BYTES, "PowerArgs too large for the group scratch");
}  // namespace ell1

// max |D_i^T b_i| and ||b_i|| for every solve of a group: out[2 i], out[2 i + 1]
// (io[i].workspace: ell1_correlation_workspace; streamed, one CTA per solve)
extern "C" int ell1_correlation_max_group(const ell1_group_t* G, double* out, void* stream) {
  if (!G || (G->count > 0 && (!out || !G->b))) return ELL1_ERR_ARG;
  ell1_group_t H = *G;
  H.team = 1;
  return run_group<CorrArgs, CorrRun>(&H, 1, 2, 0, [&](int i, int nb, CorrArgs& a, SmemPlan& sp) {
    const ell1_dict_t* D = &G->dicts[i];
    if (!G->b[i] || !G->io) return (int)ELL1_ERR_ARG;
    a.D = to_raw(D);
    a.b = G->b[i];
    a.out = out + 2 * (int64_t)i;
    Carve cv(G->io[i].workspace, G->io[i].workspace_bytes);
    if (!carve_grid(cv, a.g, nb, D->d, 0)) return (int)ELL1_ERR_ARG;
    sp = plan_smem(a.D, nb, 1, 2, false);
    a.g.shcap = sp.scratch;
    a.g.panel_bytes = 0;
    a.wmax = sp.wmax;
    return (int)ELL1_OK;
  }, stream);
}

// spectral_norm_sq of every dictionary of a group (numerics.py:224-261):
// out[2 i] = ||D_i||^2, out[2 i + 1] = iterations; v0[i]: start vector + redraws
// (stride min(d, n)); io[i].workspace: ell1_power_workspace.  One CTA per solve.
extern "C" int ell1_spectral_norm_sq_group(const ell1_group_t* G, const double* const* v0, int32_t nredraw,
                                           double tol, int32_t max_iter, double* out, void* stream) {
  if (!G || (G->count > 0 && (!out || !v0)) || max_iter < 0) return ELL1_ERR_ARG;
  ell1_group_t H = *G;
  H.team = 1;
  return run_group<PowerArgs, PowerRun>(&H, 3, 2, 0, [&](int i, int nb, PowerArgs& a, SmemPlan& sp) {
    const ell1_dict_t* D = &G->dicts[i];
    if (!v0[i]) return (int)ELL1_ERR_ARG;
    a.D = to_raw(D);
    a.D.ext = 0;
    a.v0 = v0[i]; a.nredraw = nredraw; a.tol = tol; a.max_iter = max_iter; a.out = out + 2 * (int64_t)i;
    Carve cv(G->io[i].workspace, G->io[i].workspace_bytes);
    if (!carve_grid(cv, a.g, nb, D->d, 1)) return (int)ELL1_ERR_ARG;
    a.V[0] = cv.take<double>(D->ld);
    a.V[1] = cv.take<double>(D->ld);
    a.W = cv.take<double>(D->ld);
    if (!cv.ok) return (int)ELL1_ERR_ARG;
    sp = plan_smem(a.D, nb, 3, 2, false);
    a.g.shcap = sp.scratch;
    a.g.panel_bytes = 0;
    a.wmax = sp.wmax;
    return (int)ELL1_OK;
  }, stream);
}

