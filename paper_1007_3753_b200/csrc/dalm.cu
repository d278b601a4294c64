// dalm.cu — dual augmented Lagrangian (alm.dalm_solve, alm.py:206-272) as one
// persistent cooperative launch.
//
// The y-step solves  beta A A^T y = beta A z - (A x - b)  (alm.py:172-189).
// With G = A A^T (+ s^2 I for [A, sI]) factored once per dictionary, the host
// precomputes Ginv = G^{-1} and M = Ginv A, so that
//     y = M (z - x / beta) + Ginv b / beta
// is a panel GEMV that shares one communication round with A z (the
// certificate's rhs).  The reference's residual certificate
// ||rhs - A A^T y|| <= 1e-10 max(1, ||rhs||) with one refinement step
// (y += Ginv resid) is kept exactly; failing it twice raises
// IllConditionedError.  A^T y is computed once per iteration and reused for
// the z-step of the next iteration, the x-update and the certificate.
//
// Rounds per iteration: [M v, A z] -> y (2 barriers), [A A^T y, A x] -> certificate,
// residual, trace (2 barriers).  y_cg_step mode (alm.py:192-203) follows the
// reference's single warm-started CG step.
#include "solvers_common.cuh"

namespace ell1 {

struct DalmArgs {
  DictRaw D;
  const void* M;            // Ginv A (A columns only), same layout / dtype as A
  const double* Ginv;       // d x d column-major (ld rows), float64
  const double* b;
  ell1_ctrl_t C;
  double beta;
  double ytol;
  int cg;
  GridBufs g;               // part stride 2 * ld
  double* Xg[2]; double* Zg; double* Ug;   // owned-vector backing (resume)
  double* Y[2];             // replicated y ring (ld)
  double* AX;               // slice-owned A x (ld)
  double* RHS;              // slice-owned rhs (ld)
  double* RES;              // replicated certificate residual / CG residual (ld)
  double* C0;               // slice-owned Ginv b (ld)
  ell1_state_t* st;
  double* trace;
  double* x_out; double* xprev_out; double* y_out; double* z_out;
  int max_steps;
  int rcA, rcM;
  int wmax;
  unsigned long long* prof;
};

enum { D_BN = 0, D_L1PREV, D_BY, D_RHS2, D_PASSES };
constexpr int DALM_OV = 5;      // owned: x ring (2), z, u = A^T y, v (temp)

struct DalmV {
  double bn, l1_prev, by, rhs2, rr, resid2, l1, maxu, passes;
  double S[8];
  double cg_rr, cg_curv;
  int it, hist, ix, iy, steps, conv, status, quit, phase, refine, cnt;
};

#define T0 if (threadIdx.x == 0)

template <class TA>
__device__ __forceinline__ void dalm_body(const DalmArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ DalmV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  const size_t esz = sizeof(TA);
  TA* panA = reinterpret_cast<TA*>(smem);
  TA* panM = reinterpret_cast<TA*>(reinterpret_cast<char*>(smem) + (size_t)a.rcA * D.ld * esz);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + DALM_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.steps = 0; V.refine = 0;
    V.it = 0; V.hist = 0; V.ix = 0; V.iy = 0; V.l1_prev = 0; V.passes = 0;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist; V.ix = st->rot[0]; V.iy = st->rot[1];
      V.bn = st->scal[D_BN]; V.l1_prev = st->scal[D_L1PREV]; V.passes = st->scal[D_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PA = setup_panel<TA>(E, D, panA, a.rcA);
  const Panel<TA> PM = setup_panel_at<TA>(reinterpret_cast<const TA*>(a.M), D.ld, E.c0, E.w, panM, a.rcM);
  const DictV<double> DG{a.Ginv, D.d, D.d, D.ld, 0, 0.0};
  const Panel<double> PG = setup_panel_at<double>(a.Ginv, D.ld, E.r0, (int)(E.r1 - E.r0), nullptr, 0);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const double beta = a.beta;
  const double* b = a.b;
  const double s_ext = D.s;
  auto Xp = [&](int r) { return ov + r * Wm; };
  double* Z = ov + 2 * Wm;
  double* U = ov + 3 * Wm;
  double* VV = ov + 4 * Wm;
  const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;

  if (V.phase == 0) {
    // ||b|| and c0 = Ginv b (d-side panel over this CTA's slice columns of Ginv)
    {
      const double* xs[1] = {b + E.r0};
      panel_gemv<double, 1>(E, DG, PG, xs);
      double q[1] = {0.0};
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) q[0] += b[i] * b[i];
      block_reduce<1>(E, q, 0u);
      publish<1>(E, q);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double g1[1];
      gather_slice<1, 1, 0>(E, g1, 0u, D.ld, {nullptr}, [&](int64_t i, const double* sums, const double*) {
        a.C0[i] = sums[0];
        a.AX[i] = 0.0;          // A x_0 = 0
        a.Y[0][i] = 0.0;        // y_0 = 0
      });
      for_owned(E, [&](int k) { Xp(0)[k] = 0.0; Xp(1)[k] = 0.0; U[k] = 0.0; Z[k] = 0.0; });
      T0 {
        V.bn = sqrt(g1[0]);
        if (V.bn == 0.0) {                                  // alm.py:223-226
          if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = 0.0; a.trace[3] = 0.0; a.st->ntrace = 1; }
          V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
        } else {
          if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = V.bn; a.trace[3] = 0.0; }
          V.phase = 1;
        }
      }
      __syncthreads();
      if (V.quit) goto out;
    }
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      Xp(0)[k] = a.Xg[0][j]; Xp(1)[k] = a.Xg[1][j]; Z[k] = a.Zg[j]; U[k] = a.Ug[j];
    });
    __syncthreads();
  }

  while (true) {
    T0 V.quit = (V.it >= C.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps));
    __syncthreads();
    if (V.quit) break;
    T0 { V.it++; V.steps++; V.refine = 0; }
    mark(E, -1);
    // ---- z-step (alm.py:239): z = clamp(A^T y + x / beta), v = z - x / beta
    {
      const double* x = Xp(V.ix);
      __syncthreads();
      for_owned(E, [&](int k) {
        const double xb = x[k] / beta;
        const double u = U[k] + xb;
        const double z = u > 1.0 ? 1.0 : (u < -1.0 ? -1.0 : u);
        Z[k] = z;
        VV[k] = (k < E.w) ? z - xb : s_ext * (z - xb);    // identity block of M = s Ginv
      });
    }
    const double* yprev = a.Y[V.iy];
    double* ynew = a.Y[V.iy ^ 1];
    if (!a.cg) {
      // ---- round 1: partials of M v and A z
      {
        const double* xv[1] = {VV};
        panel_gemv<TA, 1>(E, D, PM, xv, false, 0);
        if (D.ext) {                                        // M's identity block: s Ginv[:, slice]
          const double* xe[1] = {VV + E.w};
          panel_gemv<double, 1>(E, DG, PG, xe, true, 0);
        }
        const double* xz[1] = {Z};
        panel_gemv<TA, 1>(E, D, PA, xz, false, 1);
      }
      mark(E, 0);
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double q[2] = {0.0, 0.0};
        const double* aux[3] = {b, a.AX, a.C0};
        gather_slice<0, 2, 3>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          const int kk = E.w + (int)(i - E.r0);
          const double y = sums[0] + au[2] / beta;         // y = M (z - x/beta) + Ginv b / beta
          double az = sums[1];
          if (D.ext) az = az + s_ext * Z[kk];               // robust.py:93
          const double rhs = az - (au[1] - au[0]) / beta;   // alm.py:179
          ynew[i] = y;
          a.RHS[i] = rhs;
          q[0] += rhs * rhs;
          q[1] += au[0] * y;
        });
        block_reduce<2>(E, q, 0u);
        publish<2>(E, q);
      }
      mark(E, 1);
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double g2[2];
        gather<2>(E, g2, 0u);
        T0 { V.rhs2 = g2[0]; V.by = g2[1]; V.passes += 2; }
      }
    } else {
      // ---- single warm-started CG step (alm.py:192-203)
      {
        const double* xz[2] = {Z, U};
        panel_gemv<TA, 2>(E, D, PA, xz);                    // A z, A (A^T y_prev)
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double q[1] = {0.0};
        const double* aux[2] = {b, a.AX};
        gather_slice<0, 2, 2>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          const int kk = E.w + (int)(i - E.r0);
          double az = sums[0], aau = sums[1];
          if (D.ext) { az = az + s_ext * Z[kk]; aau = aau + s_ext * U[kk]; }
          const double rhs = az - (au[1] - au[0]) / beta;
          const double r = rhs - aau;
          a.RHS[i] = rhs;
          a.RES[i] = r;
          q[0] += r * r;
        });
        block_reduce<1>(E, q, 0u);
        publish<1>(E, q);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double g1[1];
        gather<1>(E, g1, 0u);
        T0 { V.cg_rr = g1[0]; V.passes += 2; }
      }
      __syncthreads();
      if (V.cg_rr == 0.0) {
        for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) ynew[i] = yprev[i];
        double q[1] = {0.0};
        for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) q[0] += b[i] * yprev[i];
        block_reduce<1>(E, q, 0u);
        publish<1>(E, q);
      } else {
        {
          const double* rs[1] = {a.RES};
          double* os[1] = {VV};
          panel_gemv_t<TA, 1>(E, D, PA, rs, os);          // A^T r
          __syncthreads();
          if (D.ext)
            for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) VV[E.w + (i - E.r0)] = s_ext * a.RES[i];
          const double* xv[1] = {VV};
          panel_gemv<TA, 1>(E, D, PA, xv);                 // A A^T r
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          double q[1] = {0.0};
          const double* aux[1] = {a.RES};
          gather_slice<0, 1, 1>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
            double ar = sums[0];
            if (D.ext) ar = ar + s_ext * VV[E.w + (int)(i - E.r0)];
            q[0] += au[0] * ar;
          });
          block_reduce<1>(E, q, 0u);
          publish<1>(E, q);
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          double g1[1];
          gather<1>(E, g1, 0u);
          T0 {
            V.cg_curv = g1[0];
            V.passes += 2;
            if (V.cg_curv <= 0.0) { V.status = ELL1_ILL_CONDITIONED; V.quit = 1; }   // alm.py:201-202
          }
          __syncthreads();
          if (V.quit) goto out;
        }
        const double step = V.cg_rr / V.cg_curv;
        double q[1] = {0.0};
        for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
          const double y = yprev[i] + step * a.RES[i];
          ynew[i] = y;
          q[0] += b[i] * y;
        }
        block_reduce<1>(E, q, 0u);
        publish<1>(E, q);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double g1[1];
        gather<1>(E, g1, 0u);
        T0 V.by = g1[0];
      }
    }

    // ---- x-step + certificate / residual round (retried once after refinement)
    while (true) {
      mark(E, 2);
      {
        const double* rs[1] = {ynew};
        double* os[1] = {U};
        panel_gemv_t<TA, 1>(E, D, PA, rs, os);            // Aty = A^T y  (alm.py:245)
      }
      __syncthreads();
      mark(E, 3);
      {
        const double* x = Xp(V.ix);
        double* xn = Xp(V.ix ^ 1);
        double s[6] = {0, 0, 0, 0, 0, 0};                   // l1, max|Aty|, max|x|, dx2, xp2, gt2
        for_owned(E, [&](int k) {
          if (k >= E.w) U[k] = s_ext * ynew[E.r0 + (k - E.w)];   // robust.py:96
          const double u = U[k];
          const double xo = x[k];
          const double xv = xo - beta * (Z[k] - u);         // alm.py:246
          xn[k] = xv;
          s[0] += fabs(xv);
          s[1] = nmax(s[1], fabs(u));
          s[2] = nmax(s[2], fabs(xv));
          if (relest) { const double dd = xv - xo; s[3] += dd * dd; s[4] += xo * xo; }
          if (gtr) { const double e = xv - C.ground_truth[gcol(E, D.n, k)]; s[5] += e * e; }
        });
        block_reduce<6>(E, s, 0x6u);
        publish<6>(E, s);
        const double* xs[2] = {U, xn};
        panel_gemv<TA, 2>(E, D, PA, xs);                   // A A^T y, A x
      }
      mark(E, 4);
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      mark(E, 5);
      {
        double S6[6];
        double q[2] = {0.0, 0.0};
        const double* xn = Xp(V.ix ^ 1);
        const double* aux[2] = {b, a.RHS};
        gather_slice<6, 2, 2>(E, S6, 0x6u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          const int kk = E.w + (int)(i - E.r0);
          double aau = sums[0], ax = sums[1];
          if (D.ext) { aau = aau + s_ext * U[kk]; ax = ax + s_ext * xn[kk]; }
          const double resid = au[1] - aau;                 // alm.py:181
          a.RES[i] = resid;
          a.AX[i] = ax;
          const double r = au[0] - ax;                      // alm.py:249
          q[0] += resid * resid;
          q[1] += r * r;
        });
        // support count of the new x (model.py:227-233) needs the global max first
        const double cut = 1e-10 * pymax(S6[2], 1.0);
        double c3[3] = {q[0], q[1], 0.0};
        for_owned(E, [&](int k) { if (fabs(xn[k]) > cut) c3[2] += 1.0; });
        block_reduce<3>(E, c3, 0u);
        publish<3>(E, c3);
        T0 { for (int k = 0; k < 6; ++k) V.S[k] = S6[k]; }
      }
      mark(E, 6);
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      mark(E, 7);
      {
        double g3[3];
        gather<3>(E, g3, 0u);
        T0 {
          V.resid2 = g3[0]; V.rr = g3[1]; V.cnt = (int)g3[2];
          V.passes += 2;
          int next = 0;                                     // 0 accept, 1 refine, 2 fail
          if (!a.cg) {
            const double scale = pymax(1.0, sqrt(V.rhs2));
            if (sqrt(V.resid2) > a.ytol * scale) next = V.refine ? 2 : 1;   // alm.py:183-188
          }
          if (next == 2) { V.status = ELL1_ILL_CONDITIONED; V.quit = 1; }
          V.refine = next == 1 ? 1 : (next == 0 ? 0 : V.refine);
          V.cnt = next == 1 ? -1 : V.cnt;
        }
        __syncthreads();
        if (V.quit) goto out;
        if (V.cnt >= 0) break;
      }
      // ---- refinement: y += Ginv resid  (alm.py:184)
      {
        const double* xs[1] = {a.RES + E.r0};
        panel_gemv<double, 1>(E, DG, PG, xs);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double q[1] = {0.0};
        const double* aux[1] = {b};
        gather_slice<0, 1, 1>(E, nullptr, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          const double y = ynew[i] + sums[0];
          ynew[i] = y;
          q[0] += au[0] * y;
        });
        block_reduce<1>(E, q, 0u);
        publish<1>(E, q);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double g1[1];
        gather<1>(E, g1, 0u);
        T0 { V.by = g1[0]; V.refine = 1; V.passes += 1; }
      }
      __syncthreads();
    }
    mark(E, 8);
    // ---- trace, convergence (alm.py:249-262), user stopping rule (alm.py:263-268)
    T0 {
      const double rn = sqrt(V.rr);
      const double l1 = V.S[0];
      if (E.b == 0) {
        double* tr = a.trace + (size_t)V.it * 4;
        tr[0] = (double)V.it; tr[1] = l1; tr[2] = rn; tr[3] = (double)V.cnt;
      }
      const double rel = rn / V.bn;
      const double scale = pymax(1.0, V.S[1]);
      const double gap = l1 - V.by / scale;
      V.ix ^= 1; V.iy ^= 1;
      if (rel <= C.tol && gap <= C.tol * pymax(1.0, l1)) {
        V.conv = 1;
      } else if (C.stop_kind != ELL1_STOP_NONE) {
        V.hist = V.hist < 2 ? V.hist + 1 : 2;
        if (stop_fires(C.stop_kind, C.stop_thr, V.hist, l1, V.l1_prev, V.S[3], V.S[4], V.S[5],
                       C.gt_norm, rel))
          V.conv = 1;
        V.l1_prev = l1;
      }
    }
    __syncthreads();
    if (V.conv) break;
  }
  T0 if (!V.conv && V.status == ELL1_OK && V.it < C.max_iter && a.max_steps > 0) V.status = ELL1_RUNNING;
  __syncthreads();

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    const bool save = V.status == ELL1_RUNNING;
    const double* x = Xp(V.ix);
    const double* xp = Xp(V.ix ^ 1);
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = x[k];
      if (a.xprev_out) a.xprev_out[j] = xp[k];
      if (a.z_out) a.z_out[j] = Z[k];
      if (save) { a.Xg[0][j] = Xp(0)[k]; a.Xg[1][j] = Xp(1)[k]; a.Zg[j] = Z[k]; a.Ug[j] = U[k]; }
    });
    if (a.y_out)
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) a.y_out[i] = a.Y[V.iy][i];
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    st->hist = V.hist;
    st->ntrace = (V.status == ELL1_ZERO_DATA) ? 1 : V.it + 1;
    st->rot[0] = V.ix; st->rot[1] = V.iy;
    st->scal[D_BN] = V.bn; st->scal[D_L1PREV] = V.l1_prev; st->scal[D_BY] = V.by;
    st->scal[D_PASSES] = V.passes;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) dalm_kernel(const __grid_constant__ DalmArgs a) {
  dalm_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_dalm_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  return grid_bytes(nb, D->d, 2) + 4 * align_up(N * 8, 256) + 7 * align_up(D->ld * 8, 256) + 4096;
}

static int dalm_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                         const ell1_dalm_opts_t* O, const ell1_io_t* io, int nb, DalmArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !O || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (!O->M || !O->Ginv || !(O->beta > 0) || C->max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.M = O->M;
  a.Ginv = O->Ginv;
  a.b = b;
  a.C = *C;
  a.beta = O->beta;
  a.ytol = O->y_tol;
  a.cg = O->y_cg_step;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 2)) return ELL1_ERR_ARG;
  a.Xg[0] = cv.take<double>(N); a.Xg[1] = cv.take<double>(N);
  a.Zg = cv.take<double>(N); a.Ug = cv.take<double>(N);
  a.Y[0] = cv.take<double>(D->ld); a.Y[1] = cv.take<double>(D->ld);
  a.AX = cv.take<double>(D->ld); a.RHS = cv.take<double>(D->ld); a.RES = cv.take<double>(D->ld);
  a.C0 = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x; a.xprev_out = io->x_prev; a.y_out = O->y_out; a.z_out = O->z_out;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, DALM_OV, 6, false);
  // resident budget shared between the A and M panels
  {
    const int64_t esz = D->dtype == ELL1_F64 ? 8 : 4;
    const int64_t room = ((int64_t)max_smem_optin() - (int64_t)sp.bytes) / (D->ld * esz);
    const int64_t wcols = (D->n + nb - 1) / nb;
    int64_t ra = room / 2 < wcols ? room / 2 : wcols;
    int64_t rm = room - ra < wcols ? room - ra : wcols;
    if (io->max_steps > 0 || room <= 0) ra = rm = 0;
    a.rcA = (int)ra;
    a.rcM = (int)rm;
    sp.panel_bytes = (size_t)align_up((ra + rm) * D->ld * esz, 16);
    sp.bytes += sp.panel_bytes;
  }
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_dalm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                         const ell1_dalm_opts_t* O, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  DalmArgs a;
  SmemPlan sp;
  const int rc0 = dalm_setup(D, b, C, O, io, nb, a, sp);
  if (rc0 != ELL1_OK) return rc0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->ld > D->d)
    for (double* p : {a.Y[0], a.Y[1], a.AX, a.RHS, a.RES, a.C0})
      if (cudaMemsetAsync(p + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(dalm_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(dalm_kernel<float>, nb, sp.bytes, s, a, a.g.bar);

}

namespace ell1 {
template <class TA>
struct DalmRun {
  static __device__ void run(const DalmArgs& a) { dalm_body<TA>(a); }
  static __device__ void reset(const DalmArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    for (double* p : {a.Y[0], a.Y[1], a.AX, a.RHS, a.RES, a.C0}) zero_pad_rows(p, a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(DalmArgs) <= ELL1_GROUP_ARG_BYTES, "DalmArgs too large for the group scratch");
}  // namespace ell1

// the team must hold both the A and the M panel: size it for 2n columns
int32_t ell1_dalm_group_team_impl(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  DictRaw r = to_raw(D);
  r.n *= 2;
  return group_team(r, DALM_OV, 6, 0);
}

extern "C" int ell1_dalm_group(const ell1_group_t* G, const ell1_dalm_opts_t* O, void* stream) {
  if (!G || (G->count > 0 && !O)) return ELL1_ERR_ARG;
  int team = G->team;
  if (team <= 0)
    for (int i = 0; i < G->count; ++i) {
      const int t = ell1_dalm_group_team_impl(&G->dicts[i]);
      if (t > team) team = t;
    }
  ell1_group_t H = *G;
  H.team = team;
  return run_group<DalmArgs, DalmRun>(&H, DALM_OV, 6, 0, [&](int i, int nb, DalmArgs& a, SmemPlan& sp) {
    return dalm_setup(&G->dicts[i], G->b[i], &G->ctrl[i], &O[i], &G->io[i], nb, a, sp);
  }, stream);
}
