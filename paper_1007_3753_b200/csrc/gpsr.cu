// gpsr.cu — projected gradient on the nonnegative split z = [x+; x-]
// (gradient_projection.gpsr_solve, gradient_projection.py:114-192) as one
// persistent cooperative launch.
//
// Per iteration: round 1 = A (g+ - g-) for the exact step (the KKT test of the
// current x, ||g||^2 and the deferred support count of the previous step ride
// on its first barrier); round 2 per halving = A (x_cand - x) (plus A x_cand on
// the 64-step refresh, gradient_projection.py:172-175) with the candidate
// residual r + A dx written speculatively; accept -> grad_x = A^T r (local).
#include "solvers_common.cuh"

namespace ell1 {

struct GpsrArgs {
  DictRaw D;
  const double* b;
  ell1_ctrl_t C;
  double lam;
  GridBufs g;               // part stride 2 * ld
  double* Zg[2]; double* Gxg;              // owned backing (resume)
  double* R[2];             // replicated residual ring: r = A x - b (current / candidate)
  ell1_state_t* st;
  double* trace;
  double* x_out; double* z_out;
  int max_steps;
  int rc;
  int wmax;
  unsigned long long* prof;
};

enum { G_FPREV = 0, G_PASSES, G_F, G_RN };
constexpr int GPSR_OV = 10;   // zp, zm, x, gx, gp, gm, cp, cm, xc, v

struct GpsrV {
  double alpha, gg, curv, kkt, Fprev, passes, F, rn;
  double S[8];
  int it, hist, steps, conv, status, quit, phase, tries, accepted, ir, pend, note, done, refresh;
};

#define T0 if (threadIdx.x == 0)

template <class TA>
__device__ __forceinline__ void gpsr_body(const GpsrArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ GpsrV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + GPSR_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.steps = 0; V.done = 0; V.note = 0;
    V.it = 0; V.hist = 0; V.Fprev = 0; V.passes = 0; V.ir = 0; V.pend = 0;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist; V.ir = st->rot[0]; V.pend = st->rot[1];
      V.Fprev = st->scal[G_FPREV]; V.passes = st->scal[G_PASSES]; V.F = st->scal[G_F];
      V.rn = st->scal[G_RN];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, reinterpret_cast<TA*>(smem), a.rc);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const double* b = a.b;
  const double s_ext = D.s;
  const double lam = a.lam;
  double* ZP = ov;             double* ZM = ov + Wm;
  double* X = ov + 2 * Wm;     double* GX = ov + 3 * Wm;
  double* GP = ov + 4 * Wm;    double* GM = ov + 5 * Wm;
  double* CP = ov + 6 * Wm;    double* CM = ov + 7 * Wm;
  double* XC = ov + 8 * Wm;    double* VV = ov + 9 * Wm;
  const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;

  if (V.phase == 0) {
    // z = 0, x = 0, r = -b, grad_x = A^T r (gradient_projection.py:134-137)
    {
      const double* rs[1] = {b};
      double* os[1] = {GX};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    double v[2] = {0.0, 0.0};
    for_owned(E, [&](int k) {
      const double c = (k < E.w) ? GX[k] : s_ext * b[E.r0 + (k - E.w)];
      v[0] = nmax(v[0], fabs(c));
      GX[k] = -c;                                           // A^T(-b) = -(A^T b) exactly
      ZP[k] = 0.0; ZM[k] = 0.0; X[k] = 0.0;
    });
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
      v[1] += b[i] * b[i];
      a.R[0][i] = -b[i];
    }
    block_reduce<2>(E, v, 1u);
    publish<2>(E, v);
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    double g2[2];
    gather<2>(E, g2, 1u);
    T0 {
      const double bn = sqrt(g2[1]);
      if (g2[0] == 0.0) {                                   // gradient_projection.py:130-132
        if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = bn; a.trace[3] = 0.0; a.st->ntrace = 1; }
        V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
      } else if (E.b == 0) {
        a.trace[0] = 0.0; a.trace[1] = 0.5 * g2[1]; a.trace[2] = bn; a.trace[3] = 0.0;   // :138
      }
      V.phase = 1;
      V.passes = 1;
    }
    __syncthreads();
    if (V.quit) goto out;
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      ZP[k] = a.Zg[0][j]; ZM[k] = a.Zg[1][j]; GX[k] = a.Gxg[j];
      X[k] = ZP[k] - ZM[k];
    });
    __syncthreads();
  }

  while (true) {
    // ---------------- round 1: KKT of the current x, masked gradient, A (g+ - g-)
    {
      double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};              // max_on, max_off, any_on, any_off, gg, count, maxx, -
      for_owned(E, [&](int k) {
        const double xk = X[k], gxk = GX[k];
        const double c = -gxk;
        if (xk != 0.0) { s[0] = nmax(s[0], fabs(c - lam * sgn(xk))); s[2] = 1.0; }
        else { s[1] = nmax(s[1], fabs(c)); s[3] = 1.0; }
        const double gp0 = gxk + lam, gm0 = lam - gxk;    // gradient_projection.py:153
        const double gp = (ZP[k] > 0.0 || gp0 < 0.0) ? gp0 : 0.0;   // :154 / gpsr_direction
        const double gm = (ZM[k] > 0.0 || gm0 < 0.0) ? gm0 : 0.0;
        GP[k] = gp; GM[k] = gm;
        s[4] += gp * gp + gm * gm;
        VV[k] = gp - gm;
        s[6] = nmax(s[6], fabs(xk));
      });
      block_reduce<8>(E, s, 0x4Fu);
      // support count of the previous accepted x needs its max first
      const double cut = 1e-10 * pymax(s[6], 1.0);
      double c1[1] = {0.0};
      for_owned(E, [&](int k) { if (fabs(X[k]) > cut) c1[0] += 1.0; });
      block_reduce<1>(E, c1, 0u);
      s[5] = c1[0];
      publish<8>(E, s);
      const double* xs[1] = {VV};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double S8[8];
      double q[1] = {0.0};
      gather_slice<8, 1, 0>(E, S8, 0x4Fu, D.ld, {nullptr}, [&](int64_t i, const double* sums, const double*) {
        double av = sums[0];
        if (D.ext) av = av + s_ext * VV[E.w + (int)(i - E.r0)];
        q[0] += av * av;
      });
      T0 {
        double kkt = S8[2] > 0.0 ? S8[0] : 0.0;
        if (S8[3] > 0.0) kkt = pymax(pymax(kkt, S8[1] - lam), 0.0);
        V.kkt = kkt;
        V.gg = S8[4];
        V.passes += 1;
        if (V.pend) {                                        // finish step `it` (trace, stop rule)
          if (E.b == 0) {
            double* tr = a.trace + (size_t)V.it * 4;
            tr[0] = (double)V.it; tr[1] = V.F; tr[2] = V.rn; tr[3] = S8[5];
          }
          V.pend = 0;
          if (C.stop_kind != ELL1_STOP_NONE) {               // gradient_projection.py:182-187
            V.hist = V.hist < 2 ? V.hist + 1 : 2;
            const bool fire = stop_fires(C.stop_kind, C.stop_thr, V.hist, V.F, V.Fprev, V.S[3], V.S[4],
                                         V.S[5], C.gt_norm, kkt);
            V.Fprev = V.F;
            if (fire) { V.conv = 1; V.done = 1; }
          }
        }
        if (!V.done) {
          if (kkt <= C.tol * lam) { V.conv = 1; V.done = 1; }                       // :147-149
          else if (V.it >= C.max_iter) V.done = 1;
          else if (a.max_steps > 0 && V.steps >= a.max_steps) V.quit = 1;
          else if (V.gg == 0.0) { V.note = 1; V.done = 1; }                          // :155-158
        }
      }
      __syncthreads();
      if (V.done || V.quit) break;
      block_reduce<1>(E, q, 0u);
      publish<1>(E, q);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double g1[1];
      gather<1>(E, g1, 0u);
      T0 {
        V.curv = g1[0];
        V.alpha = (V.curv <= 1e-14 * V.gg) ? 1e8 : V.gg / V.curv;   // gpsr_step_size (:93-111)
        V.tries = 0; V.accepted = 0;
        V.refresh = ((V.it + 1) % 64) == 0;
      }
      __syncthreads();
    }
    // ---------------- halving search (gradient_projection.py:160-170)
    while (true) {
      {
        const double alpha = V.alpha;
        double s[6] = {0, 0, 0, 0, 0, 0};                  // grad.(cand - z), l1(xc), max|xc|, dx2, xp2, gt2
        for_owned(E, [&](int k) {
          const double gxk = GX[k];
          const double cp = fmax(ZP[k] - alpha * GP[k], 0.0);
          const double cm = fmax(ZM[k] - alpha * GM[k], 0.0);
          CP[k] = cp; CM[k] = cm;
          const double xc = cp - cm;
          XC[k] = xc;
          VV[k] = xc - X[k];
          s[0] += (gxk + lam) * (cp - ZP[k]) + (lam - gxk) * (cm - ZM[k]);
          s[1] += fabs(xc);
          s[2] = nmax(s[2], fabs(xc));
          if (relest) { const double dd = xc - X[k]; s[3] += dd * dd; s[4] += X[k] * X[k]; }
          if (gtr) { const double e = xc - C.ground_truth[gcol(E, D.n, k)]; s[5] += e * e; }
        });
        block_reduce<6>(E, s, 0x4u);
        publish<6>(E, s);
        if (V.refresh) {
          const double* xs[2] = {VV, XC};
          panel_gemv<TA, 2>(E, D, PN, xs);
        } else {
          const double* xs[1] = {VV};
          panel_gemv<TA, 1>(E, D, PN, xs);
        }
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double S6[6];
        double q[2] = {0.0, 0.0};
        const bool refresh = V.refresh;
        const double* rcur = a.R[V.ir];
        double* rnew = a.R[V.ir ^ 1];
        const double* aux[2] = {b, rcur};
        auto f = [&](int64_t i, const double* sums, const double* au) {
          const int kk = E.w + (int)(i - E.r0);
          double adx = sums[0];
          if (D.ext) adx = adx + s_ext * VV[kk];
          double r;
          if (refresh) {
            double axc = sums[1];
            if (D.ext) axc = axc + s_ext * XC[kk];
            r = axc - au[0];                                 // :173
          } else {
            r = au[1] + adx;                                 // :175
          }
          rnew[i] = r;
          q[0] += adx * adx;
          q[1] += r * r;
        };
        if (refresh) gather_slice<6, 2, 2>(E, S6, 0x4u, D.ld, aux, f);
        else gather_slice<6, 1, 2>(E, S6, 0x4u, D.ld, aux, f);
        block_reduce<2>(E, q, 0u);
        publish<2>(E, q);
        T0 { for (int k = 0; k < 6; ++k) V.S[k] = S6[k]; V.passes += refresh ? 2 : 1; }
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double Q2[2];
        gather<2>(E, Q2, 0u);
        T0 {
          const double dQ = V.S[0] + 0.5 * Q2[0];            // :164
          if (dQ < 0.0) {
            V.accepted = 1;
            V.F = 0.5 * Q2[1] + lam * V.S[1];                // :179
            V.rn = sqrt(Q2[1]);
          } else {
            V.alpha *= 0.5;
            V.tries++;
          }
        }
        __syncthreads();
        if (V.accepted || V.tries > 50) break;
      }
    }
    if (!V.accepted) {                                       // :166-169
      T0 { V.note = 2; V.conv = V.kkt <= C.tol * lam; V.done = 1; }
      __syncthreads();
      break;
    }
    // ---------------- accept: z, x, r, grad_x = A^T r (:171-176)
    T0 { V.it++; V.steps++; V.ir ^= 1; V.pend = 1; }
    __syncthreads();
    for_owned(E, [&](int k) { ZP[k] = CP[k]; ZM[k] = CM[k]; X[k] = XC[k]; });
    {
      const double* rs[1] = {a.R[V.ir]};
      double* os[1] = {GX};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    if (D.ext)
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) GX[E.w + (i - E.r0)] = s_ext * a.R[V.ir][i];
    T0 V.passes += 1;
    __syncthreads();
  }
  // after the loop (:189-191): convergence = KKT of the final x
  T0 {
    if (V.status == ELL1_OK && !V.conv && !V.quit) V.conv = V.kkt <= C.tol * lam;
    if (V.quit && V.status == ELL1_OK) V.status = ELL1_RUNNING;
  }
  __syncthreads();

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    const bool save = V.status == ELL1_RUNNING;
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = X[k];
      if (a.z_out) { a.z_out[j] = ZP[k]; a.z_out[D.n + (D.ext ? D.d : 0) + j] = ZM[k]; }
      if (save) { a.Zg[0][j] = ZP[k]; a.Zg[1][j] = ZM[k]; a.Gxg[j] = GX[k]; }
    });
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    st->hist = V.hist;
    if (V.status != ELL1_ZERO_DATA) st->ntrace = V.it + 1;
    st->rot[0] = V.ir; st->rot[1] = V.pend; st->rot[2] = V.note;
    st->scal[G_FPREV] = V.Fprev; st->scal[G_PASSES] = V.passes; st->scal[G_F] = V.F; st->scal[G_RN] = V.rn;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gpsr_kernel(const __grid_constant__ GpsrArgs a) {
  gpsr_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_gpsr_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  return grid_bytes(nb, D->d, 2) + 3 * align_up(N * 8, 256) + 2 * align_up(D->ld * 8, 256) + 4096;
}

static int gpsr_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
                         double* z_out, const ell1_io_t* io, int nb, GpsrArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (!(lam > 0) || C->max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.lam = lam;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 2)) return ELL1_ERR_ARG;
  a.Zg[0] = cv.take<double>(N); a.Zg[1] = cv.take<double>(N); a.Gxg = cv.take<double>(N);
  a.R[0] = cv.take<double>(D->ld); a.R[1] = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x;
  a.z_out = z_out;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, GPSR_OV, 8, io->max_steps <= 0);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_gpsr(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
                         double* z_out, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  GpsrArgs a;
  SmemPlan sp;
  const int rc0 = gpsr_setup(D, b, C, lam, z_out, io, nb, a, sp);
  if (rc0 != ELL1_OK) return rc0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->ld > D->d)
    for (double* p : {a.R[0], a.R[1]})
      if (cudaMemsetAsync(p + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(gpsr_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(gpsr_kernel<float>, nb, sp.bytes, s, a, a.g.bar);

}

namespace ell1 {
template <class TA>
struct GpsrRun {
  static __device__ void run(const GpsrArgs& a) { gpsr_body<TA>(a); }
  static __device__ void reset(const GpsrArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    zero_pad_rows(a.R[0], a.D.d, a.D.ld, lane);
    zero_pad_rows(a.R[1], a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(GpsrArgs) <= ELL1_GROUP_ARG_BYTES, "GpsrArgs too large for the group scratch");
}  // namespace ell1

int32_t ell1_gpsr_group_team_impl(const ell1_dict_t* D) {
  return dict_ok(D) ? group_team(to_raw(D), GPSR_OV, 8, 0) : 0;
}

extern "C" int ell1_gpsr_group(const ell1_group_t* G, const double* lam, void* stream) {
  if (!G || (G->count > 0 && !lam)) return ELL1_ERR_ARG;
  return run_group<GpsrArgs, GpsrRun>(G, GPSR_OV, 8, 0, [&](int i, int nb, GpsrArgs& a, SmemPlan& sp) {
    return gpsr_setup(&G->dicts[i], G->b[i], &G->ctrl[i], lam[i], nullptr, &G->io[i], nb, a, sp);
  }, stream);
}
