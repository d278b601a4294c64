// palm.cu — primal augmented Lagrangian (alm.palm_solve, alm.py:96-159) with the
// accelerated inner shrinkage (alm._inner_shrinkage, alm.py:71-93) as one
// persistent cooperative launch.
//
// Inner step: r_in = A y_vec - b_eff (panel GEMV round), grad = A^T r_in (local
// panel GEMV^T), x_new = soft(y_vec - grad/tau, 1/(mu tau)), momentum with the
// plain (un-nudged) t recurrence.  The relative-change exit test of step s
// rides on the first barrier of step s+1 (speculative step discarded on exit),
// so an inner step costs two grid barriers.  b_eff = b + y/mu and the
// multiplier y stay slice-owned: no d-vector is ever replicated except r_in.
#include "solvers_common.cuh"

namespace ell1 {

struct PalmArgs {
  DictRaw D;
  const double* b;
  ell1_ctrl_t C;
  double mu0, rho, tau;
  GridBufs g;
  double* Xg[2];            // owned-vector backing (resume): x, previous outer x
  double* Yd;               // slice-owned multiplier y (ld)
  double* RIN;              // replicated inner residual (ld)
  ell1_state_t* st;
  double* trace;
  double* x_out; double* y_out;
  int max_steps;            // outer iterations per launch (observer mode)
  int rc;
  int wmax;
  unsigned long long* prof;
};

enum { PA_BN = 0, PA_MU, PA_L1PREV, PA_PASSES, PA_MUUSED };
constexpr int PALM_OV = 4;      // owned: x_prev (outer x), x_new, y_vec, grad

struct PalmV {
  double bn, mu, l1_prev, passes, t_prev, shrink, tolr, m;
  double S[6];
  int it, hist, steps, cap, inner, conv, status, quit, phase, brk, outer, ototal;
  double mu_used;
};

#define T0 if (threadIdx.x == 0)

template <class TA>
__device__ __forceinline__ void palm_body(const PalmArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ PalmV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + PALM_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.outer = 0;
    V.it = 0; V.hist = 0; V.l1_prev = 0; V.passes = 0; V.mu = a.mu0; V.ototal = 0; V.mu_used = a.mu0;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist; V.ototal = st->rot[0];
      V.bn = st->scal[PA_BN]; V.mu = st->scal[PA_MU]; V.l1_prev = st->scal[PA_L1PREV];
      V.passes = st->scal[PA_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, reinterpret_cast<TA*>(smem), a.rc);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const double* b = a.b;
  const double s_ext = D.s;
  const double tau = a.tau;
  double* XP = ov;
  double* XN = ov + Wm;
  double* YV = ov + 2 * Wm;
  double* GR = ov + 3 * Wm;
  const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;

  if (V.phase == 0) {
    double q[1] = {0.0};
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
      q[0] += b[i] * b[i];
      a.Yd[i] = 0.0;
    }
    for_owned(E, [&](int k) { XP[k] = 0.0; XN[k] = 0.0; });
    block_reduce<1>(E, q, 0u);
    publish<1>(E, q);
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    double g1[1];
    gather<1>(E, g1, 0u);
    T0 {
      V.bn = sqrt(g1[0]);
      if (V.bn == 0.0) {                                   // alm.py:111-114
        if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = 0.0; a.trace[3] = 0.0; a.st->ntrace = 1; }
        V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
      } else {
        if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = V.bn; a.trace[3] = 0.0; }
        V.phase = 1;
      }
    }
    __syncthreads();
    if (V.quit) goto out;
  } else {
    for_owned(E, [&](int k) { XP[k] = a.Xg[0][gcol(E, D.n, k)]; XN[k] = a.Xg[1][gcol(E, D.n, k)]; });
    __syncthreads();
  }

  while (true) {
    T0 V.quit = (V.it >= C.max_iter || (a.max_steps > 0 && V.outer >= a.max_steps));
    __syncthreads();
    if (V.quit) break;
    // ---------------- inner accelerated shrinkage (alm.py:71-93)
    T0 {
      V.outer++;
      V.ototal++;
      V.shrink = 1.0 / (V.mu * tau);
      V.tolr = 1e-2 / V.mu;
      V.cap = C.max_iter - V.it < 200 ? C.max_iter - V.it : 200;
      V.t_prev = 1.0;
      V.inner = 0;
      V.brk = 0;
    }
    __syncthreads();
    for_owned(E, [&](int k) { YV[k] = XP[k]; });
    {
      bool carry = false;
      double cprev[2] = {0.0, 0.0};                         // block partials of ||dx||^2, ||x_new||^2
      while (true) {
        // round: A y_vec (+ change test of the previous step)
        {
          double s2[2] = {carry ? cprev[0] : 0.0, carry ? cprev[1] : 0.0};
          publish<2>(E, s2);
          const double* xs[1] = {YV};
          panel_gemv<TA, 1>(E, D, PN, xs);
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          double G2[2];
          const double mu = V.mu;
          const double* aux[2] = {b, a.Yd};
          gather_slice<2, 1, 2>(E, G2, 0u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
            double ay = sums[0];
            if (D.ext) ay = ay + s_ext * YV[E.w + (int)(i - E.r0)];
            const double beff = au[0] + au[1] / mu;          // alm.py:133
            a.RIN[i] = ay - beff;                            // alm.py:84
          });
          T0 {
            V.passes += 1;
            if (carry && sqrt(G2[0]) <= V.tolr * pymax(1.0, sqrt(G2[1]))) V.brk = 1;   // alm.py:89-92
            if (!V.brk && V.inner >= V.cap) V.brk = 1;
          }
          __syncthreads();
          if (V.brk) break;
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          const double* rs[1] = {a.RIN};
          double* os[1] = {GR};
          panel_gemv_t<TA, 1>(E, D, PN, rs, os);
        }
        __syncthreads();
        T0 {
          const double tn = 0.5 * (1.0 + sqrt(4.0 * V.t_prev * V.t_prev + 1.0));   // alm.py:87
          V.m = (V.t_prev - 1.0) / tn;
          V.t_prev = tn;
          V.inner++;
          V.passes += 1;
        }
        __syncthreads();
        {
          const double shrink = V.shrink, m = V.m;
          double c2[2] = {0.0, 0.0};
          for_owned(E, [&](int k) {
            if (k >= E.w) GR[k] = s_ext * a.RIN[E.r0 + (k - E.w)];
            const double xn = soft1(YV[k] - GR[k] / tau, shrink);   // alm.py:85
            const double xo = XP[k];
            YV[k] = xn + m * (xn - xo);                      // alm.py:88
            const double dd = xn - xo;
            c2[0] += dd * dd;
            c2[1] += xn * xn;
            XP[k] = xn;
          });
          block_reduce<2>(E, c2, 0u);
          cprev[0] = c2[0]; cprev[1] = c2[1];
          carry = true;
        }
      }
    }
    // ---------------- outer step: r = b - A x, y += mu r, trace (alm.py:137-142)
    T0 V.it += V.inner;
    {
      double s[5] = {0, 0, 0, 0, 0};                         // l1, max|x|, dx2, xp2, gt2
      for_owned(E, [&](int k) {
        const double xv = XP[k];
        s[0] += fabs(xv);
        s[1] = nmax(s[1], fabs(xv));
        if (relest) { const double xo = XN[k]; const double dd = xv - xo; s[2] += dd * dd; s[3] += xo * xo; }
        if (gtr) { const double e = xv - C.ground_truth[gcol(E, D.n, k)]; s[4] += e * e; }
      });
      block_reduce<5>(E, s, 0x2u);
      publish<5>(E, s);
      const double* xs[1] = {XP};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double S5[5];
      double q[1] = {0.0};
      const double mu = V.mu;
      const double* aux[2] = {b, a.Yd};
      gather_slice<5, 1, 2>(E, S5, 0x2u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
        double ax = sums[0];
        if (D.ext) ax = ax + s_ext * XP[E.w + (int)(i - E.r0)];
        const double r = au[0] - ax;                         // alm.py:138
        q[0] += r * r;
        a.Yd[i] = au[1] + mu * r;                            // alm.py:140
      });
      const double cut = 1e-10 * pymax(S5[1], 1.0);
      double c2[2] = {q[0], 0.0};
      for_owned(E, [&](int k) { if (fabs(XP[k]) > cut) c2[1] += 1.0; });
      block_reduce<2>(E, c2, 0u);
      publish<2>(E, c2);
      T0 { for (int k = 0; k < 5; ++k) V.S[k] = S5[k]; V.passes += 1; }
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double G2[2];
      gather<2>(E, G2, 0u);
      T0 {
        const double rn = sqrt(G2[0]);
        const double l1 = V.S[0];
        if (E.b == 0) {
          double* tr = a.trace + (size_t)V.ototal * 4;
          tr[0] = (double)V.it; tr[1] = l1; tr[2] = rn; tr[3] = G2[1];
        }
        const double rel = rn / V.bn;
        V.mu_used = V.mu;
        if (rel <= C.tol) {
          V.conv = 1;                                        // alm.py:146-148
        } else {
          if (C.stop_kind != ELL1_STOP_NONE) {
            V.hist = V.hist < 2 ? V.hist + 1 : 2;
            if (stop_fires(C.stop_kind, C.stop_thr, V.hist, l1, V.l1_prev, V.S[2], V.S[3], V.S[4],
                           C.gt_norm, rel))
              V.conv = 1;
            V.l1_prev = l1;
          }
          if (!V.conv) V.mu *= a.rho;                        // alm.py:155
        }
      }
      __syncthreads();
      // keep the outer iterate for the next relative-estimate test
      if (relest) for_owned(E, [&](int k) { XN[k] = XP[k]; });
      if (V.conv) break;
    }
  }
  T0 if (!V.conv && V.status == ELL1_OK && V.it < C.max_iter && a.max_steps > 0) V.status = ELL1_RUNNING;
  __syncthreads();

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    const bool save = V.status == ELL1_RUNNING;
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = XP[k];
      if (save) { a.Xg[0][j] = XP[k]; a.Xg[1][j] = XN[k]; }
    });
    if (a.y_out)
      for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) a.y_out[i] = a.Yd[i];
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    st->hist = V.hist;
    if (V.status != ELL1_ZERO_DATA) st->ntrace = V.ototal + 1;
    st->rot[0] = V.ototal;
    st->scal[PA_MUUSED] = V.mu_used;
    st->scal[PA_BN] = V.bn; st->scal[PA_MU] = V.mu; st->scal[PA_L1PREV] = V.l1_prev;
    st->scal[PA_PASSES] = V.passes;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) palm_kernel(const __grid_constant__ PalmArgs a) {
  palm_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_palm_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  return grid_bytes(nb, D->d, 1) + 2 * align_up(N * 8, 256) + 2 * align_up(D->ld * 8, 256) + 4096;
}

static int palm_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                         const ell1_palm_opts_t* O, const ell1_io_t* io, int nb, PalmArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !O || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  if (!(O->mu0 > 0) || !(O->rho > 1) || !(O->tau > 0) || C->max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.mu0 = O->mu0; a.rho = O->rho; a.tau = O->tau;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  a.Xg[0] = cv.take<double>(N);
  a.Xg[1] = cv.take<double>(N);
  a.Yd = cv.take<double>(D->ld);
  a.RIN = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x;
  a.y_out = O->y_out;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, PALM_OV, 5, io->max_steps <= 0);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_palm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                         const ell1_palm_opts_t* O, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  PalmArgs a;
  SmemPlan sp;
  const int rc0 = palm_setup(D, b, C, O, io, nb, a, sp);
  if (rc0 != ELL1_OK) return rc0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->ld > D->d)
    for (double* p : {a.Yd, a.RIN})
      if (cudaMemsetAsync(p + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(palm_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(palm_kernel<float>, nb, sp.bytes, s, a, a.g.bar);

}

namespace ell1 {
template <class TA>
struct PalmRun {
  static __device__ void run(const PalmArgs& a) { palm_body<TA>(a); }
  static __device__ void reset(const PalmArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    zero_pad_rows(a.Yd, a.D.d, a.D.ld, lane);
    zero_pad_rows(a.RIN, a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(PalmArgs) <= ELL1_GROUP_ARG_BYTES, "PalmArgs too large for the group scratch");
}  // namespace ell1

int32_t ell1_palm_group_team_impl(const ell1_dict_t* D) {
  return dict_ok(D) ? group_team(to_raw(D), PALM_OV, 5, 0) : 0;
}

extern "C" int ell1_palm_group(const ell1_group_t* G, const ell1_palm_opts_t* O, void* stream) {
  if (!G || (G->count > 0 && !O)) return ELL1_ERR_ARG;
  return run_group<PalmArgs, PalmRun>(G, PALM_OV, 5, 0, [&](int i, int nb, PalmArgs& a, SmemPlan& sp) {
    return palm_setup(&G->dicts[i], G->b[i], &G->ctrl[i], &O[i], &G->io[i], nb, a, sp);
  }, stream);
}
