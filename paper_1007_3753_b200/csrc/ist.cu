// ist.cu — SpaRSA-style iterative shrinkage over a continuation schedule
// (shrinkage.ist_solve, shrinkage.py:105-181) as one persistent cooperative
// launch.  Stages, alpha doublings, BB steps, stalls and stopping rules run on
// the device with the reference's formulas:
//   attempt : cand = soft(x - g/alpha, lam/alpha); A cand (panel GEMV round);
//             dF = g'(cand - x) + 1/2 ||A cand - A x||^2 + lam sum(|cand| - |x|)
//   accept  : g_new = A^T(A cand - b) (local GEMV^T); alpha = BB(s, y);
//             KKT / support / BB reductions in one barrier.
#include "solvers_common.cuh"

namespace ell1 {

struct IstArgs {
  DictRaw D;
  const double* b;
  ell1_ctrl_t C;
  const double* stages;      // host-built schedule (shrinkage.py:43-58)
  int nstages;
  GridBufs g;
  double* Xg[2]; double* Gg[2];
  double* RC;                // replicated A cand - b (ld)
  double* AXs[2];            // slice-owned ring: A x (current), A cand (candidate)
  ell1_state_t* st;
  double* trace;
  double* x_out;
  int max_steps;             // accepted steps per launch (observer mode)
  int rc;
  int wmax;
  unsigned long long* prof;
};

enum { I_ALPHA = 0, I_LAM, I_KKT, I_FPREV, I_DF, I_PASSES };
constexpr int IST_OV = 5;      // owned: x, cand, g ring (2), spare

struct IstV {
  double alpha, lam, kkt, Fprev, dF, passes, thr;
  double S[8], Q[2];
  int it, hist, si, active, fin, conv, status, quit, phase, steps, accepted, stalled, tries;
  int ix, ig, iax, done;
};

#define T0 if (threadIdx.x == 0)

template <class TA>
__device__ __forceinline__ void ist_body(const IstArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ IstV V;
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem + a.g.panel_bytes / 8;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + IST_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.steps = 0; V.done = 0;
    V.it = 0; V.hist = 0; V.si = 0; V.active = 0; V.alpha = 1.0; V.Fprev = 0; V.kkt = 0;
    V.ix = 0; V.ig = 0; V.iax = 0; V.passes = 0; V.dF = 0;
    if (V.phase != 0) {
      V.it = st->iterations; V.hist = st->hist;
      V.si = st->rot[0]; V.active = st->rot[1]; V.ix = st->rot[2]; V.ig = st->rot[3]; V.iax = st->rot[4];
      V.alpha = st->scal[I_ALPHA]; V.lam = st->scal[I_LAM]; V.kkt = st->scal[I_KKT];
      V.Fprev = st->scal[I_FPREV]; V.passes = st->scal[I_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, reinterpret_cast<TA*>(smem), a.rc);
  const int Wm = a.wmax;
  const ell1_ctrl_t& C = a.C;
  const double* b = a.b;
  const double s_ext = D.s;
  const double lam_t = a.stages[a.nstages - 1];
  auto Xp = [&](int r) { return ov + r * Wm; };          // x / cand
  auto Gp = [&](int r) { return ov + (2 + r) * Wm; };    // g ring
  const bool relest = C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = C.stop_kind == ELL1_STOP_GROUND_TRUTH;

  if (V.phase == 0) {
    // x = 0, A x = 0, g = A^T(A x - b) = -A^T b (shrinkage.py:126-132)
    {
      const double* rs[1] = {b};
      double* os[1] = {Gp(0)};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    double v[2] = {0.0, 0.0};
    for_owned(E, [&](int k) {
      const double c = (k < E.w) ? Gp(0)[k] : s_ext * b[E.r0 + (k - E.w)];
      v[0] = nmax(v[0], fabs(c));
      Gp(0)[k] = -c;
      Xp(0)[k] = 0.0; Xp(1)[k] = 0.0;
    });
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) {
      v[1] += b[i] * b[i];
      a.AXs[0][i] = 0.0;
    }
    block_reduce<2>(E, v, 1u);
    publish<2>(E, v);
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    double g2[2];
    gather<2>(E, g2, 1u);
    T0 {
      if (g2[0] == 0.0) {                                   // shrinkage.py:121-123
        if (E.b == 0) { a.trace[0] = 0.0; a.trace[1] = 0.0; a.trace[2] = sqrt(g2[1]); a.trace[3] = 0.0; a.st->ntrace = 1; }
        V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
      }
      V.phase = 1;
      V.passes = 1;
    }
    __syncthreads();
    if (V.quit) goto out;
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      Xp(0)[k] = a.Xg[0][j]; Xp(1)[k] = a.Xg[1][j]; Gp(0)[k] = a.Gg[0][j]; Gp(1)[k] = a.Gg[1][j];
    });
    __syncthreads();
  }

  while (true) {
    // ---------------- stage entry (shrinkage.py:134-140)
    if (!V.active) {
      T0 {
        if (V.si >= a.nstages) V.done = 1;
        else { V.lam = a.stages[V.si]; V.fin = V.lam == lam_t; }
      }
      __syncthreads();
      if (V.done) break;
      {
        double k4[4] = {0, 0, 0, 0};
        const double* x = Xp(V.ix);
        const double* gg = Gp(V.ig);
        const double lam = V.lam;
        for_owned(E, [&](int k) {
          const double c = -gg[k];
          if (x[k] != 0.0) { k4[0] = nmax(k4[0], fabs(c - lam * sgn(x[k]))); k4[2] = 1.0; }
          else { k4[1] = nmax(k4[1], fabs(c)); k4[3] = 1.0; }
        });
        block_reduce<4>(E, k4, 0xFu);
        publish<4>(E, k4);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double K[4];
        gather<4>(E, K, 0xFu);
        T0 {
          double kkt = K[2] > 0.0 ? K[0] : 0.0;
          if (K[3] > 0.0) kkt = pymax(pymax(kkt, K[1] - V.lam), 0.0);
          V.kkt = kkt;
          if (kkt <= C.tol * V.lam) {
            if (V.fin) V.conv = 1;
            V.si++;                                           // next stage
          } else {
            V.active = 1;
            V.stalled = 0;
          }
        }
        __syncthreads();
        continue;
      }
    }
    // ---------------- one accepted step (shrinkage.py:141-179)
    T0 V.quit = V.it >= C.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps);
    __syncthreads();
    if (V.quit) {
      if (V.it >= C.max_iter) {                             // while-loop exhausted
        T0 {
          V.active = 0;
          if (!V.conv) V.done = 1;                          // shrinkage.py:175-176
          else V.si++;
        }
        __syncthreads();
        if (V.done) break;
        continue;
      }
      break;                                                // step budget of this launch
    }
    T0 { V.tries = 0; V.accepted = 0; }
    __syncthreads();
    while (true) {
      T0 V.thr = V.lam / V.alpha;
      __syncthreads();
      {
        const double alpha = V.alpha, thr = V.thr;
        const double* x = Xp(V.ix);
        double* cd = Xp(V.ix ^ 1);
        const double* gg = Gp(V.ig);
        double s[6] = {0, 0, 0, 0, 0, 0};                   // g.dl, sum(|c|-|x|), max|c|, dx2, xp2, gt2
        for_owned(E, [&](int k) {
          const double xo = x[k];
          const double c = soft1(xo - gg[k] / alpha, thr);  // shrinkage.py:144
          cd[k] = c;
          const double dl = c - xo;
          s[0] += gg[k] * dl;
          s[1] += fabs(c) - fabs(xo);
          s[2] = nmax(s[2], fabs(c));
          if (relest) { s[3] += dl * dl; s[4] += xo * xo; }
          if (gtr) { const double e = c - C.ground_truth[gcol(E, D.n, k)]; s[5] += e * e; }
        });
        block_reduce<6>(E, s, 0x4u);
        publish<6>(E, s);
        const double* xs[1] = {cd};
        panel_gemv<TA, 1>(E, D, PN, xs);
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double S6[6];
        double q[3] = {0.0, 0.0, 0.0};                      // ||A cand - A x||^2, ||b - A cand||^2, sum|cand|
        const double* cd = Xp(V.ix ^ 1);
        double* acn = a.AXs[V.iax ^ 1];
        const double* aux[2] = {b, a.AXs[V.iax]};
        gather_slice<6, 1, 2>(E, S6, 0x4u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
          double ac = sums[0];
          if (D.ext) ac = ac + s_ext * cd[E.w + (int)(i - E.r0)];
          acn[i] = ac;
          a.RC[i] = ac - au[0];                             // shrinkage.py:155 (A cand - b)
          const double da = ac - au[1];
          q[0] += da * da;
          const double r = au[0] - ac;
          q[1] += r * r;
        });
        for_owned(E, [&](int k) { q[2] += fabs(cd[k]); });
        block_reduce<3>(E, q, 0u);
        publish<3>(E, q);
        T0 { for (int k = 0; k < 6; ++k) V.S[k] = S6[k]; V.passes += 1; }
      }
      if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      {
        double Q3[3];
        gather<3>(E, Q3, 0u);
        T0 {
          V.Q[0] = Q3[1]; V.Q[1] = Q3[2];
          const double dF = V.S[0] + 0.5 * Q3[0] + V.lam * V.S[1];   // shrinkage.py:91-102
          V.dF = dF;
          if (dF < 0.0) V.accepted = 1;
          else {
            V.alpha = V.alpha * 2.0 < 1e30 ? V.alpha * 2.0 : 1e30;    // shrinkage.py:150
            V.tries++;
          }
        }
        __syncthreads();
        if (V.accepted || V.tries >= 50) break;
      }
    }
    if (!V.accepted) {                                      // stage stalled (shrinkage.py:151-153)
      T0 {
        V.active = 0;
        if (V.fin && V.kkt <= C.tol * V.lam) V.conv = 1;
        if (!V.fin) V.si++;                                 // shrinkage.py:172-173
        else if (V.it >= C.max_iter && !V.conv) V.done = 1;
        else V.si++;
      }
      __syncthreads();
      if (V.done) break;
      continue;
    }
    // ---------------- accepted: g_new, BB step, trace, KKT (shrinkage.py:154-171)
    {
      const double* rs[1] = {a.RC};
      double* os[1] = {Gp(V.ig ^ 1)};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    {
      const double* x = Xp(V.ix);
      const double* cd = Xp(V.ix ^ 1);
      const double* go = Gp(V.ig);
      double* gn = Gp(V.ig ^ 1);
      const double lam = V.lam;
      const double cut = 1e-10 * pymax(V.S[2], 1.0);
      double s[7] = {0, 0, 0, 0, 0, 0, 0};                  // ss, sy, max_on, max_off, any_on, any_off, count
      for_owned(E, [&](int k) {
        if (k >= E.w) gn[k] = s_ext * a.RC[E.r0 + (k - E.w)];
        const double sk = cd[k] - x[k];
        const double yk = gn[k] - go[k];
        s[0] += sk * sk;
        s[1] += sk * yk;
        const double c = -gn[k];
        if (cd[k] != 0.0) { s[2] = nmax(s[2], fabs(c - lam * sgn(cd[k]))); s[4] = 1.0; }
        else { s[3] = nmax(s[3], fabs(c)); s[5] = 1.0; }
        if (fabs(cd[k]) > cut) s[6] += 1.0;
      });
      block_reduce<7>(E, s, 0x3Cu);
      publish<7>(E, s);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double K[7];
      gather<7>(E, K, 0x3Cu);
      T0 {
        V.it++; V.steps++;
        V.passes += 1;
        const double ratio = K[0] > 0.0 ? K[1] / K[0] : 0.0;            // shrinkage.py:72-82
        V.alpha = ratio > 1e-30 ? (ratio < 1e30 ? ratio : 1e30) : 1e-30;
        V.ix ^= 1; V.ig ^= 1; V.iax ^= 1;
        const double F = 0.5 * V.Q[0] + V.lam * V.Q[1];
        if (E.b == 0) {
          double* tr = a.trace + (size_t)(V.it - 1) * 4;
          tr[0] = (double)V.it; tr[1] = F; tr[2] = sqrt(V.Q[0]); tr[3] = K[6];
        }
        double kkt = K[4] > 0.0 ? K[2] : 0.0;
        if (K[5] > 0.0) kkt = pymax(pymax(kkt, K[3] - V.lam), 0.0);
        V.kkt = kkt;
        V.hist = V.hist < 2 ? V.hist + 1 : 2;
        if (kkt <= C.tol * V.lam) {                                      // shrinkage.py:167-170
          if (V.fin) V.conv = 1;
          V.active = 0;
          V.si++;
          if (V.fin || V.it >= C.max_iter) V.done = 1;      // shrinkage.py:175-176
        } else if (stop_fires(C.stop_kind, C.stop_thr, V.hist, F, V.Fprev, V.S[3], V.S[4], V.S[5],
                              C.gt_norm, kkt)) {
          V.conv = 1; V.done = 1;                                        // shrinkage.py:171-173
        }
        V.Fprev = F;
      }
      __syncthreads();
      if (V.done) break;
    }
  }
  T0 if (!V.done && V.status == ELL1_OK && a.max_steps > 0) V.status = ELL1_RUNNING;
  __syncthreads();

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    const bool save = V.status == ELL1_RUNNING;
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = Xp(V.ix)[k];
      if (save) { a.Xg[0][j] = Xp(0)[k]; a.Xg[1][j] = Xp(1)[k]; a.Gg[0][j] = Gp(0)[k]; a.Gg[1][j] = Gp(1)[k]; }
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
    st->rot[0] = V.si; st->rot[1] = V.active; st->rot[2] = V.ix; st->rot[3] = V.ig; st->rot[4] = V.iax;
    st->scal[I_ALPHA] = V.alpha; st->scal[I_LAM] = V.lam; st->scal[I_KKT] = V.kkt;
    st->scal[I_FPREV] = V.Fprev; st->scal[I_DF] = V.dF; st->scal[I_PASSES] = V.passes;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) ist_kernel(const __grid_constant__ IstArgs a) {
  ist_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_ist_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  return grid_bytes(nb, D->d, 1) + 4 * align_up(N * 8, 256) + 3 * align_up(D->ld * 8, 256) + 4096;
}

static int ist_setup(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, const double* stages,
                     int32_t nstages, const ell1_io_t* io, int nb, IstArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !C || !stages || nstages < 1 || !io || !io->state || !io->trace || !io->x)
    return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.C = *C;
  a.stages = stages;
  a.nstages = nstages;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  a.Xg[0] = cv.take<double>(N); a.Xg[1] = cv.take<double>(N);
  a.Gg[0] = cv.take<double>(N); a.Gg[1] = cv.take<double>(N);
  a.RC = cv.take<double>(D->ld);
  a.AXs[0] = cv.take<double>(D->ld); a.AXs[1] = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, IST_OV, 7, io->max_steps <= 0);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_ist(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
                        const double* stages, int32_t nstages, const ell1_io_t* io, void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  IstArgs a;
  SmemPlan sp;
  const int rc = ist_setup(D, b, C, stages, nstages, io, nb, a, sp);
  if (rc != ELL1_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->ld > D->d)
    if (cudaMemsetAsync(a.RC + D->d, 0, (D->ld - D->d) * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(ist_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(ist_kernel<float>, nb, sp.bytes, s, a, a.g.bar);
}

namespace ell1 {
template <class TA>
struct IstRun {
  static __device__ void run(const IstArgs& a) { ist_body<TA>(a); }
  static __device__ void reset(const IstArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    zero_pad_rows(a.RC, a.D.d, a.D.ld, lane);
  }
};
static_assert(sizeof(IstArgs) <= ELL1_GROUP_ARG_BYTES, "IstArgs too large for the group scratch");
}  // namespace ell1

int32_t ell1_ist_group_team_impl(const ell1_dict_t* D) {
  return dict_ok(D) ? group_team(to_raw(D), IST_OV, 7, 0) : 0;
}

extern "C" int ell1_ist_group(const ell1_group_t* G, const double* const* stages, const int32_t* nstages,
                              void* stream) {
  if (!G || (G->count > 0 && (!stages || !nstages))) return ELL1_ERR_ARG;
  return run_group<IstArgs, IstRun>(G, IST_OV, 7, 0, [&](int i, int nb, IstArgs& a, SmemPlan& sp) {
    return ist_setup(&G->dicts[i], G->b[i], &G->ctrl[i], stages[i], nstages[i], &G->io[i], nb, a, sp);
  }, stream);
}
