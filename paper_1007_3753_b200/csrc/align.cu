// align.cu — alignment solvers batched across images.
//
// Reference: robust.py:223-515.  Each instance is a tall regression
// b ~ B w + e with sparse gross error e (B: d x m, m small — the
// transformation parameters of one image alignment step).  The reference
// solves one image per call with numpy; here a batch of images (each with
// its own B) runs in one launch, one CTA per image:
//   * B (row-major, numpy's layout) is staged in shared memory once as columns
//     of d + 1 doubles (odd stride: conflict-free staging and column walks);
//     the d-vectors (b, e, y / w-step residuals) live in registers, a fixed
//     set of rows per thread (RPT rows, 256 threads apart; RPT = 8 up to
//     d = 2048, 32 up to d = 8192);
//   * the column Gram G = B^T B is formed by fixed-order block reductions and
//     factored G = R^T R by warp 0 (not PD -> IllConditionedError, robust.py:254-258);
//   * every B^T v is one m-wide block reduction (lanes -> xor tree -> warps,
//     fixed order), every gram.solve two warp-parallel triangular solves.
// Solvers: PALM (the paper's choice for alignment, robust.py:470-515) and
// block IST (robust.py:427-467, step 1/alpha with alpha from the reference's
// power iteration on B^T B).
#include "ell1_b200.h"
#include "engine.cuh"
#include "solvers_common.cuh"

namespace ell1 {
namespace {

constexpr int AT = 256;                 // threads per image
constexpr int AW = AT / 32;
constexpr int MAXM = 32;                // columns of B (parameters) supported
// rows per thread kept in registers: RPT_S (d <= AT * RPT_S = 2048) for the
// common image sizes; RPT_L (d <= 8192) for large images (the d-vectors then
// partly live in local memory — correct, slower)
constexpr int RPT_S = 8;
constexpr int RPT_L = 32;
constexpr int MAXD = AT * RPT_L;

struct AlignSh {
  double red[AW][MAXM + 2];
  double out[MAXM + 2];
  double R[MAXM][MAXM];                 // upper Cholesky factor of B^T B
  double w[MAXM];
  double t[MAXM];
  int flag;
};

// sum over the CTA of k per-thread values (fixed order); results in S.out[0..k)
__device__ __forceinline__ void block_sum(AlignSh& S, double* v, int k) {
  const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int c = 0; c < k; ++c) {
    double s = v[c];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) S.red[wi][c] = s;
  }
  __syncthreads();
  if ((int)threadIdx.x < k) {
    double s = S.red[0][threadIdx.x];
    for (int ww = 1; ww < AW; ++ww) s += S.red[ww][threadIdx.x];
    S.out[threadIdx.x] = s;
  }
  __syncthreads();
}

// g = B^T v for the rows this thread holds; result in S.out[0..m)
template <int RPT>
__device__ __forceinline__ void bt_times(AlignSh& S, const double* Bs, int d, int m, const double (&v)[RPT]) {
  double p[MAXM];
  for (int c = 0; c < m; ++c) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = threadIdx.x + q * AT;
      if (i < d) s = fma(Bs[(int64_t)c * (d + 1) + i], v[q], s);
    }
    p[c] = s;
  }
  block_sum(S, p, m);
}

// S.w = G^{-1} S.out via R^T z = g, R w = z (warp 0; gram.solve, numerics.py:62-72)
__device__ __forceinline__ void gram_solve(AlignSh& S, int m) {
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    double z = l < m ? S.out[l] : 0.0;
    for (int i = 0; i < m; ++i) {                       // forward: R^T z = g
      const double zi = __shfl_sync(0xffffffffu, z, i) / S.R[i][i];
      if (l == i) z = zi;
      if (l > i && l < m) z = fma(-S.R[i][l], zi, z);
    }
    for (int i = m - 1; i >= 0; --i) {                  // backward: R w = z
      const double wi = __shfl_sync(0xffffffffu, z, i) / S.R[i][i];
      if (l == i) z = wi;
      if (l < i) z = fma(-S.R[l][i], wi, z);
    }
    if (l < m) S.w[l] = z;
  }
  __syncthreads();
}

// B's staging area of this CTA: shared memory, or (images whose (d+1) m
// doubles exceed the SM's shared memory) this CTA's slice of a.Bstage —
// the same column layout, read through L1/L2.
__device__ __forceinline__ double* stage_ptr(const ell1_align_t& a, double* sm) {
  return a.Bstage ? a.Bstage + (size_t)blockIdx.x * a.m * (a.d + 1) : sm;
}

__device__ __forceinline__ double soft(double x, double a) {
  return x > a ? x - a : (x < -a ? x + a : 0.0);          // _fastkernels.pyx:14-27
}

// stage B, form G = B^T B, factor; returns false (status set) when not PD
template <int RPT>
__device__ bool setup(AlignSh& S, double* Bs, const ell1_align_t& a, int j, double (&b)[RPT]) {
  const int d = a.d, m = a.m;
  const double* Bj = a.B + (int64_t)j * a.b_stride;
  for (int64_t t = threadIdx.x; t < (int64_t)d * m; t += AT) {   // row-major image, read coalesced
    const int64_t i = t / m, c = t - i * m;
    Bs[c * (d + 1) + i] = Bj[i * a.ldb + c];
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = threadIdx.x + q * AT;
    b[q] = i < d ? a.rhs[(int64_t)j * a.ld_rhs + i] : 0.0;
  }
  __syncthreads();
  for (int c = 0; c < m; ++c) {                          // row c of G (columns c..m-1)
    double p[MAXM];
    for (int k = c; k < m; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        if (i < d) s = fma(Bs[(int64_t)c * (d + 1) + i], Bs[(int64_t)k * (d + 1) + i], s);
      }
      p[k - c] = s;
    }
    block_sum(S, p, m - c);
    if ((int)threadIdx.x < m - c) S.R[c][c + threadIdx.x] = S.out[threadIdx.x];
    __syncthreads();
  }
  // upper Cholesky G = R^T R in place (warp 0, row-oriented)
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    int bad = 0;
    for (int i = 0; i < m; ++i) {
      double piv = S.R[i][i];
      for (int k = 0; k < i; ++k) piv -= S.R[k][i] * S.R[k][i];
      if (!(piv > 0.0)) { bad = 1; break; }
      const double rii = sqrt(piv);
      __syncwarp();
      if (l > i && l < m) {
        double v = S.R[i][l];
        for (int k = 0; k < i; ++k) v -= S.R[k][i] * S.R[k][l];
        S.R[i][l] = v / rii;
      }
      __syncwarp();
      if (l == 0) S.R[i][i] = rii;
      __syncwarp();
    }
    if (l == 0) S.flag = bad;
  }
  __syncthreads();
  if (S.flag) {
    if (threadIdx.x == 0) a.status[j] = ELL1_NOT_PD;
    return false;
  }
  return true;
}

template <int RPT>
__device__ __forceinline__ void store_out(const ell1_align_t& a, int j, const AlignSh& S, const double (&e)[RPT]) {
  if ((int)threadIdx.x < a.m) a.w[(int64_t)j * a.m + threadIdx.x] = S.w[threadIdx.x];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = threadIdx.x + q * AT;
    if (i < a.d) a.e[(int64_t)j * a.d + i] = e[q];
  }
}

// ---------------------------------------------------------------- PALM
// robust.py:470-515: w = G^{-1} B^T (b - e + y/mu); e = soft(b - Bw + y/mu, 1/mu)
// (inner sweeps to 1e-2/mu relative change, <= 100 per mu), y += mu r, mu *= rho
template <int RPT>
__global__ void __launch_bounds__(AT) align_palm_kernel(const ell1_align_t a) {
  extern __shared__ double Bsm[];
  double* const Bs = stage_ptr(a, Bsm);
  __shared__ AlignSh S;
  const int d = a.d, m = a.m;
  for (int j = blockIdx.x; j < a.count; j += gridDim.x) {
    double b[RPT], e[RPT], y[RPT], bw[RPT], tv[RPT];
    if (!setup(S, Bs, a, j, b)) continue;
    double bb = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) { e[q] = 0.0; y[q] = 0.0; bb = fma(b[q], b[q], bb); }
    block_sum(S, &bb, 1);
    const double bnorm = sqrt(S.out[0]);
    bt_times(S, Bs, d, m, b);
    gram_solve(S, m);                                    // w = gram.solve(B^T b)
    int it = 0;
    if (bnorm != 0.0) {
      double mu = a.mu0;
      while (it < a.max_iter) {
        const int inner = a.max_iter - it < 100 ? a.max_iter - it : 100;
        for (int s = 0; s < inner; ++s) {
          ++it;
#pragma unroll
          for (int q = 0; q < RPT; ++q) tv[q] = b[q] - e[q] + y[q] / mu;
          bt_times(S, Bs, d, m, tv);
          gram_solve(S, m);
          double nrm[2] = {0.0, 0.0};                    // ||e_new - e||^2, ||e_new||^2
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int i = threadIdx.x + q * AT;
            double s2 = 0.0;
            if (i < d)
              for (int c = 0; c < m; ++c) s2 = fma(Bs[(int64_t)c * (d + 1) + i], S.w[c], s2);
            bw[q] = s2;
            const double en = i < d ? soft(b[q] - s2 + y[q] / mu, 1.0 / mu) : 0.0;
            const double df = en - e[q];
            nrm[0] = fma(df, df, nrm[0]);
            nrm[1] = fma(en, en, nrm[1]);
            e[q] = en;
          }
          block_sum(S, nrm, 2);
          const double change = sqrt(S.out[0]), en2 = sqrt(S.out[1]);
          if (change <= 1e-2 / mu * (en2 > 1.0 ? en2 : 1.0)) break;
        }
        double rr = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const double r = b[q] - bw[q] - e[q];
          y[q] = fma(mu, r, y[q]);
          rr = fma(r, r, rr);
        }
        block_sum(S, &rr, 1);
        if (sqrt(S.out[0]) <= a.tol * bnorm) break;
        mu *= a.rho;
      }
    }
    store_out(a, j, S, e);
    if (threadIdx.x == 0) { a.status[j] = ELL1_OK; if (a.iterations) a.iterations[j] = it; }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- block IST
// robust.py:427-467: w += B^T r / alpha, e = soft(e + r/alpha, lam/alpha); stop
// when max|B^T r| <= tol and kkt(e, r, lam) <= tol lam.  alpha = 1.01 (||B||^2 + 1)
// with ||B||^2 from the reference's power iteration (numerics.py:224-261) run on
// B^T (B v) from the host-drawn start vectors.
template <int RPT>
__global__ void __launch_bounds__(AT) align_ist_kernel(const ell1_align_t a) {
  extern __shared__ double Bsm[];
  double* const Bs = stage_ptr(a, Bsm);
  __shared__ AlignSh S;
  __shared__ double v[MAXM];
  const int d = a.d, m = a.m;
  for (int j = blockIdx.x; j < a.count; j += gridDim.x) {
    double b[RPT], e[RPT], r[RPT];
    if (!setup(S, Bs, a, j, b)) continue;
    // lambda: 1e-2 max|b - B w0|, w0 = gram.solve(B^T b) (robust.py:270-273)
    double lam = a.lam;
    if (!(lam > 0.0)) {
      bt_times(S, Bs, d, m, b);
      gram_solve(S, m);
      double mx = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        if (i < d) {
          double s2 = 0.0;
          for (int c = 0; c < m; ++c) s2 = fma(Bs[(int64_t)c * (d + 1) + i], S.w[c], s2);
          mx = nmax(mx, fabs(b[q] - s2));
        }
      }
      mx = warp_max(mx);
      if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5][0] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = S.red[0][0];
        for (int ww = 1; ww < AW; ++ww) t = nmax(t, S.red[ww][0]);
        S.out[0] = 1e-2 * t;
      }
      __syncthreads();
      lam = S.out[0];
    }
    // power iteration on B^T B (spectral_norm_sq, dim = m < d)
    int draw = 0;
    if ((int)threadIdx.x < m) v[threadIdx.x] = a.v0[threadIdx.x];
    __syncthreads();
    double theta = 0.0;
    for (int k = 0; k < 1000; ++k) {
      double u[RPT];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        double s2 = 0.0;
        if (i < d)
          for (int c = 0; c < m; ++c) s2 = fma(Bs[(int64_t)c * (d + 1) + i], v[c], s2);
        u[q] = s2;
      }
      bt_times(S, Bs, d, m, u);                          // S.out = B^T (B v)
      if (threadIdx.x == 0) {
        double th = 0.0, res = 0.0, nw = 0.0;
        for (int c = 0; c < m; ++c) th = fma(v[c], S.out[c], th);
        for (int c = 0; c < m; ++c) { const double t = S.out[c] - th * v[c]; res = fma(t, t, res); }
        for (int c = 0; c < m; ++c) nw = fma(S.out[c], S.out[c], nw);
        S.t[0] = th;
        S.t[1] = sqrt(res);
        S.t[2] = sqrt(nw);
      }
      __syncthreads();
      theta = S.t[0];
      if (S.t[1] <= 1e-6 * (theta > 2.2250738585072014e-308 ? theta : 2.2250738585072014e-308)) break;
      const double nw = S.t[2];
      __syncthreads();
      if (nw == 0.0) ++draw;                             // start vector in the nullspace: next draw
      if ((int)threadIdx.x < m)
        v[threadIdx.x] = nw == 0.0 ? a.v0[(draw % 4) * m + threadIdx.x] : S.out[threadIdx.x] / nw;
      __syncthreads();
    }
    const double alpha = 1.01 * (theta + 1.0);
    // iterate from w = 0, e = 0 (robust.py:457-466)
    if ((int)threadIdx.x < m) S.w[threadIdx.x] = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) { e[q] = 0.0; r[q] = b[q]; }
    __syncthreads();
    bt_times(S, Bs, d, m, r);                            // B^T r at (0, 0)
    int it = 0;
    for (; it < a.max_iter;) {
      ++it;
      if ((int)threadIdx.x < m) S.w[threadIdx.x] += S.out[threadIdx.x] / alpha;
#pragma unroll
      for (int q = 0; q < RPT; ++q) e[q] = soft(e[q] + r[q] / alpha, lam / alpha);
      __syncthreads();
      double kk = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        double s2 = 0.0;
        if (i < d)
          for (int c = 0; c < m; ++c) s2 = fma(Bs[(int64_t)c * (d + 1) + i], S.w[c], s2);
        r[q] = i < d ? b[q] - s2 - e[q] : 0.0;
        if (i < d) {                                     // kkt_from_correlation(e, r, lam), model.py:160-173
          const double viol = e[q] != 0.0 ? fabs(r[q] - lam * (e[q] > 0.0 ? 1.0 : -1.0))
                                          : fabs(r[q]) - lam;
          kk = nmax(kk, viol);
        }
      }
      kk = warp_max(kk);
      bt_times(S, Bs, d, m, r);                          // also the next step's gradient
      if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5][MAXM + 1] = kk;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = S.red[0][MAXM + 1], g = 0.0;
        for (int ww = 1; ww < AW; ++ww) t = nmax(t, S.red[ww][MAXM + 1]);
        for (int c = 0; c < m; ++c) g = nmax(g, fabs(S.out[c]));
        S.flag = g <= a.tol && nmax(t, 0.0) <= a.tol * lam;
      }
      __syncthreads();
      if (S.flag) break;
    }
    store_out(a, j, S, e);
    if (threadIdx.x == 0) { a.status[j] = ELL1_OK; if (a.iterations) a.iterations[j] = it; }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- homotopy
// robust.py:374-424: walk the weight down from the peak least-squares
// residual, moving the active error coordinates along their sign between
// events, re-solving w from the normal equations after each step; then a
// block-coordinate cleanup at the target weight.
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void block_min2(AlignSh& S, double v0, double v1) {
  v0 = warp_min(v0);
  v1 = warp_min(v1);
  if ((threadIdx.x & 31) == 0) { S.red[threadIdx.x >> 5][0] = v0; S.red[threadIdx.x >> 5][1] = v1; }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = S.red[0][threadIdx.x];
    for (int ww = 1; ww < AW; ++ww) t = fmin(t, S.red[ww][threadIdx.x]);
    S.out[threadIdx.x] = t;
  }
  __syncthreads();
}

template <int RPT>
__global__ void __launch_bounds__(AT) align_homotopy_kernel(const ell1_align_t a) {
  extern __shared__ double Bsm[];
  double* const Bs = stage_ptr(a, Bsm);
  __shared__ AlignSh S;
  const int d = a.d, m = a.m;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  for (int j = blockIdx.x; j < a.count; j += gridDim.x) {
    double b[RPT], e[RPT], c[RPT], tv[RPT], rb[RPT];
    if (!setup(S, Bs, a, j, b)) continue;
    // w = w_solve(e) (robust.py:386-387); rb = b - B w, c = rb - e
    auto w_solve_c = [&]() {
#pragma unroll
      for (int q = 0; q < RPT; ++q) tv[q] = b[q] - e[q];
      bt_times(S, Bs, d, m, tv);
      gram_solve(S, m);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        double s2 = 0.0;
        if (i < d)
          for (int k = 0; k < m; ++k) s2 = fma(Bs[(int64_t)k * (d + 1) + i], S.w[k], s2);
        rb[q] = i < d ? b[q] - s2 : 0.0;
        c[q] = rb[q] - e[q];
      }
    };
#pragma unroll
    for (int q = 0; q < RPT; ++q) e[q] = 0.0;
    w_solve_c();
    double mx = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) mx = nmax(mx, fabs(c[q]));
    block_min2(S, -mx, 0.0);
    const double lam0 = -S.out[0];
    const double target = a.lam > 0.0 ? a.lam : 1e-2 * lam0;
    int it = 0;
    if (!(lam0 <= target || lam0 == 0.0)) {
      double lam = lam0;
      for (; it < a.max_iter; ++it) {
        if (lam <= target) break;
        // gamma = min(lam - target, min_inactive(lam - |c|), min_closing(-e / dir))
        double g_in = INF, g_cl = INF;
        bool act[RPT];
        double dir[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          const double ac = fabs(c[q]);
          act[q] = i < d && (ac >= lam * (1.0 - 1e-9) || e[q] != 0.0);
          dir[q] = ac > 0.0 ? (c[q] > 0.0 ? 1.0 : -1.0) : (e[q] > 0.0 ? 1.0 : (e[q] < 0.0 ? -1.0 : 0.0));
          if (i < d && !act[q]) g_in = fmin(g_in, lam - ac);
          if (act[q] && e[q] * dir[q] < 0.0) g_cl = fmin(g_cl, -e[q] / dir[q]);
        }
        block_min2(S, g_in, g_cl);
        double gamma = lam - target;
        gamma = fmin(gamma, S.out[0]);
        gamma = fmin(gamma, S.out[1]);
        gamma = nmax(gamma, 1e-12 * lam0);                 // anti-stall floor
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          if (act[q]) e[q] = e[q] + gamma * dir[q];
        lam = lam - gamma;
        w_solve_c();
      }
      // block-coordinate cleanup at the target weight
      lam = target;
      for (int k = 0; k < a.max_iter; ++k) {
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          e[q] = i < d ? soft(rb[q], lam) : 0.0;
        }
        w_solve_c();
        double kk = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          if (i < d) {
            const double viol = e[q] != 0.0 ? fabs(c[q] - lam * (e[q] > 0.0 ? 1.0 : -1.0)) : fabs(c[q]) - lam;
            kk = nmax(kk, viol);
          }
        }
        block_min2(S, -kk, 0.0);
        if (nmax(-S.out[0], 0.0) <= a.tol * lam) break;
      }
    }
    store_out(a, j, S, e);
    if (threadIdx.x == 0) { a.status[j] = ELL1_OK; if (a.iterations) a.iterations[j] = it; }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- barrier Newton (gp)
// robust.py:276-371: log-barrier walk of the central path in (w, e, u) with
// -u <= e <= u; the bound and error blocks are eliminated so each Newton step
// factors one m x m weighted Gram B^T diag(weight) B; Armijo backtracking
// (<= 50 halvings, slope 0.01); t x 10 when the decrement^2 <= 1/4; exit
// through the polished iterate (e truncated at 1e-7 max|e|, w re-solved).
__device__ __forceinline__ double block_sum1(AlignSh& S, double v) {
  block_sum(S, &v, 1);
  return S.out[0];
}

// upper Cholesky of the weighted Gram B^T diag(wt) B into S.R; false if not PD
template <int RPT>
__device__ bool weighted_gram_factor(AlignSh& S, const double* Bs, int d, int m, const double (&wt)[RPT]) {
  for (int c = 0; c < m; ++c) {
    double p[MAXM];
    for (int k = c; k < m; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        if (i < d) s = fma(Bs[(int64_t)c * (d + 1) + i] * wt[q], Bs[(int64_t)k * (d + 1) + i], s);
      }
      p[k - c] = s;
    }
    block_sum(S, p, m - c);
    if ((int)threadIdx.x < m - c) S.R[c][c + threadIdx.x] = S.out[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    int bad = 0;
    for (int i = 0; i < m; ++i) {
      double piv = S.R[i][i];
      for (int k = 0; k < i; ++k) piv -= S.R[k][i] * S.R[k][i];
      if (!(piv > 0.0)) { bad = 1; break; }
      const double rii = sqrt(piv);
      __syncwarp();
      if (l > i && l < m) {
        double v = S.R[i][l];
        for (int k = 0; k < i; ++k) v -= S.R[k][i] * S.R[k][l];
        S.R[i][l] = v / rii;
      }
      __syncwarp();
      if (l == 0) S.R[i][i] = rii;
      __syncwarp();
    }
    if (l == 0) S.flag = bad;
  }
  __syncthreads();
  return !S.flag;
}

template <int RPT>
__global__ void __launch_bounds__(AT) align_gp_kernel(const ell1_align_t a) {
  extern __shared__ double Bsm[];
  double* const Bs = stage_ptr(a, Bsm);
  __shared__ AlignSh S;
  __shared__ double R0[MAXM][MAXM];        // factor of B^T B (the step factor reuses S.R)
  __shared__ double wv[MAXM], dw[MAXM];
  const int d = a.d, m = a.m;
  for (int j = blockIdx.x; j < a.count; j += gridDim.x) {
    double b[RPT], e[RPT], u[RPT], r[RPT];
    if (!setup(S, Bs, a, j, b)) continue;
    for (int t = threadIdx.x; t < MAXM * MAXM; t += AT) R0[t / MAXM][t % MAXM] = S.R[t / MAXM][t % MAXM];
    __syncthreads();
    auto use_gram = [&]() {
      for (int t = threadIdx.x; t < MAXM * MAXM; t += AT) S.R[t / MAXM][t % MAXM] = R0[t / MAXM][t % MAXM];
      __syncthreads();
    };
    // B w for this thread's rows from a shared m-vector
    auto bmul = [&](const double* vec, double (&out)[RPT]) {
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        double s2 = 0.0;
        if (i < d)
          for (int k = 0; k < m; ++k) s2 = fma(Bs[(int64_t)k * (d + 1) + i], vec[k], s2);
        out[q] = s2;
      }
    };
    double tmp[RPT];
    // lambda default: 1e-2 max|b - B w0| (robust.py:270-273)
    bt_times(S, Bs, d, m, b);
    gram_solve(S, m);
    if ((int)threadIdx.x < m) wv[threadIdx.x] = S.w[threadIdx.x];
    __syncthreads();
    double lam = a.lam;
    double bmax = 0.0;
    {
      bmul(wv, tmp);
      double mx = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        if (i < d) { mx = nmax(mx, fabs(b[q] - tmp[q])); bmax = nmax(bmax, fabs(b[q])); }
      }
      block_min2(S, -mx, -bmax);
      if (!(lam > 0.0)) lam = 1e-2 * (-S.out[0]);
      bmax = -S.out[1];
    }
    int status = ELL1_OK, it = 0;
    // polished(e): truncate |e| <= 1e-7 max|e|, w = gram.solve(B^T (b - e_t)); returns kkt <= tol lam
    auto polish = [&](double (&et)[RPT]) -> bool {
      double mx = 0.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) mx = nmax(mx, fabs(e[q]));
      block_min2(S, -mx, 0.0);
      const double top = -S.out[0];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        et[q] = (top > 0.0 && fabs(e[q]) <= 1e-7 * top) ? 0.0 : e[q];
        tmp[q] = b[q] - et[q];
      }
      use_gram();
      bt_times(S, Bs, d, m, tmp);
      gram_solve(S, m);
      double kk = 0.0;
      bmul(S.w, tmp);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int i = threadIdx.x + q * AT;
        if (i < d) {
          const double c = b[q] - tmp[q] - et[q];
          const double viol = et[q] != 0.0 ? fabs(c - lam * (et[q] > 0.0 ? 1.0 : -1.0)) : fabs(c) - lam;
          kk = nmax(kk, viol);
        }
      }
      block_min2(S, -kk, 0.0);
      return nmax(-S.out[0], 0.0) <= a.tol * lam;
    };
    double et[RPT];
    bool done = false;
    if (!(lam > 0.0)) {
      status = ELL1_LAMBDA_NONPOS;
    } else {
      double t = 1.0 / lam;
      const double u0 = bmax > 1.0 ? bmax : 1.0;
#pragma unroll
      for (int q = 0; q < RPT; ++q) { e[q] = 0.0; u[q] = u0; }
      for (; it < a.max_iter; ++it) {
        bmul(wv, tmp);
        double rr = 0.0, ae = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          r[q] = i < d ? b[q] - tmp[q] - e[q] : 0.0;
          rr = fma(r[q], r[q], rr);
          ae += fabs(e[q]);
        }
        double v2[2] = {rr, ae};
        block_sum(S, v2, 2);
        const double rr_all = S.out[0];
        const double obj = 0.5 * rr_all + lam * S.out[1];
        if (2.0 * d / t <= a.tol * (1.0 + obj)) {
          if (polish(et)) { done = true; break; }
        }
        // Newton system (robust.py:307-330)
        double g_e[RPT], g_u[RPT], dsum[RPT], ddiff[RPT], rhs_e[RPT], den[RPT], wt[RPT], up[RPT], um[RPT];
        double lsum = 0.0, usum = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          if (i < d) {
            up[q] = u[q] + e[q];
            um[q] = u[q] - e[q];
            const double p = 1.0 / up[q], qq_ = 1.0 / um[q];
            g_e[q] = -t * r[q] + (qq_ - p);
            g_u[q] = t * lam - p - qq_;
            const double pp = p * p, qq = qq_ * qq_;
            dsum[q] = pp + qq;
            ddiff[q] = pp - qq;
            const double dred = 4.0 * pp * qq / dsum[q];
            rhs_e[q] = -g_e[q] + ddiff[q] * (g_u[q] / dsum[q]);
            den[q] = t + dred;
            wt[q] = t * dred / den[q];
            lsum += log(up[q]) + log(um[q]);
            usum += u[q];
          } else {
            up[q] = um[q] = 1.0; g_e[q] = g_u[q] = dsum[q] = ddiff[q] = rhs_e[q] = 0.0; den[q] = 1.0; wt[q] = 0.0;
          }
        }
        // g_w = -t B^T r
        bt_times(S, Bs, d, m, r);
        double gw[MAXM];
        for (int c = 0; c < m; ++c) gw[c] = -t * S.out[c];
        // rhs_w = -g_w - t B^T (rhs_e / den)
#pragma unroll
        for (int q = 0; q < RPT; ++q) tmp[q] = rhs_e[q] / den[q];
        bt_times(S, Bs, d, m, tmp);
        double rw[MAXM];
        for (int c = 0; c < m; ++c) rw[c] = -gw[c] - t * S.out[c];
        if (!weighted_gram_factor(S, Bs, d, m, wt)) { status = ELL1_ILL_CONDITIONED; break; }
        if ((int)threadIdx.x < m) S.out[threadIdx.x] = rw[threadIdx.x];
        __syncthreads();
        gram_solve(S, m);                                  // dw = step_fac.solve(...)
        if ((int)threadIdx.x < m) dw[threadIdx.x] = S.w[threadIdx.x];
        __syncthreads();
        double bdw[RPT], de[RPT], du[RPT];
        bmul(dw, bdw);
        double dec = 0.0, smin[2] = {1.0, 1.0};
        // 0.99 min(up/-dup) over dup < 0, same for um (fraction to the boundary)
        double f1 = __longlong_as_double(0x7ff0000000000000LL), f2 = f1;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = threadIdx.x + q * AT;
          if (i < d) {
            de[q] = (rhs_e[q] - t * bdw[q]) / den[q];
            du[q] = -(g_u[q] + ddiff[q] * de[q]) / dsum[q];
            dec += g_e[q] * de[q] + g_u[q] * du[q];
            const double dup = du[q] + de[q], dum = du[q] - de[q];
            if (dup < 0.0) f1 = fmin(f1, up[q] / -dup);
            if (dum < 0.0) f2 = fmin(f2, um[q] / -dum);
          } else {
            de[q] = du[q] = 0.0;
          }
        }
        (void)smin;
        double v3[3] = {dec, lsum, usum};
        block_sum(S, v3, 3);
        double gwdw = 0.0;
        for (int c = 0; c < m; ++c) gwdw = fma(gw[c], dw[c], gwdw);
        const double decrement_sq = -(gwdw + S.out[0]);
        const double F_t = t * (0.5 * rr_all + lam * S.out[2]) - S.out[1];
        block_min2(S, f1, f2);
        double sstep = 1.0;
        if (S.out[0] < __longlong_as_double(0x7ff0000000000000LL)) sstep = fmin(sstep, 0.99 * S.out[0]);
        if (S.out[1] < __longlong_as_double(0x7ff0000000000000LL)) sstep = fmin(sstep, 0.99 * S.out[1]);
        // Armijo backtracking (<= 50 halvings, robust.py:346-366)
        bool accepted = false;
        double en[RPT], un[RPT];
        for (int h = 0; h <= 50; ++h) {
          double mn1 = __longlong_as_double(0x7ff0000000000000LL), mn2 = mn1;
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int i = threadIdx.x + q * AT;
            en[q] = e[q] + sstep * de[q];
            un[q] = u[q] + sstep * du[q];
            if (i < d) { mn1 = fmin(mn1, un[q] + en[q]); mn2 = fmin(mn2, un[q] - en[q]); }
          }
          block_min2(S, mn1, mn2);
          if (S.out[0] > 0.0 && S.out[1] > 0.0) {
            double rn2 = 0.0, us = 0.0, ls = 0.0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
              const int i = threadIdx.x + q * AT;
              if (i < d) {
                const double rn = r[q] - sstep * bdw[q] - sstep * de[q];
                rn2 = fma(rn, rn, rn2);
                us += un[q];
                ls += log(un[q] + en[q]) + log(un[q] - en[q]);
              }
            }
            double v4[3] = {rn2, us, ls};
            block_sum(S, v4, 3);
            const double F_new = t * (0.5 * S.out[0] + lam * S.out[1]) - S.out[2];
            if (F_new <= F_t - 0.01 * sstep * decrement_sq) { accepted = true; break; }
          }
          sstep *= 0.5;
        }
        if (!accepted) { status = ELL1_BREAKDOWN; break; }
        if ((int)threadIdx.x < m) wv[threadIdx.x] += sstep * dw[threadIdx.x];
#pragma unroll
        for (int q = 0; q < RPT; ++q) { e[q] = en[q]; u[q] = un[q]; }
        __syncthreads();
        if (decrement_sq <= 0.25) t *= 10.0;
      }
      if (status == ELL1_OK && !done) polish(et);           // budget exhausted: polished(e)
    }
    if (status == ELL1_OK) {
      store_out(a, j, S, et);
    }
    if (threadIdx.x == 0) { a.status[j] = status; if (a.iterations) a.iterations[j] = it; }
    __syncthreads();
  }
}

// robust.ist_block_step (robust.py:433-445): one block soft-threshold sweep,
// r = b - B w - e, w' = w + B^T r / alpha, e' = soft(e + r / alpha, lam / alpha);
// one CTA, any d (rows strided over the threads), fixed-order reductions.
__global__ void __launch_bounds__(AT) align_ist_step_kernel(int d, int m, const double* __restrict__ B, int64_t ldb,
                                                            const double* __restrict__ b, const double* __restrict__ w,
                                                            const double* __restrict__ e, double lam, double alpha,
                                                            double* __restrict__ w_next, double* __restrict__ e_next) {
  __shared__ AlignSh S;
  if (threadIdx.x < MAXM) S.w[threadIdx.x] = threadIdx.x < (unsigned)m ? w[threadIdx.x] : 0.0;
  __syncthreads();
  double p[MAXM];
  for (int c = 0; c < MAXM; ++c) p[c] = 0.0;
  for (int i = threadIdx.x; i < d; i += AT) {
    const double* Bi = B + (int64_t)i * ldb;
    double bw = 0.0;
    for (int c = 0; c < m; ++c) bw = fma(Bi[c], S.w[c], bw);
    const double r = b[i] - bw - e[i];
    e_next[i] = soft(e[i] + r / alpha, lam / alpha);
    for (int c = 0; c < m; ++c) p[c] = fma(Bi[c], r, p[c]);
  }
  block_sum(S, p, m);
  if ((int)threadIdx.x < m) w_next[threadIdx.x] = S.w[threadIdx.x] + S.out[threadIdx.x] / alpha;
}

template <int RPT>
const void* align_kernel_t(int kind) {
  return kind == 0   ? (const void*)align_palm_kernel<RPT>
         : kind == 1 ? (const void*)align_ist_kernel<RPT>
         : kind == 2 ? (const void*)align_homotopy_kernel<RPT>
                     : (const void*)align_gp_kernel<RPT>;
}

// test hook (ell1_test_align_large_rows): run every image through the
// RPT_L variant — bit-identical to RPT_S where both apply (same row map and
// accumulation order; the extra row slots are masked)
int g_force_large = 0;

bool use_large(int d) { return g_force_large || d > AT * RPT_S; }

const void* align_kernel(int kind, int d) {
  return use_large(d) ? align_kernel_t<RPT_L>(kind) : align_kernel_t<RPT_S>(kind);
}

// launch geometry: shared-memory staging when it fits next to the kernel's
// static shared memory, else global staging (grid CTAs x (d+1) m doubles)
struct AlignPlan {
  size_t smem;        // dynamic shared memory of the launch
  int grid;
  size_t stage;       // bytes of global staging (0: shared)
};

bool align_plan(int kind, int count, int d, int m, AlignPlan& P) {
  const void* k = align_kernel(kind, d);
  int dev = 0, sms = 148, optin = 0, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return false;
  const size_t need = (size_t)(d + 1) * m * 8;
  const bool shared = need + fa.sharedSizeBytes <= (size_t)optin;
  P.smem = shared ? need : 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem) != cudaSuccess)
    return false;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, AT, P.smem);
  P.grid = sms * (per > 0 ? per : 1);
  if (P.grid > count) P.grid = count;
  P.stage = shared ? 0 : need * (size_t)P.grid;
  return true;
}

int launch_align(int kind, const ell1_align_t* A, void* stream) {
  if (!A || A->count < 0 || A->m < 1 || A->m > MAXM || A->d <= A->m || A->d > MAXD || !A->B || !A->rhs ||
      !A->w || !A->e || !A->status || A->ldb < A->m || A->ld_rhs < A->d || A->b_stride < A->ldb * A->d)
    return ELL1_ERR_ARG;
  if (kind == 1 && !A->v0) return ELL1_ERR_ARG;
  if (A->count == 0) return ELL1_OK;
  AlignPlan P;
  if (!align_plan(kind, A->count, A->d, A->m, P)) return ELL1_ERR_CUDA;
  ell1_align_t a = *A;
  if (P.stage == 0) a.Bstage = nullptr;
  else if (!A->Bstage) return ELL1_ERR_ARG;            // caller must provide ell1_align_stage_bytes()
  cudaStream_t s = (cudaStream_t)stream;
  if (!use_large(a.d)) {
    if (kind == 0) align_palm_kernel<RPT_S><<<P.grid, AT, P.smem, s>>>(a);
    else if (kind == 1) align_ist_kernel<RPT_S><<<P.grid, AT, P.smem, s>>>(a);
    else if (kind == 2) align_homotopy_kernel<RPT_S><<<P.grid, AT, P.smem, s>>>(a);
    else align_gp_kernel<RPT_S><<<P.grid, AT, P.smem, s>>>(a);
  } else {
    if (kind == 0) align_palm_kernel<RPT_L><<<P.grid, AT, P.smem, s>>>(a);
    else if (kind == 1) align_ist_kernel<RPT_L><<<P.grid, AT, P.smem, s>>>(a);
    else if (kind == 2) align_homotopy_kernel<RPT_L><<<P.grid, AT, P.smem, s>>>(a);
    else align_gp_kernel<RPT_L><<<P.grid, AT, P.smem, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

}  // namespace
}  // namespace ell1

extern "C" size_t ell1_align_stage_bytes(int32_t kind, int32_t count, int32_t d, int32_t m) {
  if (kind < 0 || kind > 3 || count <= 0 || m < 1 || m > ell1::MAXM || d <= m || d > ell1::MAXD) return 0;
  ell1::AlignPlan P;
  if (!ell1::align_plan(kind, count, d, m, P)) return 0;
  return P.stage;
}

extern "C" int ell1_align_ist_step(int32_t d, int32_t m, const double* B, int64_t ldb, const double* b,
                                   const double* w, const double* e, double lam, double alpha, double* w_next,
                                   double* e_next, void* stream) {
  if (d < 1 || m < 1 || m > ell1::MAXM || ldb < m || !B || !b || !w || !e || !w_next || !e_next || !(alpha > 0))
    return ELL1_ERR_ARG;
  ell1::align_ist_step_kernel<<<1, ell1::AT, 0, (cudaStream_t)stream>>>(d, m, B, ldb, b, w, e, lam, alpha, w_next,
                                                                        e_next);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" void ell1_test_align_large_rows(int32_t on) { ell1::g_force_large = on != 0; }

extern "C" int ell1_align_palm_batch(const ell1_align_t* A, void* stream) {
  return ell1::launch_align(0, A, stream);
}

extern "C" int ell1_align_ist_batch(const ell1_align_t* A, void* stream) {
  return ell1::launch_align(1, A, stream);
}

extern "C" int ell1_align_homotopy_batch(const ell1_align_t* A, void* stream) {
  return ell1::launch_align(2, A, stream);
}

extern "C" int ell1_align_gp_batch(const ell1_align_t* A, void* stream) {
  return ell1::launch_align(3, A, stream);
}
