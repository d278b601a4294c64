// shard.cu — device primitives of the column-sharded single-instance FISTA
// (BASELINE config 4: A = [A_0 ... A_{G-1}] by columns, one rank per GPU, one
// NCCL allreduce of the d-length partial A x per iteration).
//
//   ell1_gemv        y = A x          (panel partials + fixed-order row reduction)
//   ell1_gemv_t      g = A^T r        (panel GEMV^T, local to each column)
//   ell1_shard_prox  x_next = soft(y - g_y/L, lam/L) over the local columns with
//                    the backtracking / stopping partial sums (shrinkage.py:199-213)
//   ell1_shard_resid r_next = (A x_next) - b, ||r||^2, ||r_y'||^2 (replicated d side)
//   ell1_shard_kkt   KKT / support partials of the local columns (model.py:160-173, 227-233)
// All reductions are deterministic (fixed order); scalar partials are
// returned per rank for the host driver to combine across ranks.
#include "solvers_common.cuh"

namespace ell1 {

struct GvArgs {
  DictRaw D;
  const double* x;
  double* y;
  GridBufs g;
};

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gemv_partial_kernel(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const double* xs[1] = {a.x + E.c0};
  panel_gemv<TA, 1>(E, D, PN, xs);
}

// y[r0(o) + j] = sum_c part[o][c][j] in fixed order (block o reduces the
// region of row slice o; 16-byte loads, consecutive threads -> consecutive rows)
__global__ void __launch_bounds__(NTHR) gemv_reduce_kernel(const double* part, int rp, int nb, int64_t d,
                                                           double* y) {
  const int o = blockIdx.x;
  const int64_t r0 = (d * o) / nb, r1 = (d * (o + 1)) / nb;
  const int rows = (int)(r1 - r0);
  const double* R = part + (size_t)o * nb * rp;
  for (int j = 2 * (int)threadIdx.x; j < rows; j += 2 * NTHR) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
    for (int c = 0; c < nb; ++c) {
      const double2 t = ldcg2(R + (size_t)c * rp + j);
      s0 += t.x;
      s1 += t.y;
    }
    y[r0 + j] = s0;
    if (j + 1 < rows) y[r0 + j + 1] = s1;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gemv_t_kernel(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const double* rs[1] = {a.x};
  double* os[1] = {a.y + E.c0};
  panel_gemv_t<TA, 1>(E, D, PN, rs, os);
}

// ---- elementwise + partial-sum kernels (grid-stride, CTA partials, then one CTA folds)
constexpr int SP = 8;

__global__ void __launch_bounds__(NTHR) shard_prox_kernel(int64_t n, const double* x, const double* xp,
                                                          const double* gx, const double* gxp, double* xn,
                                                          double m, double L, double thr, const double* gt,
                                                          double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};   // |xn|, gy.dl, dl.dl, max|xn|, (xn-x)^2, x^2, (xn-gt)^2, -
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = x[k];
    const double yk = xk + m * (xk - xp[k]);
    const double gk = (1.0 + m) * gx[k] - m * gxp[k];
    const double u = soft1(yk - gk / L, thr);
    xn[k] = u;
    const double dl = u - yk;
    s[0] += fabs(u);
    s[1] += gk * dl;
    s[2] += dl * dl;
    s[3] = nmax(s[3], fabs(u));
    const double dd = u - xk;
    s[4] += dd * dd;
    s[5] += xk * xk;
    if (gt) { const double e = u - gt[k]; s[6] += e * e; }
  }
  block_reduce<SP>(E, s, 1u << 3);
  if (threadIdx.x < SP) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

__global__ void __launch_bounds__(NTHR) shard_kkt_kernel(int64_t n, const double* x, const double* g, double lam,
                                                         double cut, double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};   // max_on, max_off, any_on, any_off, count, -, -, -
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = x[k];
    const double c = -g[k];
    if (xk != 0.0) { s[0] = nmax(s[0], fabs(c - lam * sgn(xk))); s[2] = 1.0; }
    else { s[1] = nmax(s[1], fabs(c)); s[3] = 1.0; }
    if (fabs(xk) > cut) s[4] += 1.0;
  }
  block_reduce<SP>(E, s, 0xFu);
  if (threadIdx.x < SP) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

__global__ void __launch_bounds__(NTHR) shard_resid_kernel(int64_t d, const double* ax, const double* b,
                                                           const double* rx, double mn, double* rn, double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * NTHR + threadIdx.x; i < d; i += (int64_t)gridDim.x * NTHR) {
    const double r = ax[i] - b[i];
    rn[i] = r;
    s[0] += r * r;
    const double ry = (1.0 + mn) * r - mn * rx[i];
    s[1] += ry * ry;
  }
  block_reduce<2>(E, s, 0u);
  if (threadIdx.x < 2) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

// fold CTA partials [nblk][SP] -> out[SP] (fixed order), maxmask selects max
__global__ void fold_kernel(const double* part, int nblk, unsigned maxmask, double* out) {
  const int k = threadIdx.x;
  if (k >= SP) return;
  const bool mx = (maxmask >> k) & 1u;
  double s = mx ? -INFINITY : 0.0;
  for (int c = 0; c < nblk; ++c) {
    const double t = part[(int64_t)c * SP + k];
    s = mx ? nmax(s, t) : s + t;
  }
  out[k] = s;
}

constexpr int EW_BLOCKS = 148 * 2;

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_gemv_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, D->d, 1) + (size_t)EW_BLOCKS * SP * 8 + 4096;
}

extern "C" int ell1_gemv(const ell1_dict_t* D, const double* x, double* y, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !x || !y) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, 0);
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = x; a.y = y;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_partial_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_partial_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  gemv_reduce_kernel<<<nb, NTHR, 0, s>>>(a.g.part, a.g.rp, nb, D->d, y);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_gemv_t(const ell1_dict_t* D, const double* r, double* g, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !r || !g) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, 0);
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = r; a.y = g;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_t_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_t_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

static int ew_blocks(int64_t n) {
  int64_t b = (n + NTHR - 1) / NTHR;
  if (b > EW_BLOCKS) b = EW_BLOCKS;
  return b < 1 ? 1 : (int)b;
}

extern "C" int ell1_shard_prox(int64_t n, const double* x, const double* xp, const double* gx,
                               const double* gxp, double* xn, double m, double L, double lam,
                               const double* gt, double* out8, void* ws, void* stream) {
  if (n < 0 || !out8 || !ws || !(L > 0)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(n);
  double* part = (double*)ws;
  shard_prox_kernel<<<nb, NTHR, 0, s>>>(n, x, xp, gx, gxp, xn, m, L, lam / L, gt, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 1u << 3, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_shard_kkt(int64_t n, const double* x, const double* g, double lam, double cut,
                              double* out8, void* ws, void* stream) {
  if (n < 0 || !out8 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(n);
  double* part = (double*)ws;
  shard_kkt_kernel<<<nb, NTHR, 0, s>>>(n, x, g, lam, cut, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 0xFu, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_shard_resid(int64_t d, const double* ax, const double* b, const double* rx, double mn,
                                double* rn, double* out8, void* ws, void* stream) {
  if (d < 0 || !out8 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(d);
  double* part = (double*)ws;
  shard_resid_kernel<<<nb, NTHR, 0, s>>>(d, ax, b, rx, mn, rn, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 0u, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
