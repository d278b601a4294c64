// shard_hom.cu — device reductions of the column-sharded single-instance
// Homotopy (reference homotopy.py:128-244).
//
// The dictionary is split by columns across ranks; the two A^T passes per
// breakpoint (homotopy.py:186-188 correlation, :225-226 w = A^T v) run on each
// rank's panel (ell1_gemv_t), the active columns A_I, the factor and x_I are
// replicated.  These kernels produce the per-rank candidates that are folded
// across ranks (first index wins ties, as numpy's argmin/argmax):
//   ell1_hom_absmax     max |c| and its first index              (lambda_0, j_0, lam_emp)
//   ell1_hom_gammas     add-event step lengths on the rank's off-support columns
//                       (homotopy.py:78-105: (lam -+ c) / (1 -+ w), floor 1e-10 lam)
//   ell1_hom_gamma_minus  remove-event step length over the (replicated) support
//   ell1_hom_xstats     sum |x_I|, support count at 1e-10 max(max|x|, 1) (model.py:227-233)
// One CTA each, rows strided over the threads in increasing order, then a
// fixed-order (value, index) reduction: deterministic and rank-independent.
#include <cmath>
#include "ell1_b200.h"
#include "engine.cuh"

namespace ell1 {
namespace {

constexpr int HT = 1024;

// (value, index) min with the lower index on ties; idx < 0 = empty
__device__ __forceinline__ void vi_min(double& v, long long& i, double v2, long long i2) {
  if (i2 < 0) return;
  if (i < 0 || v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}
__device__ __forceinline__ void vi_max(double& v, long long& i, double v2, long long i2) {
  if (i2 < 0) return;
  if (i < 0 || v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

template <bool MAX>
__device__ __forceinline__ void block_vi(double& v, long long& i) {
  __shared__ double sv[HT / 32];
  __shared__ long long si[HT / 32];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (MAX) vi_max(v, i, v2, i2); else vi_min(v, i, v2, i2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sv[w] = v; si[w] = i; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      if (MAX) vi_max(v, i, sv[k], si[k]); else vi_min(v, i, sv[k], si[k]);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(HT) hom_absmax_kernel(int64_t n, const double* __restrict__ c, double* out) {
  double v = 0.0;
  long long i = -1;
  for (int64_t k = threadIdx.x; k < n; k += HT) vi_max(v, i, fabs(c[k]), k);
  block_vi<true>(v, i);
  if (threadIdx.x == 0) { out[0] = i < 0 ? 0.0 : v; out[1] = (double)i; }
}

// off-support add events: ra = (lam - c) / (1 - w), rb = (lam + c) / (1 + w)
__global__ void __launch_bounds__(HT) hom_gammas_kernel(int64_t n, const double* __restrict__ c,
                                                        const double* __restrict__ w,
                                                        const unsigned char* __restrict__ mask, double lam,
                                                        double* out) {
  const double floor = 1e-10 * (lam > 1e-30 ? lam : 1e-30);
  double va = INFINITY, vb = INFINITY;
  long long ia = -1, ib = -1;
  for (int64_t k = threadIdx.x; k < n; k += HT) {
    if (mask[k]) continue;
    const double ra = (lam - c[k]) / (1.0 - w[k]);
    const double rb = (lam + c[k]) / (1.0 + w[k]);
    if (isfinite(ra) && ra > floor) vi_min(va, ia, ra, k);
    if (isfinite(rb) && rb > floor) vi_min(vb, ib, rb, k);
  }
  block_vi<false>(va, ia);
  block_vi<false>(vb, ib);
  if (threadIdx.x == 0) {
    out[0] = ia < 0 ? INFINITY : va; out[1] = (double)ia;
    out[2] = ib < 0 ? INFINITY : vb; out[3] = (double)ib;
  }
}

// remove events over the support: -x_I / d_I, finite and > 0; ties go to the
// lowest column index keys[k] (the reference scans the support in index order)
__global__ void __launch_bounds__(HT) hom_gamma_minus_kernel(int64_t m, const double* __restrict__ x,
                                                             const double* __restrict__ d,
                                                             const long long* __restrict__ keys, double* out) {
  __shared__ long long kpos[1];
  double v = INFINITY;
  long long i = -1;
  for (int64_t k = threadIdx.x; k < m; k += HT) {
    const double r = -x[k] / d[k];
    if (isfinite(r) && r > 0.0) vi_min(v, i, r, keys[k]);
  }
  block_vi<false>(v, i);                       // thread 0: (value, lowest key)
  __shared__ long long bk;
  if (threadIdx.x == 0) { kpos[0] = -1; bk = i; }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < m; k += HT)  // the support position of that key
    if (bk >= 0 && keys[k] == bk) kpos[0] = k;
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = bk < 0 ? INFINITY : v; out[1] = (double)kpos[0]; }
}

__global__ void __launch_bounds__(HT) hom_xstats_kernel(int64_t m, const double* __restrict__ x, double* out) {
  __shared__ double red[HT / 32];
  __shared__ double bc;
  double s = 0.0, mx = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += HT) { s += fabs(x[k]); mx = fmax(mx, fabs(x[k])); }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < HT / 32; ++k) mx = fmax(mx, red[k]);
    bc = 1e-10 * (mx > 1.0 ? mx : 1.0);
  }
  __syncthreads();
  const double cut = bc;
  double cnt = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += HT) cnt += fabs(x[k]) > cut ? 1.0 : 0.0;
  __syncthreads();
  // fixed-order sums: warps in order
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < HT / 32; ++k) t += red[k];
    out[0] = t;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < HT / 32; ++k) t += red[k];
    out[1] = t;
  }
}

}  // namespace
}  // namespace ell1

using namespace ell1;

extern "C" int ell1_hom_absmax(int64_t n, const double* c, double* out2, void* stream) {
  if (n < 0 || (n && !c) || !out2) return ELL1_ERR_ARG;
  hom_absmax_kernel<<<1, HT, 0, (cudaStream_t)stream>>>(n, c, out2);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_hom_gammas(int64_t n, const double* c, const double* w, const unsigned char* mask, double lam,
                               double* out4, void* stream) {
  if (n < 0 || (n && (!c || !w || !mask)) || !out4) return ELL1_ERR_ARG;
  hom_gammas_kernel<<<1, HT, 0, (cudaStream_t)stream>>>(n, c, w, mask, lam, out4);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_hom_gamma_minus(int64_t m, const double* x, const double* d, const int64_t* keys,
                                    double* out2, void* stream) {
  if (m < 0 || (m && (!x || !d || !keys)) || !out2) return ELL1_ERR_ARG;
  hom_gamma_minus_kernel<<<1, HT, 0, (cudaStream_t)stream>>>(m, x, d, (const long long*)keys, out2);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_hom_xstats(int64_t m, const double* x, double* out2, void* stream) {
  if (m < 0 || (m && !x) || !out2) return ELL1_ERR_ARG;
  hom_xstats_kernel<<<1, HT, 0, (cudaStream_t)stream>>>(m, x, out2);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
