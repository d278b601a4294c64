// chol.cu — dense Cholesky factor + solve of PDIPA's weighted normal matrix
// M = A diag(w) A^T (pdipa.py:43-62: _factor_with_jitter, then
// factor.solve(rhs) inside _eliminate), replacing numpy/LAPACK's potrf/potrs.
//
// Blocked right-looking factorisation, NB = 64 columns per panel:
//   chol_panel_kernel   one CTA factors the NB x NB diagonal block in shared
//                       memory (pivot <= 0 or not finite -> status = k + 1,
//                       LAPACK's convention; the host then retries with the
//                       reference's jitter)
//   chol_trsm_kernel    L21 = A21 L11^-T, one thread per row below the panel
//   dgemm (DMMA)        trailing update A22 -= L21 L21^T (dmma_gemm.cu)
// Solve: L y = rhs, L^T x = y, 32-column blocks in one CTA (the small
// triangles by one warp, the rank-32 updates by the whole CTA).
#include "dmma_gemm.cuh"
#include "ell1_b200.h"
#include "engine.cuh"

namespace ell1 {
namespace {

constexpr int NB = 64;
constexpr int PT = 256;

// a / d with the reciprocal of d already at hand (rinv = 1.0 / d, correctly
// rounded): one multiply and two fused corrections give the correctly rounded
// quotient (Markstein's sequence) in ~30 cycles of dependent latency instead of
// the ~300 of a full double-precision division — the triangular solves are
// chains of such divisions
__device__ __forceinline__ double div_by(double a, double d, double rinv) {
  const double q = a * rinv;
  const double r = fma(-q, d, a);
  return fma(r, rinv, q);
}

__global__ void chol_copy_kernel(int64_t d, const double* __restrict__ M, int64_t ldm, double* __restrict__ L,
                                 int64_t ldl, double jitter, int* status) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *status = 0;
  const int64_t tot = d * d;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / d, i = t - j * d;
    double v = M[j * ldm + i];
    if (i == j) v += jitter;
    L[j * ldl + i] = v;
  }
}

// factor the nb x nb diagonal block at (kb, kb) in place (lower triangle)
__global__ void __launch_bounds__(PT) chol_panel_kernel(double* __restrict__ L, int64_t ld, int64_t kb, int nb,
                                                        int* status) {
  __shared__ double T[NB][NB + 1];
  if (*(volatile int*)status != 0) return;
  for (int t = threadIdx.x; t < nb * nb; t += PT) {
    const int c = t / nb, r = t - c * nb;
    T[r][c] = L[(kb + c) * ld + kb + r];
  }
  __syncthreads();
  // two barriers per column: every thread reads the pivot itself (no thread-0
  // section), and the trailing update maps thread -> (row, column group) with no
  // index divisions; T[r][c] with r across lanes is conflict-free (pitch NB + 1)
  static_assert(PT == 4 * NB, "row x column-group mapping");
  const int r = threadIdx.x & (NB - 1), c0 = threadIdx.x >> 6;
  for (int j = 0; j < nb; ++j) {
    const double dj = T[j][j];
    if (!(dj > 0.0) || !isfinite(dj)) {                       // uniform: every thread sees the same pivot
      if (threadIdx.x == 0) *status = (int)(kb + j) + 1;
      return;
    }
    const double piv = sqrt(dj);
    for (int i = j + 1 + threadIdx.x; i < nb; i += PT) T[i][j] /= piv;
    __syncthreads();
    if (threadIdx.x == 0) T[j][j] = piv;
    if (r > j && r < nb) {
      const double lr = T[r][j];
      for (int c = j + 1 + c0; c <= r; c += 4) T[r][c] -= lr * T[c][j];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nb * nb; t += PT) {
    const int c = t / nb, r2 = t - c * nb;
    if (r2 >= c) L[(kb + c) * ld + kb + r2] = T[r2][c];
  }
}

// rows i in [r0, d): L[i, kb:kb+nb] <- L[i, kb:kb+nb] L11^-T
__global__ void __launch_bounds__(PT) chol_trsm_kernel(double* __restrict__ L, int64_t ld, int64_t d, int64_t kb,
                                                       int nb, const int* status) {
  __shared__ double T[NB][NB + 1];
  __shared__ double Tinv[NB];
  if (*(volatile int*)status != 0) return;
  for (int t = threadIdx.x; t < nb * nb; t += PT) {
    const int c = t / nb, r = t - c * nb;
    T[r][c] = L[(kb + c) * ld + kb + r];
  }
  if (threadIdx.x < nb) Tinv[threadIdx.x] = 1.0 / L[(kb + threadIdx.x) * ld + kb + threadIdx.x];
  __syncthreads();
  const int64_t i = kb + nb + (int64_t)blockIdx.x * PT + threadIdx.x;
  if (i >= d) return;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) x[c] = c < nb ? L[(kb + c) * ld + i] : 0.0;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    if (c < nb) {
      double v = x[c];
#pragma unroll
      for (int p = 0; p < c; ++p) v -= x[p] * T[c][p];
      x[c] = div_by(v, T[c][c], Tinv[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c < nb) L[(kb + c) * ld + i] = x[c];
}

// x = (L L^T)^-1 rhs, one CTA per right-hand side (column blockIdx.x of
// rhs / x, strides ldr / ldx); y staged in shared memory (d doubles)
__global__ void __launch_bounds__(1024) chol_solve_kernel(int64_t d, const double* __restrict__ L, int64_t ld,
                                                          const double* __restrict__ rhs_all, int64_t ldr,
                                                          double* __restrict__ x_all, int64_t ldx) {
  extern __shared__ double y[];
  // the 32 x 32 diagonal block of a step, staged one step ahead (double-buffered)
  // so the warp's 32 dependent steps read shared memory, not global memory
  __shared__ double Dg[2][32][33];
  const double* __restrict__ rhs = rhs_all + (int64_t)blockIdx.x * ldr;
  double* __restrict__ x = x_all + (int64_t)blockIdx.x * ldx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  auto stage = [&](int buf, int64_t jb, int w, int t0, int nt) {   // Dg[buf][r][c] = L[jb + r, jb + c], r >= c
    for (int t = t0; t < 32 * 32; t += nt) {
      const int c = t >> 5, r = t & 31;
      if (r < w && c < w && r >= c) Dg[buf][r][c] = L[(jb + c) * ld + jb + r];
    }
  };
  for (int64_t i = tid; i < d; i += blockDim.x) y[i] = rhs[i];
  stage(0, 0, (int)(d < 32 ? d : 32), tid, blockDim.x);
  __syncthreads();
  // Forward L y = rhs in 32-column blocks with one step of lookahead: in step k
  // warp 0 applies block k-1 to the 32 rows of block k and solves their triangle
  // while the other warps apply block k-1 to the rows below and stage the next
  // diagonal block — one barrier per block, the triangle off the update's
  // critical path.  Every y_i still receives the blocks in ascending order.
  int buf = 0;
  for (int64_t jb = 0; jb < d; jb += 32, buf ^= 1) {
    const int w = (int)((d - jb) < 32 ? (d - jb) : 32);
    const int64_t jp = jb - 32;
    if (warp == 0) {
      if (jb > 0 && lane < w) {
        double s = y[jb + lane];
        for (int j = 0; j < 32; ++j) s -= L[(jp + j) * ld + jb + lane] * y[jp + j];
        y[jb + lane] = s;
      }
      __syncwarp();
      double v = lane < w ? y[jb + lane] : 0.0;
      const double dl = lane < w ? Dg[buf][lane][lane] : 1.0, rl = 1.0 / dl;
      for (int j = 0; j < w; ++j) {
        const double xj = div_by(__shfl_sync(0xffffffffu, v, j), __shfl_sync(0xffffffffu, dl, j),
                                 __shfl_sync(0xffffffffu, rl, j));
        if (lane == j) v = xj;
        if (lane > j && lane < w) v -= Dg[buf][lane][j] * xj;
      }
      if (lane < w) y[jb + lane] = v;
    } else {
      if (jb > 0)
        for (int64_t i = jb + 32 + (tid - 32); i < d; i += blockDim.x - 32) {
          double s = y[i];
          for (int j = 0; j < 32; ++j) s -= L[(jp + j) * ld + i] * y[jp + j];
          y[i] = s;
        }
      if (jb + 32 < d) stage(buf ^ 1, jb + 32, (int)((d - jb - 32) < 32 ? (d - jb - 32) : 32), tid - 32, blockDim.x - 32);
    }
    __syncthreads();
  }
  // Backward L^T x = y, blocks from the end, the same lookahead:
  // x_i = (y_i - sum_{j>i} L_ji x_j) / L_ii
  {
    const int64_t jb = d >= 32 ? d - 32 : 0;
    buf = 0;
    stage(0, jb, (int)(d - jb), tid, blockDim.x);
    __syncthreads();
  }
  for (int64_t je = d; je > 0; je -= 32, buf ^= 1) {
    const int64_t jb = je >= 32 ? je - 32 : 0;
    const int w = (int)(je - jb);
    const int64_t pb = je;                                    // previous (higher) block [pb, pb + pw)
    const int pw = (int)((d - pb) < 32 ? (d - pb) : 32);
    if (warp == 0) {
      if (je < d) {
        // y_i -= sum_{j in previous block} L_ji x_j for the rows of this block
        for (int r = 0; r < w; ++r) {
          const int64_t i = jb + r;
          double s = lane < pw ? L[i * ld + pb + lane] * y[pb + lane] : 0.0;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) y[i] -= s;
        }
        __syncwarp();
      }
      double v = lane < w ? y[jb + lane] : 0.0;
      const double dl = lane < w ? Dg[buf][lane][lane] : 1.0, rl = 1.0 / dl;
      for (int j = w - 1; j >= 0; --j) {
        const double xj = div_by(__shfl_sync(0xffffffffu, v, j), __shfl_sync(0xffffffffu, dl, j),
                                 __shfl_sync(0xffffffffu, rl, j));
        if (lane == j) v = xj;
        if (lane < j) v -= Dg[buf][j][lane] * xj;
      }
      if (lane < w) y[jb + lane] = v;
    } else {
      if (je < d)
        for (int64_t i = warp - 1; i < jb; i += nw - 1) {     // one warp per row i (coalesced in j)
          double s = lane < pw ? L[i * ld + pb + lane] * y[pb + lane] : 0.0;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) y[i] -= s;
        }
      if (jb > 0) {
        const int64_t jb2 = jb >= 32 ? jb - 32 : 0;
        stage(buf ^ 1, jb2, (int)(jb - jb2), tid - 32, blockDim.x - 32);
      }
    }
    __syncthreads();
  }
  for (int64_t i = tid; i < d; i += blockDim.x) x[i] = y[i];
}

}  // namespace
}  // namespace ell1

using namespace ell1;

extern "C" int ell1_chol_factor_dense(int64_t d, const double* M, int64_t ldm, double jitter, double* L, int64_t ldl,
                                      int* status, void* stream) {
  if (d < 1 || !M || !L || !status || ldm < d || ldl < d) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tot = d * d;
  const unsigned g = (unsigned)((tot + 255) / 256 < 148 * 8 ? (tot + 255) / 256 : 148 * 8);
  chol_copy_kernel<<<g, 256, 0, s>>>(d, M, ldm, L, ldl, jitter, status);
  for (int64_t kb = 0; kb < d; kb += NB) {
    const int nb = (int)((d - kb) < NB ? (d - kb) : NB);
    chol_panel_kernel<<<1, PT, 0, s>>>(L, ldl, kb, nb, status);
    const int64_t below = d - kb - nb;
    if (below <= 0) break;
    chol_trsm_kernel<<<(unsigned)((below + PT - 1) / PT), PT, 0, s>>>(L, ldl, d, kb, nb, status);
    // trailing update A22 -= L21 L21^T (full square; the lower triangle is used)
    double* L21 = L + kb * ldl + kb + nb;
    double* A22 = L + (kb + nb) * ldl + kb + nb;
    if (!dgemm(0, 1, below, below, nb, L21, ldl, L21, ldl, A22, ldl, s, -1.0, 1.0)) return ELL1_ERR_CUDA;
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_chol_solve_dense(int64_t d, const double* L, int64_t ldl, const double* rhs, double* x,
                                     void* stream) {
  return ell1_chol_solve_dense_multi(d, L, ldl, 1, rhs, d, x, d, stream);
}

extern "C" int ell1_chol_solve_dense_multi(int64_t d, const double* L, int64_t ldl, int64_t nrhs, const double* rhs,
                                           int64_t ldr, double* x, int64_t ldx, void* stream) {
  if (d < 1 || nrhs < 0 || !L || !rhs || !x || ldl < d || ldr < d || ldx < d || nrhs > 0x7fffffff)
    return ELL1_ERR_ARG;
  if (nrhs == 0) return ELL1_OK;
  const size_t smem = (size_t)d * 8;
  if (smem > 200 * 1024) return ELL1_ERR_ARG;
  if (cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return ELL1_ERR_CUDA;
  const int threads = d >= 1024 ? 1024 : (d >= 256 ? 256 : 128);
  chol_solve_kernel<<<(unsigned)nrhs, threads, smem, (cudaStream_t)stream>>>(d, L, ldl, rhs, ldr, x, ldx);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
