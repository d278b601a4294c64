// batched.cuh — shared-dictionary batched solvers (BASELINE configs 3 and 5).
//
// B instances share one dictionary D (d x N, N = n or n + d for [A, sI]).  The
// instance vectors are stored column-major as matrices (N x B for x-like,
// ld x B for r-like), so every dictionary product of an iteration is one
// GEMM over all active instances (the library's own tensor-core GEMMs: DMMA
// for float64 storage, dmma_gemm.cu; tcgen05 3xTF32 for float32, tc_gemm.cu), and the solver
// arithmetic in between runs in per-instance epilogue kernels (one CTA per
// instance, fixed-order block reductions) that reproduce the single-instance
// control flow of the reference (backtracking, continuation, stopping rules)
// with per-instance masks.  A C++ host loop in the library sequences the
// launches, reads one device counter per backtracking round, and compacts the
// active instances to the front of every matrix as they converge.
#pragma once
#include <cstdlib>
#include "dmma_gemm.cuh"
#include "solvers_common.cuh"
#include "tc_gemm.cuh"

namespace ell1 {

constexpr int BT = 256;                 // threads per instance CTA
constexpr int BW = BT / 32;

// fixed-order CTA reduction of K values (sum / max by mask), all threads get them
template <int K>
__device__ __forceinline__ void cta_reduce(double (&v)[K], unsigned maxmask, double* sh) {
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = ((maxmask >> k) & 1u) ? warp_max(v[k]) : warp_sum(v[k]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[w * K + k] = v[k];
  }
  __syncthreads();
  if ((int)threadIdx.x < K) {
    const int k = threadIdx.x;
    const bool mx = (maxmask >> k) & 1u;
    double s = sh[k];
    for (int ww = 1; ww < BW; ++ww) s = mx ? nmax(s, sh[ww * K + k]) : s + sh[ww * K + k];
    sh[BW * K + k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sh[BW * K + k];
  __syncthreads();
}

// --------------------------------------------------------------- host helpers
// Pinned host mailbox (per thread, 16 ints) for the per-round device counter
// read-backs of the batched host loops: a pageable 8-byte D2H is a staged
// copy (~7 us on the B200 box), a pinned one is a direct DMA.
inline int* host_mailbox() {
  static thread_local int* box = nullptr;
  static thread_local int fallback[16];
  if (!box) {
    void* p = nullptr;
    if (cudaMallocHost(&p, 64) == cudaSuccess) box = (int*)p;
    else box = fallback;
  }
  return box;
}

// ---------------------------------------------------------------- 3xTF32 fp32 GEMMs
// fp32 products of the batched solvers run on the tensor pipe as 3xTF32: both
// operands are split a = a_hi + a_lo (both TF32-representable) and
//   A X ~= A_lo X_hi + A_hi X_lo + A_hi X_hi     (fp32 accumulation)
// keeps fp32-level accuracy (the dropped A_lo X_lo term is ~2^-22 relative).
// One tcgen05 kernel accumulates the three products in TMEM (tc_gemm.cu).
// The dictionary split is made once per solve, in both orientations
// (column-major for A^T R, row-major for A X: the kernel reads K-major
// operands); the right operand is split tile by tile inside the kernel.
// There is no other fp32 path: a call the kernel cannot take is an error.
struct F32Split {
  const float* Ahi;         // split dictionary, same layout as D->A (column-major, ld)
  const float* Alo;
  const float* Arhi;        // split dictionary, row-major (ld rows of pr floats)
  const float* Arlo;
  int64_t pr;
  int64_t pc;               // column stride of Ahi / Alo (the dictionary's ld)
};

__device__ __forceinline__ float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

static __global__ void split_tf32_kernel(const float* __restrict__ src, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = src[i];
    const float h = tf32_rna(x);
    hi[i] = h;
    lo[i] = tf32_rna(x - h);
  }
}

// row-major split of a column-major (rows x n, stride ld) matrix: hi/lo[i * pr + k] from src[k * ld + i]
static __global__ void split_tf32_t_kernel(const float* __restrict__ src, float* __restrict__ hi,
                                           float* __restrict__ lo, int64_t rows, int64_t ld, int64_t n,
                                           int64_t pr) {
  __shared__ float t[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, i = i0 + threadIdx.x;
    t[r][threadIdx.x] = (k < n && i < rows) ? src[k * ld + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, k = k0 + threadIdx.x;
    if (i < rows && k < pr) {
      const float x = t[threadIdx.x][r];
      const float h = tf32_rna(x);
      hi[i * pr + k] = h;
      lo[i * pr + k] = tf32_rna(x - h);
    }
  }
}

inline bool split_tf32(const float* src, float* hi, float* lo, int64_t n, cudaStream_t s) {
  if (n <= 0) return true;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  split_tf32_kernel<<<(unsigned)g, 256, 0, s>>>(src, hi, lo, n);
  return cudaGetLastError() == cudaSuccess;
}

// Y (m x B) = op(A) X with fp32 operands through the 3xTF32 split of A (sp)
// Xlo (optional): X arrives split by its producer (X = rna_tf32 hi, Xlo = lo)
inline bool sgemm_split(cudaStream_t st, int transA, int m, int B, int k, const F32Split* sp, const float* X,
                        int64_t ldx, float* Y, int64_t ldy, const float* Xlo = nullptr) {
  if (!sp) return false;
  return transA ? tc3_gemm(m, B, k, sp->Ahi, sp->Alo, sp->pc, X, ldx, Y, ldy, st, Xlo)
                : tc3_gemm(m, B, k, sp->Arhi, sp->Arlo, sp->pr, X, ldx, Y, ldy, st, Xlo);
}

// Y(ld x B) = A(ld x n, column-major) X(n x B, ldx)      (A columns only)
inline bool gemm_AX(cudaStream_t st, const ell1_dict_t* D, const void* X, int64_t ldx, void* Y, int64_t ldy,
                    int B, const F32Split* sp = nullptr, const float* Xlo = nullptr) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64)
    return dgemm(0, 0, D->ld, B, D->n, (const double*)D->A, D->ld, (const double*)X, ldx, (double*)Y, ldy, st);
  return sgemm_split(st, 0, (int)D->ld, B, (int)D->n, sp, (const float*)X, ldx, (float*)Y, ldy, Xlo);
}

// G(n x B) = A^T R(ld x B)
inline bool gemm_AtR(cudaStream_t st, const ell1_dict_t* D, const void* R, int64_t ldr, void* G, int64_t ldg,
                     int B, const F32Split* sp = nullptr, const float* Rlo = nullptr) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64)
    return dgemm(1, 0, D->n, B, D->ld, (const double*)D->A, D->ld, (const double*)R, ldr, (double*)G, ldg, st);
  return sgemm_split(st, 1, (int)D->n, B, (int)D->ld, sp, (const float*)R, ldr, (float*)G, ldg, Rlo);
}

// workspace floats for one dictionary split (both orientations)
inline int64_t f32split_dict_floats(const ell1_dict_t* D) {
  return 2 * align_up(D->n * D->ld, 64) + 2 * align_up(D->ld * align_up(D->n, 4), 64);
}

// workspace floats of f32split_setup (the right operand is split inside the GEMM)
inline int64_t f32split_floats(const ell1_dict_t* D, int64_t xcap) {
  (void)xcap;
  return f32split_dict_floats(D);
}

// split a column-major (ld x n) fp32 dictionary A into sp's four arrays
inline bool f32split_dict(F32Split& sp, Carve& cv, const ell1_dict_t* D, const float* A, cudaStream_t s) {
  float* hi = cv.take<float>(D->n * D->ld);
  float* lo = cv.take<float>(D->n * D->ld);
  const int64_t pr = align_up(D->n, 4);
  float* rhi = cv.take<float>(D->ld * pr);
  float* rlo = cv.take<float>(D->ld * pr);
  if (!cv.ok) return false;
  sp.Ahi = hi; sp.Alo = lo; sp.Arhi = rhi; sp.Arlo = rlo; sp.pr = pr; sp.pc = D->ld;
  if (!split_tf32(A, hi, lo, D->n * D->ld, s)) return false;
  dim3 g((unsigned)((pr + 31) / 32), (unsigned)((D->ld + 31) / 32));
  split_tf32_t_kernel<<<g, dim3(32, 8), 0, s>>>(A, rhi, rlo, D->ld, D->ld, D->n, pr);
  return cudaGetLastError() == cudaSuccess;
}

inline bool f32split_setup(F32Split& sp, Carve& cv, const ell1_dict_t* D, int64_t xcap, cudaStream_t s) {
  (void)xcap;
  return f32split_dict(sp, cv, D, (const float*)D->A, s);
}

}  // namespace ell1
