// batched.cuh — shared-dictionary batched solvers (BASELINE configs 3 and 5).
//
// B instances share one dictionary D (d x N, N = n or n + d for [A, sI]).  The
// instance vectors are stored column-major as matrices (N x B for x-like,
// ld x B for r-like), so every dictionary product of an iteration is one
// GEMM over all active instances (cuBLAS D/SGEMM on the B200), and the solver
// arithmetic in between runs in per-instance epilogue kernels (one CTA per
// instance, fixed-order block reductions) that reproduce the single-instance
// control flow of the reference (backtracking, continuation, stopping rules)
// with per-instance masks.  A C++ host loop in the library sequences the
// launches, reads one device counter per backtracking round, and compacts the
// active instances to the front of every matrix as they converge.
#pragma once
#include <cublas_v2.h>
#include "solvers_common.cuh"

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
struct Blas {
  cublasHandle_t h = nullptr;
  int dev = -1;
};

inline cublasHandle_t blas_handle(cudaStream_t s) {
  static thread_local Blas B[16];
  int dev = 0;
  cudaGetDevice(&dev);
  Blas& b = B[dev & 15];
  if (!b.h) {
    if (cublasCreate(&b.h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    b.dev = dev;
  }
  cublasSetStream(b.h, s);
  return b.h;
}

// Y(ld x B) = A(ld x n, column-major) X(n x B, ldx)      (A columns only)
inline bool gemm_AX(cublasHandle_t h, const ell1_dict_t* D, const void* X, int64_t ldx, void* Y,
                    int64_t ldy, int B) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64) {
    const double one = 1.0, zero = 0.0;
    return cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)D->ld, B, (int)D->n, &one,
                       (const double*)D->A, (int)D->ld, (const double*)X, (int)ldx, &zero, (double*)Y,
                       (int)ldy) == CUBLAS_STATUS_SUCCESS;
  }
  const float one = 1.0f, zero = 0.0f;
  return cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)D->ld, B, (int)D->n, &one, (const float*)D->A,
                     (int)D->ld, (const float*)X, (int)ldx, &zero, (float*)Y, (int)ldy) ==
         CUBLAS_STATUS_SUCCESS;
}

// G(n x B) = A^T R(ld x B)
inline bool gemm_AtR(cublasHandle_t h, const ell1_dict_t* D, const void* R, int64_t ldr, void* G,
                     int64_t ldg, int B) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64) {
    const double one = 1.0, zero = 0.0;
    return cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)D->n, B, (int)D->ld, &one,
                       (const double*)D->A, (int)D->ld, (const double*)R, (int)ldr, &zero, (double*)G,
                       (int)ldg) == CUBLAS_STATUS_SUCCESS;
  }
  const float one = 1.0f, zero = 0.0f;
  return cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)D->n, B, (int)D->ld, &one, (const float*)D->A,
                     (int)D->ld, (const float*)R, (int)ldr, &zero, (float*)G, (int)ldg) ==
         CUBLAS_STATUS_SUCCESS;
}

}  // namespace ell1
