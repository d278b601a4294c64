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
#include <cstdlib>
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

// fp32 GEMM path of the batched solvers: 2 = 3xTF32 split on the tensor pipe,
// 0 = SIMT SGEMM (ELL1_FP32_GEMM=simt), -1 = not used yet.
inline int& fp32_gemm_mode() {
  static int mode = -1;
  return mode;
}

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

// ---------------------------------------------------------------- 3xTF32 fp32 GEMMs
// fp32 products of the batched solvers run on the tensor pipe as three TF32
// GEMMs with split operands (a = a_hi + a_lo, both TF32-representable):
//   A X ~= A_lo X_hi + A_hi X_lo + A_hi X_hi     (fp32 accumulation)
// which keeps fp32-level accuracy (the dropped A_lo X_lo term is ~2^-22
// relative) at TF32 tensor-core throughput.  The dictionary split is made
// once per solve; the right operand is split per product into caller
// workspace.  Opt-in (ELL1_FP32_GEMM=tf32x3): measured on B200 at config 3
// the three launches per product (skinny n x B GEMMs, B <= 1024) cost more
// than one SIMT SGEMM and the DALM certificate refines more often, so SIMT
// SGEMM stays the default.
struct F32Split {
  const float* Ahi;         // split dictionary, same layout as D->A
  const float* Alo;
  float* Xhi;               // right-operand scratch (xcap floats each)
  float* Xlo;
  int64_t xcap;
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

inline bool split_tf32(const float* src, float* hi, float* lo, int64_t n, cudaStream_t s) {
  if (n <= 0) return true;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  split_tf32_kernel<<<(unsigned)g, 256, 0, s>>>(src, hi, lo, n);
  return cudaGetLastError() == cudaSuccess;
}

inline bool use_tf32x3() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("ELL1_FP32_GEMM");
    v = (env && (env[0] == 't' || env[0] == 'T')) ? 1 : 0;   // opt-in: ELL1_FP32_GEMM=tf32x3
    fp32_gemm_mode() = v ? 2 : 0;
  }
  return v == 1;
}

// Y (m x B) = op(A) X with fp32 operands through the 3xTF32 split (sp) or SIMT SGEMM
inline bool sgemm_split(cublasHandle_t h, cublasOperation_t opA, int m, int B, int k, const float* A,
                        int lda, const F32Split* sp, const float* X, int64_t ldx, float* Y, int64_t ldy,
                        int64_t xrows) {
  const float one = 1.0f, zero = 0.0f;
  if (!sp || !use_tf32x3()) {
    return cublasSgemm(h, opA, CUBLAS_OP_N, m, B, k, &one, A, lda, X, (int)ldx, &zero, Y, (int)ldy) ==
           CUBLAS_STATUS_SUCCESS;
  }
  const int64_t xn = ldx * (int64_t)(B - 1) + xrows;
  if (xn > sp->xcap) return false;
  cudaStream_t s;
  cublasGetStream(h, &s);
  if (!split_tf32(X, sp->Xhi, sp->Xlo, xn, s)) return false;
  const cublasComputeType_t ct = CUBLAS_COMPUTE_32F_FAST_TF32;
  const void* terms[3][2] = {{sp->Alo, sp->Xhi}, {sp->Ahi, sp->Xlo}, {sp->Ahi, sp->Xhi}};
  for (int t = 0; t < 3; ++t) {
    const float* beta = t == 0 ? &zero : &one;
    if (cublasGemmEx(h, opA, CUBLAS_OP_N, m, B, k, &one, terms[t][0], CUDA_R_32F, lda, terms[t][1], CUDA_R_32F,
                     (int)ldx, beta, Y, CUDA_R_32F, (int)ldy, ct, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return false;
  }
  return true;
}

// Y(ld x B) = A(ld x n, column-major) X(n x B, ldx)      (A columns only)
inline bool gemm_AX(cublasHandle_t h, const ell1_dict_t* D, const void* X, int64_t ldx, void* Y,
                    int64_t ldy, int B, const F32Split* sp = nullptr) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64) {
    const double one = 1.0, zero = 0.0;
    return cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)D->ld, B, (int)D->n, &one,
                       (const double*)D->A, (int)D->ld, (const double*)X, (int)ldx, &zero, (double*)Y,
                       (int)ldy) == CUBLAS_STATUS_SUCCESS;
  }
  return sgemm_split(h, CUBLAS_OP_N, (int)D->ld, B, (int)D->n, (const float*)D->A, (int)D->ld, sp,
                     (const float*)X, ldx, (float*)Y, ldy, D->n);
}

// G(n x B) = A^T R(ld x B)
inline bool gemm_AtR(cublasHandle_t h, const ell1_dict_t* D, const void* R, int64_t ldr, void* G,
                     int64_t ldg, int B, const F32Split* sp = nullptr) {
  if (B <= 0) return true;
  if (D->dtype == ELL1_F64) {
    const double one = 1.0, zero = 0.0;
    return cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)D->n, B, (int)D->ld, &one,
                       (const double*)D->A, (int)D->ld, (const double*)R, (int)ldr, &zero, (double*)G,
                       (int)ldg) == CUBLAS_STATUS_SUCCESS;
  }
  return sgemm_split(h, CUBLAS_OP_T, (int)D->n, B, (int)D->ld, (const float*)D->A, (int)D->ld, sp,
                     (const float*)R, ldr, (float*)G, ldg, D->ld);
}

// workspace floats for the dictionary split + the right-operand scratch
inline int64_t f32split_floats(const ell1_dict_t* D, int64_t xcap) {
  return 2 * align_up(D->n * D->ld, 64) + 2 * align_up(xcap, 64);
}

inline bool f32split_setup(F32Split& sp, Carve& cv, const ell1_dict_t* D, int64_t xcap, cudaStream_t s) {
  float* hi = cv.take<float>(D->n * D->ld);
  float* lo = cv.take<float>(D->n * D->ld);
  sp.Xhi = cv.take<float>(xcap);
  sp.Xlo = cv.take<float>(xcap);
  sp.xcap = xcap;
  sp.Ahi = hi; sp.Alo = lo;
  if (!cv.ok) return false;
  return split_tf32((const float*)D->A, hi, lo, D->n * D->ld, s);
}

}  // namespace ell1
