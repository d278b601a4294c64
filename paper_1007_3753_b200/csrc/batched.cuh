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
struct Blas {
  cublasHandle_t h = nullptr;
  int dev = -1;
};

// fp32 GEMM path of the batched solvers: 3 = 3xTF32 tcgen05 kernel (tc_gemm.cu,
// default), 2 = 3xTF32 split over three cuBLAS TF32 GEMMs (ELL1_FP32_GEMM=tf32x3),
// 0 = SIMT SGEMM (ELL1_FP32_GEMM=simt), -1 = not used yet.
inline int& fp32_gemm_mode() {
  static int mode = -1;
  return mode;
}

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
// fp32 products of the batched solvers run on the tensor pipe as 3xTF32: both
// operands are split a = a_hi + a_lo (both TF32-representable) and
//   A X ~= A_lo X_hi + A_hi X_lo + A_hi X_hi     (fp32 accumulation)
// keeps fp32-level accuracy (the dropped A_lo X_lo term is ~2^-22 relative).
// Default: one tcgen05 kernel accumulates the three products in TMEM
// (tc_gemm.cu).  The dictionary split is made once per solve, in both
// orientations (column-major for A^T R, row-major for A X: the kernel reads
// K-major operands); the right operand is split per product into caller
// workspace.  ELL1_FP32_GEMM=tf32x3 runs the split as three cuBLAS TF32 GEMMs,
// ELL1_FP32_GEMM=simt uses cuBLAS SIMT SGEMM.
struct F32Split {
  const float* Ahi;         // split dictionary, same layout as D->A (column-major, ld)
  const float* Alo;
  const float* Arhi;        // split dictionary, row-major (ld rows of pr floats)
  const float* Arlo;
  int64_t pr;
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

inline int fp32_mode_select() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("ELL1_FP32_GEMM");
    if (env && (env[0] == 's' || env[0] == 'S')) v = 0;
    else if (env && (env[0] == 't' || env[0] == 'T')) v = 2;
    else v = tc3_available() == 1 ? 3 : 0;
    fp32_gemm_mode() = v;
  }
  return v;
}

// Y (m x B) = op(A) X with fp32 operands through the 3xTF32 split (sp) or SIMT SGEMM
inline bool sgemm_split(cublasHandle_t h, cublasOperation_t opA, int m, int B, int k, const float* A,
                        int lda, const F32Split* sp, const float* X, int64_t ldx, float* Y, int64_t ldy,
                        int64_t xrows) {
  const float one = 1.0f, zero = 0.0f;
  const int mode = fp32_mode_select();
  if (!sp || mode == 0) {
    return cublasSgemm(h, opA, CUBLAS_OP_N, m, B, k, &one, A, lda, X, (int)ldx, &zero, Y, (int)ldy) ==
           CUBLAS_STATUS_SUCCESS;
  }
  cudaStream_t s;
  cublasGetStream(h, &s);
  if (mode == 3) {
    // the kernel splits the right operand tile by tile in shared memory
    const bool ok = opA == CUBLAS_OP_N ? tc3_gemm(m, B, k, sp->Arhi, sp->Arlo, sp->pr, X, ldx, Y, ldy, s)
                                       : tc3_gemm(m, B, k, sp->Ahi, sp->Alo, lda, X, ldx, Y, ldy, s);
    if (ok) return true;
    if (!A) return false;
    return cublasSgemm(h, opA, CUBLAS_OP_N, m, B, k, &one, A, lda, X, (int)ldx, &zero, Y, (int)ldy) ==
           CUBLAS_STATUS_SUCCESS;
  }
  const int64_t xn = ldx * (int64_t)(B - 1) + xrows;
  if (xn > sp->xcap) return false;
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

// workspace floats for one dictionary split (both orientations)
inline int64_t f32split_dict_floats(const ell1_dict_t* D) {
  return 2 * align_up(D->n * D->ld, 64) + 2 * align_up(D->ld * align_up(D->n, 4), 64);
}

// workspace floats for the dictionary split + the right-operand scratch
inline int64_t f32split_floats(const ell1_dict_t* D, int64_t xcap) {
  return f32split_dict_floats(D) + 2 * align_up(xcap, 64);
}

// split a column-major (ld x n) fp32 dictionary A into sp's four arrays
inline bool f32split_dict(F32Split& sp, Carve& cv, const ell1_dict_t* D, const float* A, cudaStream_t s) {
  float* hi = cv.take<float>(D->n * D->ld);
  float* lo = cv.take<float>(D->n * D->ld);
  const int64_t pr = align_up(D->n, 4);
  float* rhi = cv.take<float>(D->ld * pr);
  float* rlo = cv.take<float>(D->ld * pr);
  if (!cv.ok) return false;
  sp.Ahi = hi; sp.Alo = lo; sp.Arhi = rhi; sp.Arlo = rlo; sp.pr = pr;
  if (!split_tf32(A, hi, lo, D->n * D->ld, s)) return false;
  dim3 g((unsigned)((pr + 31) / 32), (unsigned)((D->ld + 31) / 32));
  split_tf32_t_kernel<<<g, dim3(32, 8), 0, s>>>(A, rhi, rlo, D->ld, D->ld, D->n, pr);
  return cudaGetLastError() == cudaSuccess;
}

inline bool f32split_setup(F32Split& sp, Carve& cv, const ell1_dict_t* D, int64_t xcap, cudaStream_t s) {
  if (!f32split_dict(sp, cv, D, (const float*)D->A, s)) return false;
  sp.Xhi = cv.take<float>(xcap);
  sp.Xlo = cv.take<float>(xcap);
  sp.xcap = xcap;
  return cv.ok;
}

}  // namespace ell1
