// gemm_abi.cu — C-ABI entry for the batched solvers' fp32 product (tc_gemm.cu),
// used by the GPU tests and for direct calls (include/ell1_b200.h).
#include "ell1_b200.h"
#include "batched.cuh"

using namespace ell1;

// K-major split of A^T for column-major A (K x M, lda): row i = column i of A
static __global__ void split_rows_kernel(const float* __restrict__ A, int64_t lda, int64_t M, int64_t K,
                                         int64_t pitch, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t i = blockIdx.y;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < pitch; k += (int64_t)gridDim.x * blockDim.x) {
    const float x = k < K ? A[i * lda + k] : 0.f;
    const float h = tf32_rna(x);
    hi[i * pitch + k] = h;
    lo[i * pitch + k] = tf32_rna(x - h);
  }
}

extern "C" size_t ell1_gemm_f32_workspace(int32_t trans, int64_t M, int64_t K) {
  if (M < 0 || K < 0) return 0;
  const int64_t pitch = align_up(K, 4);
  (void)trans;
  return (size_t)(2 * align_up(M * pitch, 64)) * 4 + 1024;
}

extern "C" int ell1_gemm_f32(int32_t trans, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                             const float* B, int64_t ldb, float* C, int64_t ldc, void* ws, size_t wsb,
                             void* stream) {
  if (M < 0 || N < 0 || K < 0 || (M && N && (!A || !B || !C)) || ldc < M || (ldb & 3) || ldb < K)
    return ELL1_ERR_ARG;
  if (trans ? lda < K : lda < M) return ELL1_ERR_ARG;
  if (M == 0 || N == 0) return ELL1_OK;
  if (wsb < ell1_gemm_f32_workspace(trans, M, K) || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t pitch = align_up(K, 4);
  Carve cv(ws, wsb);
  float* hi = cv.take<float>(M * pitch);
  float* lo = cv.take<float>(M * pitch);
  if (!cv.ok) return ELL1_ERR_ARG;
  // K-major split of op(A): row i of op(A) at hi + i * pitch
  if (trans) {
    dim3 g((unsigned)((pitch + 255) / 256), (unsigned)M);
    split_rows_kernel<<<g, 256, 0, s>>>(A, lda, M, K, pitch, hi, lo);
  } else {
    dim3 g((unsigned)((pitch + 31) / 32), (unsigned)((M + 31) / 32));
    split_tf32_t_kernel<<<g, dim3(32, 8), 0, s>>>(A, hi, lo, M, lda, K, pitch);
  }
  if (cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
  return tc3_gemm((int)M, (int)N, (int)K, hi, lo, pitch, B, ldb, C, ldc, s) ? ELL1_OK : ELL1_ERR_CUDA;
}
