// dmma_gemm.cuh — fp64 GEMM on the B200's double-precision tensor path (DMMA).
//
// The batched solvers' float64 dictionary products (config 5 in float64; the
// DALM Gram-inverse products; batched Homotopy's correlations; PDIPA's
// weighted Gram) are C = op(A) op(B) with column-major operands, beta = 0.
// tcgen05 has no fp64 kind, so the fp64 tensor work is warp-level
// mma.sync.m16n8k4.f64 (SASS DMMA): the kernel (dmma_gemm.cu) stages
// 64 x 64 x 16 operand tiles through a 4-deep cp.async shared-memory ring
// (padded, bank-conflict-free fragment reads), 4 warps each own a 32 x 32
// accumulator block in registers, and small problems split K across a
// thread-block cluster whose partial tiles are summed in rank order through
// distributed shared memory (deterministic, no workspace).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ell1 {

// C (m x n, column-major, ldc) = alpha op(A) (m x k) * op(B) (k x n) + beta C.
//   transA = 0: A is m x k column-major (lda >= m); 1: A is k x m (lda >= k).
//   transB = 0: B is k x n column-major (ldb >= k); 1: B is n x k (ldb >= n).
// Returns false on a launch error or bad argument.
bool dgemm(int transA, int transB, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
           const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s, double alpha = 1.0,
           double beta = 0.0);
// the same with a fixed tile variant (0..4) / K split (-1: heuristic), for tuning
bool dgemm_variant(int variant, int split, int transA, int transB, int64_t m, int64_t n, int64_t k,
                   const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   cudaStream_t s, double alpha = 1.0, double beta = 0.0);

}  // namespace ell1
