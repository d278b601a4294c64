// tc_gemm.cuh — fp32-accurate GEMM on the 5th-generation tensor cores (3xTF32).
//
// The batched solvers' fp32 dictionary products (configs 3 and 5 in float32
// storage) are C = A B with A (M x K) a static dictionary (or its Gram-
// preconditioned copy) and B (K x N) the instance block.  Each operand is
// held as a TF32 split x = hi + lo (hi = rna_tf32(x), lo = rna_tf32(x - hi));
// one kernel accumulates hi*hi + hi*lo + lo*hi into the same TMEM
// accumulator, so the product keeps fp32-level accuracy (the dropped lo*lo
// term is ~2^-22 relative) at TF32 tensor-pipe throughput.  The tensor pipe
// accumulates one 32-wide k-block per partial; partials are summed in IEEE
// fp32 registers (the tensor core's own long accumulation loses ~10x more).
//
// Kernel anatomy (tc_gemm.cu): one 128 x BN output tile per CTA; TMA
// (cp.async.bulk.tensor, 128B swizzle) stages the four K-major operand tiles
// of a 32-wide k-block into a ST-deep shared-memory ring guarded by mbarriers;
// four split/drain warps split the B tile in shared memory; one elected
// thread issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) into one of two
// TMEM partial buffers and releases ring slots with tcgen05.commit; the drain
// warps add each partial (tcgen05.ld) into fp32 registers and finally write C
// column-major with coalesced stores.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ell1 {

// C (M x N, column-major, ldc) = A B where
//   A is given K-major: row i of A at a_hi/a_lo + i * lda (K contiguous),
//   B is given K-major and unsplit: column j of B at b + j * ldb (K contiguous;
//   the kernel splits each staged tile itself).
// lda, ldb multiples of 4 floats, pointers 16-byte aligned.  Returns false if
// the tensor-core path cannot take the call (the caller then uses SIMT SGEMM).
// b_lo (optional): B already split by its producer — b holds rna_tf32(B) and
// b_lo rna_tf32(B - b); both arrive by TMA and the in-kernel split is skipped.
bool tc3_gemm(int M, int N, int K, const float* a_hi, const float* a_lo, int64_t lda, const float* b, int64_t ldb,
              float* C, int64_t ldc, cudaStream_t s, const float* b_lo = nullptr);

// 0 = not tried yet, 1 = available, -1 = unavailable (no driver entry point)
int tc3_available();

}  // namespace ell1
