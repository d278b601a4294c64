// tc_gemm.cu — 3xTF32 tcgen05 GEMM for the batched fp32 solvers (see tc_gemm.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "tc_gemm.cuh"

namespace ell1 {
namespace {

constexpr int TM = 128;          // tile rows (UMMA M)
constexpr int TK = 32;           // k-block: 32 fp32 = one 128-byte swizzle row
constexpr int UK = 8;            // UMMA K for kind::tf32

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// shared-memory matrix descriptor: K-major operand tile, 128-byte swizzle,
// 8-row core groups 1024 bytes apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = (uint64_t)(smem_u32(p) & 0x3FFFF) >> 4;
  return addr | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = BN
template <int BN>
__host__ __device__ constexpr uint32_t instr_desc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ float tf32_rna_dev(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <int BN, int ST>
struct Smem {
  static constexpr int A_BYTES = TM * TK * 4;         // 16 KB
  static constexpr int B_BYTES = BN * TK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int TX = 2 * A_BYTES + B_BYTES;    // bytes TMA brings per stage (B arrives unsplit)
  static constexpr int TOTAL = ST * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

// Warp roles (192 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA
// issuer, warps 2-5 = split + drain.  Per k-block the drain warps split the
// raw B tile in place (hi) and into the lo tile, and — one k-block behind the
// tensor core — add the block's TMEM partial product into fp32 registers:
// the tensor pipe's accumulation spans only 32 products, the running sum is
// IEEE fp32 (keeps the SIMT SGEMM's accuracy).  TMEM holds two BN-column
// partial buffers (MMA fills one while the other drains).
template <int BN, int ST>
__global__ void __launch_bounds__(192, 1)
    tc3_gemm_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mB, int M, int N, int K, float* __restrict__ C,
                    int64_t ldc) {
  using S = Smem<BN, ST>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + ST * S::STAGE);
  uint64_t* conv = full + ST;
  uint64_t* empty = conv + ST;
  uint64_t* tfull = empty + ST;       // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * BN;
  const int nkb = (K + TK - 1) / TK;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mAh) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mAl) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mB) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(conv + s, 128);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % ST, u = kb / ST;
        if (u > 0) mbar_wait(empty + s, (u - 1) & 1);
        uint8_t* st = smem + s * S::STAGE;
        mbar_expect_tx(full + s, S::TX);
        tma_load_2d(st, &mAh, kb * TK, m0, full + s);
        tma_load_2d(st + S::A_BYTES, &mAl, kb * TK, m0, full + s);
        tma_load_2d(st + 2 * S::A_BYTES, &mB, kb * TK, n0, full + s);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: one fresh partial per k-block, lo*hi + hi*lo + hi*hi
      constexpr uint32_t idesc = instr_desc<BN>();
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % ST, u = kb / ST, buf = kb & 1, ub = kb >> 1;
        if (ub > 0) mbar_wait(tempty + buf, (ub - 1) & 1);
        mbar_wait(conv + s, u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint8_t* st = smem + s * S::STAGE;
        const uint64_t ah = smem_desc(st), al = smem_desc(st + S::A_BYTES);
        const uint64_t bh = smem_desc(st + 2 * S::A_BYTES), bl = smem_desc(st + 2 * S::A_BYTES + S::B_BYTES);
        const uint32_t td = tmem + (uint32_t)(buf * BN);
#pragma unroll
        for (int k = 0; k < TK / UK; ++k) {
          const uint64_t dk = (uint64_t)((k * UK * 4) >> 4);      // +32 bytes along K inside the swizzle row
          umma_tf32(td, al + dk, bh + dk, idesc, k != 0);
          umma_tf32(td, ah + dk, bl + dk, idesc, 1u);
          umma_tf32(td, ah + dk, bh + dk, idesc, 1u);
        }
        umma_commit(empty + s);
        umma_commit(tfull + buf);
      }
    }
  } else {
    // ---- split + drain warps (2..5); TMEM lane quarter = warp % 4
    const int et = threadIdx.x - 64;                         // 0..127
    const int q = warp & 3;
    const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
    float acc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.f;
    auto drain = [&](int kb) {
      const int buf = kb & 1;
      mbar_wait(tfull + buf, (kb >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 64) {
        uint32_t r[64];
#pragma unroll
        for (int c = 0; c < 64; c += 16) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
              "[%16];"
              : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]),
                "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
              : "r"(tlane + (uint32_t)(buf * BN + c0 + c)));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 64; ++j) acc[c0 + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty + buf);
    };
    // split the raw B tile of k-block kb's stage: hi in place, lo into the next tile
    auto split = [&](int kb) {
      const int s = kb % ST, u = kb / ST;
      mbar_wait(full + s, u & 1);
      const uint32_t bh = smem_u32(smem + s * S::STAGE + 2 * S::A_BYTES);
      const uint32_t bl = bh + S::B_BYTES;
#pragma unroll
      for (int i = et * 16; i < S::B_BYTES; i += 128 * 16) {
        float x0, x1, x2, x3;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3) : "r"(bh + i));
        const float h0 = tf32_rna_dev(x0), h1 = tf32_rna_dev(x1), h2 = tf32_rna_dev(x2), h3 = tf32_rna_dev(x3);
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(bh + i), "f"(h0), "f"(h1), "f"(h2), "f"(h3)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(bl + i), "f"(tf32_rna_dev(x0 - h0)),
                     "f"(tf32_rna_dev(x1 - h1)), "f"(tf32_rna_dev(x2 - h2)), "f"(tf32_rna_dev(x3 - h3))
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(conv + s);
    };
    // split one k-block ahead of the drain so the tensor pipe never waits on it
    split(0);
    for (int kb = 0; kb < nkb; ++kb) {
      if (kb + 1 < nkb) split(kb + 1);
      drain(kb);
    }
    const int row = m0 + q * 32 + lane;
    if (row < M) {
#pragma unroll
      for (int j = 0; j < BN; ++j) {
        const int col = n0 + j;
        if (col < N) C[(int64_t)col * ldc + row] = acc[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_avail = 0;
std::once_flag g_once;

void init_once() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess && fn) {
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    g_avail = 1;
  } else {
    g_avail = -1;
  }
}

// 2-D K-major operand: rows of `rows` x `K` floats with pitch `ld` floats; box TK x box_rows
bool make_map(CUtensorMap* m, const float* p, int K, int rows, int64_t ld, int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)TK, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int ST>
bool launch(int M, int N, int K, const float* ah, const float* al, int64_t lda, const float* b, int64_t ldb,
            float* C, int64_t ldc, cudaStream_t s) {
  CUtensorMap mAh, mAl, mB;
  if (!make_map(&mAh, ah, K, M, lda, TM) || !make_map(&mAl, al, K, M, lda, TM) || !make_map(&mB, b, K, N, ldb, BN))
    return false;
  constexpr int smem = Smem<BN, ST>::TOTAL;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc3_gemm_kernel<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return false;
    attr = true;
  }
  dim3 grid((unsigned)((M + TM - 1) / TM), (unsigned)((N + BN - 1) / BN));
  tc3_gemm_kernel<BN, ST><<<grid, 192, smem, s>>>(mAh, mAl, mB, M, N, K, C, ldc);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace

int tc3_available() {
  std::call_once(g_once, init_once);
  return g_avail;
}

bool tc3_gemm(int M, int N, int K, const float* a_hi, const float* a_lo, int64_t lda, const float* b, int64_t ldb,
              float* C, int64_t ldc, cudaStream_t s) {
  if (M <= 0 || N <= 0) return true;
  if (K <= 0 || tc3_available() != 1) return false;
  if ((lda & 3) || (ldb & 3) || (((uintptr_t)a_hi | (uintptr_t)a_lo | (uintptr_t)b) & 15)) return false;
  // fill the 148 SMs: 128 x 128 tiles when they already give >= one wave, else 128 x 64
  const int tiles128 = ((M + TM - 1) / TM) * ((N + 127) / 128);
  if (tiles128 >= 148) return launch<128, 3>(M, N, K, a_hi, a_lo, lda, b, ldb, C, ldc, s);
  return launch<64, 4>(M, N, K, a_hi, a_lo, lda, b, ldb, C, ldc, s);
}

}  // namespace ell1
