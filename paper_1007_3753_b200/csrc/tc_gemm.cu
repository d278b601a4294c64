// tc_gemm.cu — 3xTF32 tcgen05 GEMM for the batched fp32 solvers (see tc_gemm.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
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

#ifdef TC3_TIMING
__device__ unsigned long long g_tc3_dbg[16];
#define TW(slot, cond, stmt)                                        \
  {                                                                 \
    const long long _t = clock64();                                 \
    stmt;                                                           \
    if (cond) atomicAdd(&g_tc3_dbg[slot], (unsigned long long)(clock64() - _t)); \
  }
#else
#define TW(slot, cond, stmt) stmt;
#endif

template <int BN, int ST>
struct Smem {
  static constexpr int A_BYTES = TM * TK * 4;         // 16 KB
  static constexpr int B_BYTES = BN * TK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int TX = 2 * A_BYTES + B_BYTES;    // bytes TMA brings per stage (B arrives unsplit)
  static constexpr int TOTAL = ST * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

// Warp roles (320 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA
// issuer, warps 2-5 = drain, warps 6-9 = split.  Per k-block the split warps
// split the raw B tile in place (hi) and into the lo tile; every KC k-blocks
// the drain warps add the tensor pipe's TMEM partial product into fp32 registers (the tensor
// core's own accumulation spans only KC*32 products, the running sum is IEEE
// fp32: keeps the SIMT SGEMM's accuracy).  TMEM holds four BN-column partial
// buffers (BN <= 128; the MMA runs up to three k-blocks ahead of the drain).  On
// pre-split operands (PRE) the split warps have nothing to split and drain the
// upper half of the tile columns instead: each drain thread then keeps BN/2
// sums and issues all its tcgen05.ld before one wait.
// SK = 2 splits K over a 2-CTA cluster (small GEMMs: bigger tiles, same CTA
// count); rank 1 hands its fp32 sums to rank 0 through distributed shared
// memory and rank 0 adds them in a fixed order (deterministic) and writes C.
template <int BN, int ST, int KC, int SK, bool PRE>
__global__ void __launch_bounds__(320, 1)
    tc3_gemm_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mB, const __grid_constant__ CUtensorMap mBl, int M, int N,
                    int K, float* __restrict__ C, int64_t ldc) {
  using S = Smem<BN, ST>;
  static_assert(BN % 16 == 0 && BN <= 128 && (PRE || BN % 32 == 0), "BN");
  static_assert(SK == 1 || ST * S::STAGE >= BN * TM * 4, "partial exchange buffer");
#ifdef TC3_TIMING
  const long long t_start = clock64();
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + ST * S::STAGE);
  uint64_t* conv = full + ST;
  uint64_t* empty = conv + ST;
  constexpr int NBUF = 4 * BN <= 512 ? 4 : 2;   // TMEM partial buffers (BN columns each)
  constexpr int DG = PRE ? 2 : 1;               // drain warp groups (PRE: the idle split warps drain too)
  constexpr int DC = BN / DG;                   // accumulator columns per drain thread
  static_assert(DC % 8 == 0, "drain columns");
  uint64_t* tfull = empty + ST;       // [NBUF]
  uint64_t* tempty = tfull + NBUF;    // [NBUF]
  uint32_t* tmem_slot = (uint32_t*)(tempty + NBUF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * BN;
  const int nkb_all = (K + TK - 1) / TK;
  const int kz = SK == 1 ? 0 : (int)blockIdx.z;            // == cluster rank (cluster dims 1 x 1 x SK)
  const int kh = (nkb_all + SK - 1) / SK;
  const int kb0 = kz * kh;
  const int nkb = (nkb_all - kb0 < kh ? nkb_all - kb0 : kh);   // >= 1 when K > TK * (SK - 1)
  constexpr uint32_t TCOLS = NBUF * BN <= 32 ? 32 : NBUF * BN <= 64 ? 64 : NBUF * BN <= 128 ? 128 : NBUF * BN <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mAh) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mAl) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mB) : "memory");
    if (PRE) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mBl) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(conv + s, 128);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 128 * DG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  float acc[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) acc[j] = 0.f;
  const int q = warp & 3;                                    // TMEM lane quarter of a drain warp
  const bool drainw = warp >= 2 && warp < (PRE ? 10 : 6);
  const int cb = (DG == 2 && warp >= 6) ? DC : 0;            // first tile column of this drain thread

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST, u = i / ST, kc = (kb0 + i) * TK;
        if (u > 0) TW(0, true, mbar_wait(empty + s, (u - 1) & 1));
        uint8_t* st = smem + s * S::STAGE;
        mbar_expect_tx(full + s, PRE ? S::STAGE : S::TX);
        tma_load_2d(st, &mAh, kc, m0, full + s);
        tma_load_2d(st + S::A_BYTES, &mAl, kc, m0, full + s);
        tma_load_2d(st + 2 * S::A_BYTES, &mB, kc, n0, full + s);
        if (PRE) tma_load_2d(st + 2 * S::A_BYTES + S::B_BYTES, &mBl, kc, n0, full + s);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: one fresh partial per KC k-blocks, lo*hi + hi*lo + hi*hi
      constexpr uint32_t idesc = instr_desc<BN>();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST, u = i / ST, p = i / KC, buf = p % NBUF, ub = p / NBUF;
        const bool first = i % KC == 0, last = i % KC == KC - 1 || i == nkb - 1;
        if (first && ub > 0) TW(1, true, mbar_wait(tempty + buf, (ub - 1) & 1));
        TW(2, true, mbar_wait((PRE ? full : conv) + s, u & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint8_t* st = smem + s * S::STAGE;
        const uint64_t ah = smem_desc(st), al = smem_desc(st + S::A_BYTES);
        const uint64_t bh = smem_desc(st + 2 * S::A_BYTES), bl = smem_desc(st + 2 * S::A_BYTES + S::B_BYTES);
        const uint32_t td = tmem + (uint32_t)(buf * BN);
#pragma unroll
        for (int k = 0; k < TK / UK; ++k) {
          const uint64_t dk = (uint64_t)((k * UK * 4) >> 4);      // +32 bytes along K inside the swizzle row
          umma_tf32(td, al + dk, bh + dk, idesc, (k != 0 || !first) ? 1u : 0u);
          umma_tf32(td, ah + dk, bl + dk, idesc, 1u);
          umma_tf32(td, ah + dk, bh + dk, idesc, 1u);
        }
        umma_commit(empty + s);
        if (last) umma_commit(tfull + buf);
      }
    }
  } else if (drainw) {
    // ---- drain warps (2..5, and 6..9 on pre-split operands): TMEM partials -> fp32 registers
    const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)cb;
    constexpr int CH = DC <= 64 ? DC : 32;                   // columns in flight per tcgen05.wait::ld
    for (int p = 0; p < (nkb + KC - 1) / KC; ++p) {
      const int buf = p % NBUF;
      TW(3, threadIdx.x == 64, mbar_wait(tfull + buf, (p / NBUF) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < DC; c0 += CH) {
        uint32_t r[CH];
        if constexpr (CH % 16 == 0) {
#pragma unroll
          for (int c = 0; c < CH; c += 16) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                  "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]),
                  "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
                : "r"(tlane + (uint32_t)(buf * BN + c0 + c)));
          }
        } else {                                                 // 40 / 56 columns per thread (BN = 80 / 112)
#pragma unroll
          for (int c = 0; c < CH; c += 8) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]),
                           "=r"(r[c + 5]), "=r"(r[c + 6]), "=r"(r[c + 7])
                         : "r"(tlane + (uint32_t)(buf * BN + c0 + c)));
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < CH; ++j) acc[c0 + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty + buf);
    }
  } else {
    // ---- split warps (6..9): raw B tile -> hi in place, lo into the next tile
    const int et = threadIdx.x - 192;                        // 0..127
    for (int i = 0; i < (PRE ? 0 : nkb); ++i) {
      const int s = i % ST, u = i / ST;
      TW(4, threadIdx.x == 192, mbar_wait(full + s, u & 1));
      const uint32_t bh = smem_u32(smem + s * S::STAGE + 2 * S::A_BYTES);
      const uint32_t bl = bh + S::B_BYTES;
#pragma unroll
      for (int o = et * 16; o < S::B_BYTES; o += 128 * 16) {
        float x0, x1, x2, x3;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3) : "r"(bh + o));
        const float h0 = tf32_rna_dev(x0), h1 = tf32_rna_dev(x1), h2 = tf32_rna_dev(x2), h3 = tf32_rna_dev(x3);
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(bh + o), "f"(h0), "f"(h1), "f"(h2), "f"(h3)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(bl + o), "f"(tf32_rna_dev(x0 - h0)),
                     "f"(tf32_rna_dev(x1 - h1)), "f"(tf32_rna_dev(x2 - h2)), "f"(tf32_rna_dev(x3 - h3))
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(conv + s);
    }
  }
  const int row_l = q * 32 + lane;                           // tile row of a drain thread
  if constexpr (SK == 2) {
    // rank 1 -> rank 0 partial sums through DSMEM (the operand ring is idle now)
    const uint32_t xbuf = smem_u32(smem);
    // both CTAs are past their main loops before rank 1 writes into rank 0's ring
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (kz == 1 && drainw) {
      uint32_t rbuf;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbuf) : "r"(xbuf));
#pragma unroll
      for (int j = 0; j < DC; ++j)
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(rbuf + (uint32_t)(((cb + j) * TM + row_l) * 4)), "f"(acc[j])
                     : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (kz == 0 && drainw) {
#pragma unroll
      for (int j = 0; j < DC; ++j) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xbuf + (uint32_t)(((cb + j) * TM + row_l) * 4)));
        acc[j] += v;
      }
    }
  }
  if (drainw && kz == 0) {
    const int row = m0 + row_l;
    if (row < M) {
#pragma unroll
      for (int j = 0; j < DC; ++j) {
        const int col = n0 + cb + j;
        if (col < N) C[(int64_t)col * ldc + row] = acc[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
#ifdef TC3_TIMING
  if (threadIdx.x == 0) {
    atomicAdd(&g_tc3_dbg[5], (unsigned long long)(clock64() - t_start));
    atomicAdd(&g_tc3_dbg[6], 1ull);
  }
#endif
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

template <int BN, int ST, int SK, int KC, bool PRE>
bool launch(int M, int N, int K, const float* ah, const float* al, int64_t lda, const float* b, const float* bl,
            int64_t ldb, float* C, int64_t ldc, cudaStream_t s) {
  CUtensorMap mAh, mAl, mB, mBl;
  if (!make_map(&mAh, ah, K, M, lda, TM) || !make_map(&mAl, al, K, M, lda, TM) || !make_map(&mB, b, K, N, ldb, BN))
    return false;
  if (PRE ? !make_map(&mBl, bl, K, N, ldb, BN) : false) return false;
  if (!PRE) mBl = mB;
  constexpr int smem = Smem<BN, ST>::TOTAL;
  auto kern = tc3_gemm_kernel<BN, ST, KC, SK, PRE>;
  static unsigned attr = 0;                                  // per-device bit
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr >> (dev & 31) & 1u)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
    attr |= 1u << (dev & 31);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((M + TM - 1) / TM), (unsigned)((N + BN - 1) / BN), (unsigned)SK);
  cfg.blockDim = dim3(320, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = SK;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, mAh, mAl, mB, mBl, M, N, K, C, ldc) == cudaSuccess;
}

// SMEM bytes moved per k-block (TMA fill + in-smem split + three MMA operand reads),
// the resource that bounds these tiles
constexpr double kb_cost(int bn, bool pre = false) {
  return pre ? 80.0 * 1024 + 5.0 * bn * 128 : 80.0 * 1024 + 7.0 * bn * 128;
}

}  // namespace

#ifdef TC3_TIMING
void tc3_debug(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_tc3_dbg, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_tc3_dbg, z, sizeof(z));
  }
}
#endif

int tc3_available() {
  std::call_once(g_once, init_once);
  return g_avail;
}

bool tc3_gemm(int M, int N, int K, const float* a_hi, const float* a_lo, int64_t lda, const float* b, int64_t ldb,
              float* C, int64_t ldc, cudaStream_t s, const float* b_lo) {
  if (M <= 0 || N <= 0) return true;
  if (K <= 0 || tc3_available() != 1) return false;
  if ((lda & 3) || (ldb & 3) || (((uintptr_t)a_hi | (uintptr_t)a_lo | (uintptr_t)b | (uintptr_t)b_lo) & 15))
    return false;
  // pick the tile (BN) and K split (SK) with the least per-SM smem traffic on
  // the critical path: waves x k-blocks per CTA x bytes per k-block (+ fixed costs)
  const int mt = (M + TM - 1) / TM, nkb = (K + TK - 1) / TK;
  // (80- and 112-column tiles exist for pre-split operands only: their drain takes 40 / 56 columns per thread)
  struct Opt { int bn, sk; } opts[] = {{64, 1}, {80, 1}, {96, 1}, {112, 1}, {128, 1},
                                       {64, 2}, {80, 2}, {96, 2}, {112, 2}, {128, 2}};
  double best = 1e300;
  Opt pick = {64, 1};
  for (const Opt& o : opts) {
    if (o.sk == 2 && nkb < 4) continue;
    if (o.bn % 32 != 0 && !b_lo) continue;
    const long ctas = (long)mt * ((N + o.bn - 1) / o.bn) * o.sk;
    const long waves = (ctas + 147) / 148;
    const double kbs = (double)((nkb + o.sk - 1) / o.sk);
    const double t = waves * (kbs * kb_cost(o.bn, b_lo != nullptr) + 24.0 * 1024 + (o.sk == 2 ? 24.0 * 1024 : 0.0));
    if (t < best) { best = t; pick = o; }
  }
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("ELL1_TC3_FORCE");             // diagnostics: "<bn><sk>", e.g. 1282
    force = e ? atoi(e) : 0;
  }
  static int kc = -1;
  if (kc < 0) {
    const char* e = getenv("ELL1_TC3_KC");                // diagnostics: k-blocks per TMEM partial
    kc = e && atoi(e) == 2 ? 2 : 1;
  }
  int code = force ? force : pick.bn * 10 + pick.sk;
  if (!b_lo && (code / 10) % 32 != 0) code = pick.bn * 10 + pick.sk;   // forced pre-split-only tile, raw operand
#define TC3_CASE(BN_, ST_, SK_)                                                                         \
  case BN_ * 10 + SK_:                                                                                  \
    if (b_lo) return launch<BN_, ST_, SK_, 1, true>(M, N, K, a_hi, a_lo, lda, b, b_lo, ldb, C, ldc, s); \
    return kc == 2 ? launch<BN_, ST_, SK_, 2, false>(M, N, K, a_hi, a_lo, lda, b, b, ldb, C, ldc, s)    \
                   : launch<BN_, ST_, SK_, 1, false>(M, N, K, a_hi, a_lo, lda, b, b, ldb, C, ldc, s);
#define TC3_CASE_PRE(BN_, ST_, SK_)                                                                       \
  case BN_ * 10 + SK_:                                                                                  \
    if (b_lo) return launch<BN_, ST_, SK_, 1, true>(M, N, K, a_hi, a_lo, lda, b, b_lo, ldb, C, ldc, s); \
    return false;
  switch (code) {
    TC3_CASE_PRE(80, 4, 1)
    TC3_CASE_PRE(80, 4, 2)
    TC3_CASE_PRE(112, 3, 1)
    TC3_CASE_PRE(112, 3, 2)
    TC3_CASE(64, 4, 1)
    TC3_CASE(96, 3, 1)
    TC3_CASE(128, 3, 1)
    TC3_CASE(64, 4, 2)
    TC3_CASE(96, 3, 2)
    default:
    TC3_CASE(128, 3, 2)
  }
#undef TC3_CASE
#undef TC3_CASE_PRE
}

}  // namespace ell1
