// dmma_gemm.cu — fp64 GEMM on the DMMA tensor path (see dmma_gemm.cuh).
//
// Tile: BM x BN = 64 x 64 per CTA, BK = 16 per pipeline stage, 4 warps in a
// 2 x 2 grid, each warp 32 x 32 = 2 x 4 mma.m16n8k4 tiles (8 fp64 accumulator
// fragments = 32 doubles per thread).  Operand tiles keep the global layout's
// contiguous direction contiguous in shared memory ("k-major" [BK][BM+8] for
// a column-major A, "m-major" [BM][BK+4] for a transposed one), with pads
// chosen so a warp's fragment read is exactly two 128-byte wavefronts.
// Loads are cp.async (16-byte when every column start is 16-byte aligned,
// else 8-byte), zero-filled past the matrix edges, 4 stages in flight.
//
// Split-K: when the output has too few tiles to fill the 148 SMs, the grid's
// z dimension splits K across a cluster of S CTAs (cluster dims 1 x 1 x S);
// ranks 1..S-1 park their fp64 partial tile in their own shared memory and
// rank 0 adds them in rank order through DSMEM (deterministic).
#include <cooperative_groups.h>
#include "dmma_gemm.cuh"
#include "ell1_b200.h"

namespace cg = cooperative_groups;

namespace ell1 {
namespace dm {

constexpr int BK = 16;
constexpr int PADK = 8;                    // k-major tiles: row of BM (or BN) + 8 doubles
constexpr int PADM = 4;                    // m-major tiles: row of BK + 4 doubles

template <int TR, int MN>                  // doubles per stage for one operand tile
struct Tile {
  static constexpr int SIZE = TR ? MN * (BK + PADM) : BK * (MN + PADK);
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int BYTES>
__device__ __forceinline__ void cp_async(double* dst, const double* src, int src_bytes) {
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One operand tile (rows x BK of op(X), rows = BM or BN) into shared memory.
//   TR = 0: op(X)(i, kk) = X[kk * ld + i]  -> smem [BK][rows + PADK] (k-major)
//   TR = 1: op(X)(i, kk) = X[i * ld + kk]  -> smem [rows][BK + PADM] (row-major in k)
// VEC = 2 (16-byte copies) or 1 (8-byte copies).
template <int TR, int ROWS, int VEC, int NT>
__device__ __forceinline__ void load_tile(double* sm, const double* __restrict__ X, int64_t ld, int64_t r0,
                                          int64_t rmax, int64_t k0, int64_t kmax) {
  if (TR == 0) {
    constexpr int CH = ROWS / VEC;
#pragma unroll 4
    for (int c = threadIdx.x; c < BK * CH; c += NT) {
      const int kk = c / CH, i = (c % CH) * VEC;
      const int64_t gk = k0 + kk, gi = r0 + i;
      int valid = 0;
      if (gk < kmax) valid = (int)((rmax - gi) < VEC ? (rmax - gi) : VEC);
      if (valid < 0) valid = 0;
      const double* src = valid > 0 ? X + gk * ld + gi : X;
      cp_async<VEC * 8>(sm + kk * (ROWS + PADK) + i, src, valid * 8);
    }
  } else {
    constexpr int CH = BK / VEC;
#pragma unroll 4
    for (int c = threadIdx.x; c < ROWS * CH; c += NT) {
      const int i = c / CH, kk = (c % CH) * VEC;
      const int64_t gi = r0 + i, gk = k0 + kk;
      int valid = 0;
      if (gi < rmax) valid = (int)((kmax - gk) < VEC ? (kmax - gk) : VEC);
      if (valid < 0) valid = 0;
      const double* src = valid > 0 ? X + gi * ld + gk : X;
      cp_async<VEC * 8>(sm + i * (BK + PADM) + kk, src, valid * 8);
    }
  }
}

// fragment element (row i of the tile, k index kk) of an operand tile
template <int TR, int ROWS>
__device__ __forceinline__ double frag(const double* sm, int i, int kk) {
  return TR == 0 ? sm[kk * (ROWS + PADK) + i] : sm[i * (BK + PADM) + kk];
}

__device__ __forceinline__ void mma_f64(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Tile shape: BM x BN per CTA, warps (BM/32) x (BN/32), each warp 32 x 32
// (2 x 4 m16n8 tiles), ST pipeline stages.
template <int BM_, int BN_, int ST_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, ST = ST_;
  static constexpr int WM = BM / 32, WN = BN / 32;
  static constexpr int THREADS = WM * WN * 32;
};

// TA: op(A) = A^T; TB: op(B) = B^T (B stored n x k).  For the B operand the
// tile rows are the n index: TB = 1 -> smem [BK][BN + PADK] (k-major) and
// TB = 0 -> smem [BN][BK + PADM].
template <class CF, int TA, int TB, int VA, int VB, int SPLIT>
__global__ void __launch_bounds__(CF::THREADS)
    dgemm_kernel(int64_t m, int64_t n, int64_t k, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc) {
  constexpr int BM = CF::BM, BN = CF::BN, ST = CF::ST, NT = CF::THREADS;
  extern __shared__ __align__(16) double smem[];
  constexpr int ASZ = Tile<TA, BM>::SIZE;
  constexpr int BSZ = Tile<TB ? 0 : 1, BN>::SIZE;
  double* As = smem;
  double* Bs = smem + ST * ASZ;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  // K range of this split (multiples of BK)
  const int64_t kt_all = (k + BK - 1) / BK;
  const int z = SPLIT > 1 ? (int)blockIdx.z : 0;
  const int64_t kt0 = kt_all * z / SPLIT, kt1 = kt_all * (z + 1) / SPLIT;
  const int64_t nkt = kt1 - kt0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp % CF::WM) * 32, wn = (warp / CF::WM) * 32;
  const int g = lane >> 2, t = lane & 3;

  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  auto issue = [&](int64_t kt, int slot) {
    const int64_t kk0 = (kt0 + kt) * BK;
    load_tile<TA, BM, VA, NT>(As + slot * ASZ, A, lda, m0, m, kk0, k);
    // op(B)(kk, j): TB = 0 -> B[j * ldb + kk] (rows j, contiguous k: TR = 1);
    //               TB = 1 -> B[kk * ldb + j] (contiguous j: TR = 0)
    load_tile<TB ? 0 : 1, BN, VB, NT>(Bs + slot * BSZ, B, ldb, n0, n, kk0, k);
  };

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nkt) issue(s, s);
    cp_commit();
  }
  for (int64_t kt = 0; kt < nkt; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    const int64_t nxt = kt + ST - 1;
    if (nxt < nkt) issue(nxt, (int)(nxt % ST));
    cp_commit();
    const double* as = As + (kt % ST) * ASZ;
    const double* bs = Bs + (kt % ST) * BSZ;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[2][2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a[i][0] = frag<TA, BM>(as, wm + i * 16 + g, kk + t);
        a[i][1] = frag<TA, BM>(as, wm + i * 16 + g + 8, kk + t);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = frag<TB ? 0 : 1, BN>(bs, wn + j * 8 + g, kk + t);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_f64(acc[i][j], a[i][0], a[i][1], b[j]);
    }
  }
  cp_wait<0>();
  __syncthreads();

  if (SPLIT > 1) {
    // park partial tiles (ranks > 0) in own smem as [warp][i][j][e][lane]; rank 0 adds in rank order
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    double* park = smem;
    if (rank > 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) park[(((warp * 2 + i) * 4 + j) * 4 + e) * 32 + lane] = acc[i][j][e];
    }
    cl.sync();
    if (rank == 0) {
      for (int r = 1; r < SPLIT; ++r) {
        const double* rp = cl.map_shared_rank(park, r);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] += rp[(((warp * 2 + i) * 4 + j) * 4 + e) * 32 + lane];
      }
    }
    cl.sync();
    if (rank != 0) return;
  }
  // epilogue: c0,c1 at (g, 2t..2t+1), c2,c3 at (g + 8, 2t..2t+1) of each 16 x 8 tile
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + wn + j * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = m0 + wm + i * 16 + g + 8 * h;
        if (row < m) {
          if (col < n) C[col * ldc + row] = acc[i][j][2 * h];
          if (col + 1 < n) C[(col + 1) * ldc + row] = acc[i][j][2 * h + 1];
        }
      }
    }
  }
}

template <class CF, int TA, int TB, int VA, int VB, int SPLIT>
static bool launch(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, cudaStream_t s) {
  constexpr int ASZ = Tile<TA, CF::BM>::SIZE;
  constexpr int BSZ = Tile<TB ? 0 : 1, CF::BN>::SIZE;
  constexpr int PIPE = CF::ST * (ASZ + BSZ) * 8;
  constexpr int PARK = SPLIT > 1 ? 32 * CF::THREADS * 8 : 0;        // split-K partial tile
  constexpr int SMEM = PIPE > PARK ? PIPE : PARK;
  auto kern = dgemm_kernel<CF, TA, TB, VA, VB, SPLIT>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) return false;
    attr_dev = dev;
  }
  dim3 grid((unsigned)((m + CF::BM - 1) / CF::BM), (unsigned)((n + CF::BN - 1) / CF::BN), (unsigned)SPLIT);
  if (SPLIT == 1) {
    kern<<<grid, CF::THREADS, SMEM, s>>>(m, n, k, A, lda, B, ldb, C, ldc);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(CF::THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = SPLIT;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, m, n, k, A, lda, B, ldb, C, ldc) != cudaSuccess) return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

template <class CF, int TA, int TB, int VA, int VB>
static bool with_split(int split, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
  switch (split) {
    case 8: return launch<CF, TA, TB, VA, VB, 8>(m, n, k, A, lda, B, ldb, C, ldc, s);
    case 4: return launch<CF, TA, TB, VA, VB, 4>(m, n, k, A, lda, B, ldb, C, ldc, s);
    case 2: return launch<CF, TA, TB, VA, VB, 2>(m, n, k, A, lda, B, ldb, C, ldc, s);
    default: return launch<CF, TA, TB, VA, VB, 1>(m, n, k, A, lda, B, ldb, C, ldc, s);
  }
}

using C64x64s4 = Cfg<64, 64, 4>;
using C64x64s3 = Cfg<64, 64, 3>;
using C128x64s3 = Cfg<128, 64, 3>;
using C64x128s3 = Cfg<64, 128, 3>;
using C128x128s3 = Cfg<128, 128, 3>;

// variant = tile config (0..4), split = K split (1, 2, 4, 8); -1 = heuristic
template <int TA, int TB, int VA, int VB>
static bool run(int variant, int split, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
  int bm = 64, bn = 64;
  if (variant < 0) variant = 1;
  switch (variant) {
    case 2: bm = 128; break;
    case 3: bn = 128; break;
    case 4: bm = bn = 128; break;
    default: break;
  }
  if (split < 0) {
    const int64_t tiles = ((m + bm - 1) / bm) * ((n + bn - 1) / bn);
    const int64_t kt = (k + BK - 1) / BK;
    const int per = (bm * bn >= 128 * 128) ? 1 : (bm * bn >= 128 * 64 ? 2 : 3);   // CTAs per SM
    split = 1;
    while (split < 8 && tiles * split * 2 <= 148 * per && kt / (split * 2) >= 8) split *= 2;
  }
  switch (variant) {
    case 0: return with_split<C64x64s4, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s);
    case 2: return with_split<C128x64s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s);
    case 3: return with_split<C64x128s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s);
    case 4: return with_split<C128x128s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s);
    default: return with_split<C64x64s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s);
  }
}

}  // namespace dm

bool dgemm_variant(int variant, int split, int transA, int transB, int64_t m, int64_t n, int64_t k,
                   const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   cudaStream_t s) {
  using namespace dm;
  if (m < 0 || n < 0 || k < 0 || ldc < m) return false;
  if (m == 0 || n == 0) return true;
  if (k == 0) return cudaMemset2DAsync(C, ldc * 8, 0, m * 8, n, s) == cudaSuccess;
  // 16-byte cp.async needs every column start (and the base) 16-byte aligned
  const bool va = ((uintptr_t)A & 15) == 0 && (lda & 1) == 0;
  const bool vb = ((uintptr_t)B & 15) == 0 && (ldb & 1) == 0;
#define ELL1_DG(TA, TB)                                                                                  \
  if (transA == TA && transB == TB) {                                                                    \
    if (va && vb) return run<TA, TB, 2, 2>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s);         \
    if (va) return run<TA, TB, 2, 1>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s);               \
    if (vb) return run<TA, TB, 1, 2>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s);               \
    return run<TA, TB, 1, 1>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s);                       \
  }
  ELL1_DG(0, 0)
  ELL1_DG(1, 0)
  ELL1_DG(0, 1)
#undef ELL1_DG
  return false;
}

bool dgemm(int transA, int transB, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
           const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
  return dgemm_variant(-1, -1, transA, transB, m, n, k, A, lda, B, ldb, C, ldc, s);
}

}  // namespace ell1

using namespace ell1;

extern "C" int ell1_gemm_f64(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, const double* A,
                             int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, void* stream) {
  if (M < 0 || N < 0 || K < 0 || ldc < M || (transA ? lda < K : lda < M) || (transB ? ldb < N : ldb < K))
    return ELL1_ERR_ARG;
  if (transA && transB) return ELL1_ERR_ARG;
  if (M && N && K && (!A || !B || !C)) return ELL1_ERR_ARG;
  return dgemm(transA, transB, M, N, K, A, lda, B, ldb, C, ldc, (cudaStream_t)stream) ? ELL1_OK : ELL1_ERR_CUDA;
}

// tuning entry (tools/dgemm_bench.py): a fixed tile variant (0..4) and K split (1/2/4/8, -1 auto)
extern "C" int ell1_gemm_f64_variant(int32_t variant, int32_t split, int32_t transA, int32_t transB, int64_t M,
                                     int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                                     int64_t ldb, double* C, int64_t ldc, void* stream) {
  if (M < 0 || N < 0 || K < 0 || ldc < M || (transA ? lda < K : lda < M) || (transB ? ldb < N : ldb < K))
    return ELL1_ERR_ARG;
  if ((transA && transB) || variant < 0 || variant > 4) return ELL1_ERR_ARG;
  return dgemm_variant(variant, split, transA, transB, M, N, K, A, lda, B, ldb, C, ldc, (cudaStream_t)stream)
             ? ELL1_OK
             : ELL1_ERR_CUDA;
}
