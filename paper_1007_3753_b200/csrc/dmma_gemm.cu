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

constexpr int BK0 = 16;                    // k depth of one pipeline stage (default configs)
constexpr int PADK = 8;                    // k-major tiles: row of BM (or BN) + 8 doubles
constexpr int PADM = 4;                    // m-major tiles: row of BK + 4 doubles

template <int TR, int MN, int BK>          // doubles per stage for one operand tile
struct Tile {
  static constexpr int SIZE = TR ? MN * (BK + PADM) : BK * (MN + PADK);
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-thread cp.async plan for one operand tile (rows x BK of op(X), rows =
// BM or BN), fixed for the whole K loop: each thread owns PER chunks of VEC
// doubles; their source pointers advance by one k-tile per stage, row-edge
// byte counts are precomputed, and the k edge is only tested on the last tile.
//   TR = 0: op(X)(i, kk) = X[kk * ld + i]  -> smem [BK][rows + PADK] (k-major)
//   TR = 1: op(X)(i, kk) = X[i * ld + kk]  -> smem [rows][BK + PADM] (row-major in k)
template <int TR, int ROWS, int VEC, int NT, int BK>
struct Loader {
  static constexpr int CH = TR == 0 ? ROWS / VEC : BK / VEC;       // chunks per k (TR 0) / per row (TR 1)
  static constexpr int TOTAL = TR == 0 ? BK * CH : ROWS * CH;
  static constexpr int PER = (TOTAL + NT - 1) / NT;
  const double* src[PER];
  unsigned soff[PER];                                               // byte offset in the stage
  int bytes[PER];                                                   // row-edge clamped copy size
  int kk[PER];
  int64_t step;                                                     // doubles per k-tile
  const double* base;                                               // a valid address for empty copies

  __device__ __forceinline__ void init(const double* X, int64_t ld, int64_t r0, int64_t rmax, int64_t k0) {
    step = TR == 0 ? (int64_t)BK * ld : BK;
    base = X;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int c = threadIdx.x + q * NT;
      int kq, i;
      if (TR == 0) { kq = c / CH; i = (c % CH) * VEC; }
      else { i = c / CH; kq = (c % CH) * VEC; }
      kk[q] = c < TOTAL ? kq : BK;                                   // BK: never copies
      const int64_t gi = r0 + i;
      int b = 0;
      if (c < TOTAL && gi < rmax) b = TR == 0 ? (int)((rmax - gi) < VEC ? (rmax - gi) : VEC) * 8 : VEC * 8;
      bytes[q] = b;
      src[q] = TR == 0 ? X + (k0 + kq) * ld + gi : X + gi * ld + k0 + kq;
      soff[q] = (unsigned)(TR == 0 ? (kq * (ROWS + PADK) + i) : (i * (BK + PADM) + kq)) * 8u;
    }
  }
  __device__ __forceinline__ void copy(unsigned dst, const double* p, int b) {
    if (VEC == 2)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(p), "r"(b) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(p), "r"(b) : "memory");
  }
  // stage the k-tile starting at k0, then advance: interior tiles copy with
  // the precomputed sizes, only the last (k0 + BK > kmax) clamps the k edge
  __device__ __forceinline__ void load(unsigned stage, int64_t k0, int64_t kmax) {
    if (k0 + BK <= kmax) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        if (TOTAL % NT != 0 && kk[q] >= BK) continue;
        copy(stage + soff[q], bytes[q] ? src[q] : base, bytes[q]);
        src[q] += step;
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (kk[q] >= BK) continue;
      const int64_t left = kmax - (k0 + kk[q]);
      int b = bytes[q];
      if (TR == 0) b = left > 0 ? b : 0;
      else b = left <= 0 ? 0 : (left < VEC ? (int)left * 8 : b);
      copy(stage + soff[q], b ? src[q] : base, b);
      src[q] += step;
    }
  }
};

// fragment element (row i of the tile, k index kk) of an operand tile
template <int TR, int ROWS, int BK>
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
template <int BM_, int BN_, int ST_, int BK_ = BK0>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, ST = ST_, BK = BK_;
  static constexpr int WM = BM / 32, WN = BN / 32;
  static constexpr int THREADS = WM * WN * 32;
};

// TA: op(A) = A^T; TB: op(B) = B^T (B stored n x k).  For the B operand the
// tile rows are the n index: TB = 1 -> smem [BK][BN + PADK] (k-major) and
// TB = 0 -> smem [BN][BK + PADM].
template <class CF, int TA, int TB, int VA, int VB, int SPLIT>
__global__ void __launch_bounds__(CF::THREADS)
    dgemm_kernel(int64_t m, int64_t n, int64_t k, const double* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc, double alpha,
                 double beta) {
  constexpr int BM = CF::BM, BN = CF::BN, ST = CF::ST, NT = CF::THREADS, BK = CF::BK;
  extern __shared__ __align__(16) double smem[];
  constexpr int ASZ = Tile<TA, BM, BK>::SIZE;
  constexpr int BSZ = Tile<TB ? 0 : 1, BN, BK>::SIZE;
  double* As = smem;
  double* Bs = smem + ST * ASZ;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  // K range of this split (multiples of BK)
  const int64_t kt_all = (k + BK - 1) / BK;   // (CF::BK)
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

  // op(B)(kk, j): TB = 0 -> B[j * ldb + kk] (rows j, contiguous k: TR = 1);
  //               TB = 1 -> B[kk * ldb + j] (contiguous j: TR = 0)
  Loader<TA, BM, VA, NT, BK> la;
  Loader<TB ? 0 : 1, BN, VB, NT, BK> lb;
  la.init(A, lda, m0, m, kt0 * BK);
  lb.init(B, ldb, n0, n, kt0 * BK);
  const unsigned as0 = smem_u32(As), bs0 = smem_u32(Bs);
  int64_t kload = kt0 * BK;
  auto issue = [&](int slot) {
    la.load(as0 + (unsigned)(slot * ASZ * 8), kload, k);
    lb.load(bs0 + (unsigned)(slot * BSZ * 8), kload, k);
    kload += BK;
  };

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nkt) issue(s);
    cp_commit();
  }
  int slot_c = 0, slot_n = ST - 1;
  for (int64_t kt = 0; kt < nkt; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < nkt) issue(slot_n);
    cp_commit();
    slot_n = slot_n + 1 == ST ? 0 : slot_n + 1;
    const double* as = As + slot_c * ASZ;
    const double* bs = Bs + slot_c * BSZ;
    slot_c = slot_c + 1 == ST ? 0 : slot_c + 1;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[2][2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a[i][0] = frag<TA, BM, BK>(as, wm + i * 16 + g, kk + t);
        a[i][1] = frag<TA, BM, BK>(as, wm + i * 16 + g + 8, kk + t);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = frag<TB ? 0 : 1, BN, BK>(bs, wn + j * 8 + g, kk + t);
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
          if (beta == 0.0) {
            if (col < n) C[col * ldc + row] = alpha * acc[i][j][2 * h];
            if (col + 1 < n) C[(col + 1) * ldc + row] = alpha * acc[i][j][2 * h + 1];
          } else {
            if (col < n) C[col * ldc + row] = fma(alpha, acc[i][j][2 * h], beta * C[col * ldc + row]);
            if (col + 1 < n)
              C[(col + 1) * ldc + row] = fma(alpha, acc[i][j][2 * h + 1], beta * C[(col + 1) * ldc + row]);
          }
        }
      }
    }
  }
}

template <class CF, int TA, int TB, int VA, int VB, int SPLIT>
static bool launch(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double* C, int64_t ldc, cudaStream_t s, double alpha, double beta) {
  constexpr int ASZ = Tile<TA, CF::BM, CF::BK>::SIZE;
  constexpr int BSZ = Tile<TB ? 0 : 1, CF::BN, CF::BK>::SIZE;
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
    kern<<<grid, CF::THREADS, SMEM, s>>>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta);
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
    if (cudaLaunchKernelEx(&cfg, kern, m, n, k, A, lda, B, ldb, C, ldc, alpha, beta) != cudaSuccess) return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

template <class CF, int TA, int TB, int VA, int VB>
static bool with_split(int split, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, cudaStream_t s, double al, double be) {
  switch (split) {
    case 8: return launch<CF, TA, TB, VA, VB, 8>(m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    case 4: return launch<CF, TA, TB, VA, VB, 4>(m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    case 2: return launch<CF, TA, TB, VA, VB, 2>(m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    default: return launch<CF, TA, TB, VA, VB, 1>(m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
  }
}

using C64x64s4 = Cfg<64, 64, 4>;
using C64x64s3 = Cfg<64, 64, 3>;
using C128x64s3 = Cfg<128, 64, 3>;
using C64x64k32 = Cfg<64, 64, 3, 32>;
using C128x64k32 = Cfg<128, 64, 2, 32>;

// K split for a 64 x 64-tile launch (tuned on the batched solvers' shapes,
// tools/dgemm_bench.py): enough CTAs to fill the SMs (>= 256 in flight) while
// each split keeps >= 8 k-tiles; outputs of 512+ tiles with long K take one
// more split (shorter tails of the last wave).
static int pick_split(int64_t tiles, int64_t kt) {
  int s = 1;
  while (s < 8 && tiles * s < 256 && kt / (2 * s) >= 8) s *= 2;
  if (s < 8 && tiles >= 512 && tiles * s < 1024 && kt / (2 * s) >= 16) s *= 2;
  return s;
}

// variant = tile config (0..4), split = K split (1, 2, 4, 8); -1 = heuristic
template <int TA, int TB, int VA, int VB>
static bool run(int variant, int split, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s, double al, double be) {
  if (variant < 0) variant = 1;
  const int bm = (variant == 2 || variant == 4) ? 128 : 64, bn = 64;
  const int bk = variant >= 3 ? 32 : BK0;
  if (split < 0) split = pick_split(((m + bm - 1) / bm) * ((n + bn - 1) / bn), (k + bk - 1) / bk);
  switch (variant) {
    case 0: return with_split<C64x64s4, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    case 2: return with_split<C128x64s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    case 3: return with_split<C64x64k32, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    case 4: return with_split<C128x64k32, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
    default: return with_split<C64x64s3, TA, TB, VA, VB>(split, m, n, k, A, lda, B, ldb, C, ldc, s, al, be);
  }
}

}  // namespace dm

bool dgemm_variant(int variant, int split, int transA, int transB, int64_t m, int64_t n, int64_t k,
                   const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   cudaStream_t s, double alpha, double beta) {
  using namespace dm;
  if (m < 0 || n < 0 || k < 0 || ldc < m) return false;
  if (m == 0 || n == 0) return true;
  if (k == 0) {
    if (beta != 0.0) return false;                     // (not needed by the library)
    return cudaMemset2DAsync(C, ldc * 8, 0, m * 8, n, s) == cudaSuccess;
  }
  // 16-byte cp.async needs every column start (and the base) 16-byte aligned
  const bool va = ((uintptr_t)A & 15) == 0 && (lda & 1) == 0;
  const bool vb = ((uintptr_t)B & 15) == 0 && (ldb & 1) == 0;
#define ELL1_DG(TA, TB)                                                                                  \
  if (transA == TA && transB == TB) {                                                                    \
    if (va && vb) return run<TA, TB, 2, 2>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s, alpha, beta);         \
    if (va) return run<TA, TB, 2, 1>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s, alpha, beta);               \
    if (vb) return run<TA, TB, 1, 2>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s, alpha, beta);               \
    return run<TA, TB, 1, 1>(variant, split, m, n, k, A, lda, B, ldb, C, ldc, s, alpha, beta);                       \
  }
  ELL1_DG(0, 0)
  ELL1_DG(1, 0)
  ELL1_DG(0, 1)
#undef ELL1_DG
  return false;
}

bool dgemm(int transA, int transB, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
           const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s, double alpha, double beta) {
  return dgemm_variant(-1, -1, transA, transB, m, n, k, A, lda, B, ldb, C, ldc, s, alpha, beta);
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
  return dgemm_variant(variant, split, transA, transB, M, N, K, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, 1.0,
                       0.0)
             ? ELL1_OK
             : ELL1_ERR_CUDA;
}
