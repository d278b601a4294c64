// shard.cu — device primitives of the column-sharded single-instance FISTA
// (BASELINE config 4: A = [A_0 ... A_{G-1}] by columns, one rank per GPU, one
// NCCL allreduce of the d-length partial A x per iteration).
//
//   ell1_gemv        y = A x          (panel partials + fixed-order row reduction)
//   ell1_gemv_t      g = A^T r        (panel GEMV^T, local to each column)
//   ell1_sfista_pre  one backtracking trial up to the collective: prox on the
//                    local columns + the rank's scalar slot, then A_r x_next
//   ell1_sfista_post after the allreduce: residual, the FISTA decisions on the
//                    device, A_r^T r_next, rotation, KKT partials (next slot)
//   ell1_shard_resid / ell1_shard_kkt  set-up helpers (r = -b, max|A^T b|)
// All reductions are deterministic (fixed order), so every rank folds the
// allreduced slots to bit-identical control decisions.
#include <cstdlib>
#include "solvers_common.cuh"

namespace ell1 {

struct GvArgs {
  DictRaw D;
  const double* x;
  double* y;
  GridBufs g;
  const int* gate;            // NULL, or run only while *gate != 0 (device-side control)
};

__device__ __forceinline__ bool gated_off(const int* gate) {
  return gate != nullptr && *(const volatile int*)gate == 0;
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gemv_partial_kernel(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  if (gated_off(a.gate)) return;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const double* xs[1] = {a.x + E.c0};
  panel_gemv<TA, 1>(E, D, PN, xs);
}

// y[r0(o) + j] = sum_c part[o][c][j] in fixed order (block o reduces the
// region of row slice o; 16-byte loads, consecutive threads -> consecutive rows)
__global__ void __launch_bounds__(NTHR) gemv_reduce_kernel(const double* part, int rp, int nb, int64_t d,
                                                           double* y, const int* gate) {
  if (gated_off(gate)) return;
  const int o = blockIdx.x;
  const int64_t r0 = (d * o) / nb, r1 = (d * (o + 1)) / nb;
  const int rows = (int)(r1 - r0);
  const double* R = part + (size_t)o * nb * rp;
  for (int j = 2 * (int)threadIdx.x; j < rows; j += 2 * NTHR) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
    for (int c = 0; c < nb; ++c) {
      const double2 t = ldcg2(R + (size_t)c * rp + j);
      s0 += t.x;
      s1 += t.y;
    }
    y[r0 + j] = s0;
    if (j + 1 < rows) y[r0 + j + 1] = s1;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gemv_t_kernel(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  if (gated_off(a.gate)) return;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  if (threadIdx.x == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const double* rs[1] = {a.x};
  double* os[1] = {a.y + E.c0};
  panel_gemv_t<TA, 1>(E, D, PN, rs, os);
}

// ---- GEMV^T for long fp32 columns (config 4 panels: d = 65536 rows per column)
// A bulk-copy pipeline instead of register-staged loads: one producer lane
// streams, per stage, the next RC-row chunk of CB columns (CB bulk copies of
// RC x 4 bytes) and the matching RC doubles of r into an ST-deep shared-memory
// ring (mbarrier complete_tx); 16 consumer warps accumulate the CB column dots
// in fp64 registers (row pairs strided over the consumers) and release the slot.  Each
// column block ends in one fixed-order block reduction, so the result is
// deterministic.  2 stages x (4 columns x 4096 rows) = 128 KB of A (+ 64 KB
// of r) in flight per SM keeps HBM busy, and each copy is a 16 KB contiguous
// run of one column: over the whole 64 GiB single-GPU dictionary that beats
// 16 columns x 1024 rows (4 KB runs in 16 places 256 KB apart) by 12%, 6.73
// vs 5.99 TB/s, and equals it at the 8 GiB 8-way shard (7.04 vs 7.05;
// tools/gts_variants.sh).  Each staged r chunk serves GB = 4 column blocks
// (the r reads from L2 drop 4x): 6.73 -> 6.95 TB/s over 64 GiB.  The
// register-staged engine path holds ~32 KB per SM and reached 4.8 TB/s.
namespace gts {
#ifndef ELL1_GTS_CB
#define ELL1_GTS_CB 4
#endif
#ifndef ELL1_GTS_RC
#define ELL1_GTS_RC 4096
#endif
#ifndef ELL1_GTS_GB
#define ELL1_GTS_GB 4
#endif
constexpr int CB = ELL1_GTS_CB;           // columns per A stage
constexpr int RC = ELL1_GTS_RC;           // rows per chunk (row pairs strided over the consumers)
constexpr int GB = ELL1_GTS_GB;           // A stages (column blocks) sharing one staged r chunk
#ifndef ELL1_GTS_STA
#define ELL1_GTS_STA 2
#endif
constexpr int STA = ELL1_GTS_STA;         // A ring depth
constexpr int STR = 2;                    // r ring depth
constexpr int CW = 16;                    // consumer warps
constexpr int THREADS = (CW + 1) * 32;    // + producer warp
constexpr int KP = RC / (2 * CW * 32);    // row pairs per consumer thread and chunk
constexpr int A_BYTES = CB * RC * 4;
constexpr int R_BYTES = RC * 8;
constexpr int SMEM = STA * A_BYTES + STR * R_BYTES + 2 * (STA + STR) * 8 + CW * CB * GB * 8 + 64;
}  // namespace gts

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Column groups of GB blocks x CB columns walk the rows chunk by chunk; each
// r chunk is staged once per group and serves its GB column blocks (the r
// traffic from L2 is n / (GB CB) x d x 8 bytes per pass).  Per column, a
// thread accumulates its rows in increasing order over the chunks, then one
// fixed-order block reduction per group: bit-identical for any GB.
__global__ void __launch_bounds__(gts::THREADS, 1)
    gemv_t_stream_kernel(const float* __restrict__ A, int64_t ld, int64_t d, int64_t n, const double* __restrict__ r,
                         double* __restrict__ g, const int* gate) {
  using namespace gts;
  if (gated_off(gate)) return;
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* abuf = sm;                                     // [STA][A_BYTES]
  unsigned char* rbuf = sm + STA * A_BYTES;                     // [STR][R_BYTES]
  uint64_t* afull = (uint64_t*)(rbuf + STR * R_BYTES);
  uint64_t* aempty = afull + STA;
  uint64_t* rfull = aempty + STA;
  uint64_t* rempty = rfull + STR;
  double* red = (double*)(rempty + STR);                        // [CW][GB * CB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // balanced contiguous column ranges per CTA, in blocks of CB, grouped by GB
  const int64_t nblk = (n + CB - 1) / CB;
  const int64_t b0 = nblk * blockIdx.x / gridDim.x, b1 = nblk * (blockIdx.x + 1) / gridDim.x;
  const int64_t ngrp = (b1 - b0 + GB - 1) / GB;
  const int nch = (int)((d + RC - 1) / RC);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STA; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(afull + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(aempty + s)), "r"(CW));
    }
    for (int s = 0; s < STR; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(rfull + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(rempty + s)), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
  };
  if (warp == CW) {
    if (lane == 0) {
      // ---- producer
      int64_t as = 0, rs = 0;                                 // A / r steps issued
      for (int64_t gp = 0; gp < ngrp; ++gp) {
        const int64_t gb0 = b0 + gp * GB;
        const int nbg = (int)((b1 - gb0) < GB ? (b1 - gb0) : GB);
        for (int ch = 0; ch < nch; ++ch, ++rs) {
          const int64_t row0 = (int64_t)ch * RC;
          const int rows = (int)((d - row0) < RC ? (d - row0) : RC);
          {
            const int s = (int)(rs % STR);
            if (rs >= STR) wait(rempty + s, (unsigned)(((rs / STR) - 1) & 1));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(rfull + s)),
                         "r"((unsigned)(rows * 8))
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(rbuf + (size_t)s * R_BYTES)),
                "l"(r + row0), "r"(rows * 8), "r"(su32(rfull + s))
                : "memory");
          }
          for (int bi = 0; bi < nbg; ++bi, ++as) {
            const int s = (int)(as % STA);
            if (as >= STA) wait(aempty + s, (unsigned)(((as / STA) - 1) & 1));
            const int64_t c0 = (gb0 + bi) * CB;
            const int cols = (int)((n - c0) < CB ? (n - c0) : CB);
            unsigned char* st = abuf + (size_t)s * A_BYTES;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(afull + s)),
                         "r"((unsigned)(cols * rows * 4))
                         : "memory");
            for (int c = 0; c < cols; ++c)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      su32(st + (size_t)c * RC * 4)),
                  "l"(A + (c0 + c) * ld + row0), "r"(rows * 4), "r"(su32(afull + s))
                  : "memory");
          }
        }
      }
    }
    return;
  }
  // ---- consumers: thread t owns rows 2t, 2t + 1 (+ 1024 k) of every chunk
  const int tc = threadIdx.x;                           // 0 .. CW*32-1
  int64_t as = 0, rs = 0;
  for (int64_t gp = 0; gp < ngrp; ++gp) {
    const int64_t gb0 = b0 + gp * GB;
    const int nbg = (int)((b1 - gb0) < GB ? (b1 - gb0) : GB);
    double acc[GB][CB];
#pragma unroll
    for (int bi = 0; bi < GB; ++bi)
#pragma unroll
      for (int c = 0; c < CB; ++c) acc[bi][c] = 0.0;
    for (int ch = 0; ch < nch; ++ch, ++rs) {
      const int64_t row0 = (int64_t)ch * RC;
      const int rows = (int)((d - row0) < RC ? (d - row0) : RC);
      const int sr = (int)(rs % STR);
      wait(rfull + sr, (unsigned)((rs / STR) & 1));
      const unsigned char* rst = rbuf + (size_t)sr * R_BYTES;
      double2 rv[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int i = 2 * tc + 2 * CW * 32 * k;
        rv[k] = i < rows ? *reinterpret_cast<const double2*>(rst + (size_t)i * 8) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int bi = 0; bi < GB; ++bi) {
        if (bi < nbg) {
          const int sa = (int)(as % STA);
          wait(afull + sa, (unsigned)((as / STA) & 1));
          const unsigned char* st = abuf + (size_t)sa * A_BYTES;
          const int64_t c0 = (gb0 + bi) * CB;
          const int cols = (int)((n - c0) < CB ? (n - c0) : CB);
#pragma unroll
          for (int k = 0; k < KP; ++k) {
            const int i = 2 * tc + 2 * CW * 32 * k;
            if (i < rows) {
#pragma unroll
              for (int c = 0; c < CB; ++c) {
                if (c < cols) {
                  const float2 av = *reinterpret_cast<const float2*>(st + ((size_t)c * RC + i) * 4);
                  acc[bi][c] = fma((double)av.x, rv[k].x, acc[bi][c]);
                  acc[bi][c] = fma((double)av.y, rv[k].y, acc[bi][c]);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(aempty + sa)) : "memory");
          ++as;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(rempty + sr)) : "memory");
    }
    // column group done: fixed-order reduction (lanes -> xor tree, then warps in order)
#pragma unroll
    for (int bi = 0; bi < GB; ++bi)
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        double v = acc[bi][c];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp * GB * CB + bi * CB + c] = v;
      }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
    const int64_t gc0 = gb0 * CB;
    const int64_t gcols = ((b1 * CB < n ? b1 * CB : n) - gc0) < GB * CB ? ((b1 * CB < n ? b1 * CB : n) - gc0)
                                                                        : GB * CB;
    if (tc < gcols) {
      double v = red[tc];
      for (int w = 1; w < CW; ++w) v += red[w * GB * CB + tc];
      g[gc0 + tc] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
  }
}

// ---- GEMV partials for long fp32 columns (config 4: A_r x over the whole
// dictionary).  The same bulk-copy ring as the GEMV^T: per stage CB = 2
// columns x RC = 8192 rows (32 KB contiguous runs; over 64 GiB 7.21 TB/s vs
// 6.92 for 4 x 4096 and 6.93 for 8 x 2048, tools/gvs_variants.sh); CTA b walks its balanced
// column range one RC-row chunk at a time, 16 consumer warps accumulate the
// chunk's rows (row pairs strided over the threads) across the range's
// columns in column order, then write them slice-major into the partial
// buffer the fixed-order gemv_reduce_kernel folds (the engine's layout).
namespace gvs {
#ifndef ELL1_GVS_CB
#define ELL1_GVS_CB 2
#endif
#ifndef ELL1_GVS_RC
#define ELL1_GVS_RC 8192
#endif
#ifndef ELL1_GVS_ST
#define ELL1_GVS_ST 3
#endif
constexpr int CB = ELL1_GVS_CB;           // columns per stage
constexpr int RC = ELL1_GVS_RC;           // rows per chunk
constexpr int ST = ELL1_GVS_ST;           // ring depth
constexpr int CW = 16;                    // consumer warps
constexpr int THREADS = (CW + 1) * 32;
constexpr int KP = RC / (2 * CW * 32);    // row pairs per consumer thread and chunk
constexpr int A_BYTES = CB * RC * 4;
constexpr int SMEM = ST * A_BYTES + 2 * ST * 8 + 64;
}  // namespace gvs

__global__ void __launch_bounds__(gvs::THREADS, 1)
    gemv_stream_kernel(const float* __restrict__ A, int64_t ld, int64_t d, int64_t n, const double* __restrict__ x,
                       double* __restrict__ part, int rp, const int* gate) {
  using namespace gvs;
  if (gated_off(gate)) return;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + ST * A_BYTES);
  uint64_t* empty = full + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = gridDim.x, b = blockIdx.x;
  const int64_t c0 = (n * b) / nb, c1 = (n * (b + 1)) / nb;
  const int64_t nblk = (c1 - c0 + CB - 1) / CB;
  const int nch = (int)((d + RC - 1) / RC);
  const int64_t total = nblk * nch;                       // (row chunk, column block) steps, blocks inner
  if (threadIdx.x == 0) {
    for (int k = 0; k < ST; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + k)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + k)), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
  };
  if (warp == CW) {
    if (lane == 0) {
      for (int64_t t = 0; t < total; ++t) {
        const int s = (int)(t % ST);
        const int64_t u = t / ST;
        if (u > 0) wait(empty + s, (unsigned)((u - 1) & 1));
        const int ch = (int)(t / nblk);
        const int64_t blk = t % nblk;
        const int64_t row0 = (int64_t)ch * RC;
        const int rows = (int)((ld - row0) < RC ? (ld - row0) : RC);   // padded rows: 16-byte multiples
        const int64_t cb = c0 + blk * CB;
        const int cols = (int)((c1 - cb) < CB ? (c1 - cb) : CB);
        unsigned char* st = sm + (size_t)s * A_BYTES;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)),
                     "r"((unsigned)(cols * rows * 4))
                     : "memory");
        for (int c = 0; c < cols; ++c)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(st + (size_t)c * RC * 4)),
              "l"(A + (cb + c) * ld + row0), "r"(rows * 4), "r"(su32(full + s))
              : "memory");
      }
    }
    return;
  }
  const int tc = threadIdx.x;                            // 0 .. CW*32-1
  const int64_t reg = (int64_t)nb * rp;
  double acc[KP][2];
#pragma unroll
  for (int k = 0; k < KP; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int64_t t = 0; t < total; ++t) {
    const int s = (int)(t % ST);
    const int ch = (int)(t / nblk);
    const int64_t blk = t % nblk;
    const int64_t cb = c0 + blk * CB;
    const int cols = (int)((c1 - cb) < CB ? (c1 - cb) : CB);
    double xv[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) xv[c] = c < cols ? __ldg(x + cb + c) : 0.0;
    wait(full + s, (unsigned)((t / ST) & 1));
    const unsigned char* st = sm + (size_t)s * A_BYTES;
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      if (c < cols) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const float2 v = *reinterpret_cast<const float2*>(st + ((size_t)c * RC + 2 * tc + 2 * CW * 32 * k) * 4);
          acc[k][0] = fma((double)v.x, xv[c], acc[k][0]);
          acc[k][1] = fma((double)v.y, xv[c], acc[k][1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
    if (blk == nblk - 1) {
      // row chunk done: this CTA's partial of its rows, slice-major
      const int64_t row0 = (int64_t)ch * RC;
#pragma unroll
      for (int k = 0; k < KP; ++k)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t i = row0 + 2 * tc + 2 * CW * 32 * k + e;
          if (i < d) {
            const int64_t o = slice_owner(d, nb, i);
            part[o * reg + (int64_t)b * rp + (i - slice_r0(d, nb, o))] = acc[k][e];
          }
          acc[k][e] = 0.0;
        }
    }
  }
}

static bool gemv_t_stream_ok(const ell1_dict_t* D) {
  return D->dtype == ELL1_F32 && !D->ext && D->d >= 4096 && D->d % 32 == 0 && D->ld % 4 == 0;
}

// ---- elementwise + partial-sum kernels (grid-stride, CTA partials, then one CTA folds)
constexpr int SP = 8;

__global__ void __launch_bounds__(NTHR) shard_kkt_kernel(int64_t n, const double* x, const double* g, double lam,
                                                         double cut, double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};   // max_on, max_off, any_on, any_off, count, -, -, -
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = x[k];
    const double c = -g[k];
    if (xk != 0.0) { s[0] = nmax(s[0], fabs(c - lam * sgn(xk))); s[2] = 1.0; }
    else { s[1] = nmax(s[1], fabs(c)); s[3] = 1.0; }
    if (fabs(xk) > cut) s[4] += 1.0;
  }
  block_reduce<SP>(E, s, 0xFu);
  if (threadIdx.x < SP) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

__global__ void __launch_bounds__(NTHR) shard_resid_kernel(int64_t d, const double* ax, const double* b,
                                                           const double* rx, double mn, double* rn, double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * NTHR + threadIdx.x; i < d; i += (int64_t)gridDim.x * NTHR) {
    const double r = ax[i] - b[i];
    rn[i] = r;
    s[0] += r * r;
    const double ry = (1.0 + mn) * r - mn * rx[i];
    s[1] += ry * ry;
  }
  block_reduce<2>(E, s, 0u);
  if (threadIdx.x < 2) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

// fold CTA partials [nblk][SP] -> out[SP] (fixed order), maxmask selects max
__global__ void fold_kernel(const double* part, int nblk, unsigned maxmask, double* out) {
  const int k = threadIdx.x;
  if (k >= SP) return;
  const bool mx = (maxmask >> k) & 1u;
  double s = mx ? -INFINITY : 0.0;
  for (int c = 0; c < nblk; ++c) {
    const double t = part[(int64_t)c * SP + k];
    s = mx ? nmax(s, t) : s + t;
  }
  out[k] = s;
}

constexpr int EW_BLOCKS = 148 * 2;

// ---------------------------------------------------------------------------
// Device-controlled column-sharded FISTA rounds (ell1_sfista_pre / _post).
// Each kernel reduces its per-CTA partials with the "last CTA folds" pattern
// (ticket counter, fixed CTA order), so a round is 6 launches + 1 collective
// and nothing leaves the device.  Scalar arithmetic follows shrinkage.py
// (:199-213 backtracking, :184-196 t-sequence, :259-297 continuation, stop
// rules model.py:176-224, KKT model.py:160-173) with the same expressions as
// the single-GPU fista_kernel; the file is built with -fmad=false.
constexpr int SLOT = 16;                       // doubles per rank in xchg

struct SfWs {
  double* part;                                // [EW_BLOCKS][SP]
  unsigned* ticket;                            // [NTICKET]
};

__device__ __forceinline__ bool last_cta(unsigned* ticket) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// thread k < SP of the last CTA: fixed-order fold of the CTA partials
__device__ __forceinline__ double fold_parts(const double* part, int nblk, int k, bool mx) {
  double s = mx ? -INFINITY : 0.0;
  for (int c = 0; c < nblk; ++c) {
    const double t = ((const volatile double*)part)[(int64_t)c * SP + k];
    s = mx ? nmax(s, t) : s + t;
  }
  return s;
}

// K1: prox step on the local columns (shrinkage.py:204-207 with y, g_y as
// exact linear combinations of the cached iterates) + the rank's 8 partials.
__global__ void __launch_bounds__(NTHR) sf_prox_kernel(const ell1_shard_ctl_t* __restrict__ ctl, int64_t n,
                                                       ell1_sfista_bufs_t V, SfWs w) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  const int world = ctl->world, rank = ctl->rank;
  double* slots = V.xchg + 0;                  // caller passes xchg + ld as V.xchg here
  if (blockIdx.x == 0)
    for (int i = (int)threadIdx.x; i < world * SLOT; i += NTHR)
      if (i / SLOT != rank) slots[i] = 0.0;
  if (ctl->state != ELL1_SF_RUNNING) return;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  const double m = ctl->m, L = ctl->L, thr = ctl->lam_k / ctl->L;
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};   // |xn|, gy.dl, dl.dl, max|xn|, (xn-x)^2, x^2, (xn-gt)^2, -
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = V.x[k];
    const double yk = xk + m * (xk - V.xp[k]);
    const double gk = (1.0 + m) * V.g[k] - m * V.gp[k];
    const double u = soft1(yk - gk / L, thr);
    V.xn[k] = u;
    const double dl = u - yk;
    s[0] += fabs(u);
    s[1] += gk * dl;
    s[2] += dl * dl;
    s[3] = nmax(s[3], fabs(u));
    const double dd = u - xk;
    s[4] += dd * dd;
    s[5] += xk * xk;
    if (V.gt) { const double e = u - V.gt[k]; s[6] += e * e; }
  }
  block_reduce<SP>(E, s, 1u << 3);
  if (threadIdx.x < SP) w.part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
  if (last_cta(w.ticket + 0)) {
    if (threadIdx.x < SP) slots[rank * SLOT + threadIdx.x] = fold_parts(w.part, gridDim.x, threadIdx.x, threadIdx.x == 3);
    if (threadIdx.x == 0) w.ticket[0] = 0u;
  }
}

// K4: replicated residual r_n = A x_n - b (+ ||r_n||^2, ||r_y'||^2), then the
// decisions (one thread of the last CTA).
__global__ void __launch_bounds__(NTHR) sf_decide_kernel(ell1_shard_ctl_t* __restrict__ ctl, int64_t d,
                                                         int64_t ld, ell1_sfista_bufs_t V, SfWs w) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  const int st = ctl->state;
  if (st == ELL1_SF_FINISHED) return;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[2] = {0.0, 0.0};
  if (ctl->run_trial) {
    const double mn = ctl->mn;
    for (int64_t i = (int64_t)blockIdx.x * NTHR + threadIdx.x; i < d; i += (int64_t)gridDim.x * NTHR) {
      const double r = V.xchg[i] - V.b[i];
      V.rn[i] = r;
      s[0] += r * r;
      const double ry = (1.0 + mn) * r - mn * V.r[i];
      s[1] += ry * ry;
    }
  }
  block_reduce<2>(E, s, 0u);
  if (threadIdx.x < 2) w.part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
  if (!last_cta(w.ticket + 1)) return;
  __shared__ double rs[2];
  if (threadIdx.x < 2) rs[threadIdx.x] = fold_parts(w.part, gridDim.x, threadIdx.x, false);
  __syncthreads();
  if (threadIdx.x != 0) return;
  w.ticket[1] = 0u;
  ell1_shard_ctl_t& C = *ctl;
  const int world = C.world;
  const double* slots = V.xchg + ld;
  C.adv = 0;
  // (1) the previous accepted iteration's KKT (rode on this round's allreduce)
  if (C.pending) {
    double max_on = -INFINITY, max_off = -INFINITY, cnt = 0.0;
    bool any_on = false, any_off = false;
    for (int r = 0; r < world; ++r) {
      const double* q = slots + r * SLOT + SP;
      max_on = pymax(max_on, q[0]);
      max_off = pymax(max_off, q[1]);
      any_on = any_on || q[2] > 0.0;
      any_off = any_off || q[3] > 0.0;
      cnt += q[4];
    }
    double kk = 0.0;
    if (any_on) kk = max_on;
    if (any_off) kk = pymax(pymax(kk, max_off - C.lam_used), 0.0);
    V.trace[(C.it - 1) * 4 + 3] = rint(cnt);
    C.pending = 0;
    const bool conv = C.lam_used == C.lam_bar && kk <= C.tol * C.lam_bar;
    const bool kfire = C.stop_kind == ELL1_STOP_KKT && kk <= C.stop_thr;
    if (conv || kfire) C.converged = 1;
    if (conv || kfire || st == ELL1_SF_FINAL) {
      if (C.run_trial) C.passes += 1;          // the speculative trial's A x pass ran
      C.state = ELL1_SF_FINISHED;
      C.run_trial = 0;
      return;
    }
  }
  if (st != ELL1_SF_RUNNING) {                  // FINAL without a pending row: nothing left
    C.state = ELL1_SF_FINISHED;
    C.run_trial = 0;
    return;
  }
  // (2) this round's trial (shrinkage.py:199-213)
  double p[SP];
  for (int k = 0; k < SP; ++k) p[k] = 0.0;
  double mx = -INFINITY;
  for (int r = 0; r < world; ++r) {
    const double* q = slots + r * SLOT;
    p[0] = p[0] + q[0]; p[1] = p[1] + q[1]; p[2] = p[2] + q[2];
    p[4] = p[4] + q[4]; p[5] = p[5] + q[5]; p[6] = p[6] + q[6];
    mx = pymax(mx, q[3]);
  }
  p[3] = mx;
  C.trials += 1;
  C.passes += 1;
  const double l1 = p[0];
  const double Fn = 0.5 * rs[0] + C.lam_k * l1;
  if (!C.exact) {
    const double Q = C.f_y + p[1] + 0.5 * C.L * p[2] + C.lam_k * l1;
    if (!(Fn <= Q + 1e-12 * pymax(1.0, fabs(Q)))) {
      C.L *= C.eta;
      C.growths += 1;
      if (C.growths >= 101) {                   // shrinkage.py:24,203
        C.status = ELL1_BREAKDOWN;
        C.state = ELL1_SF_FINISHED;
        C.run_trial = 0;
      }
      return;
    }
  }
  // accepted: iteration it+1 done; rotation + A^T r_n + KKT partials follow (adv)
  C.growths = 0;
  C.it += 1;
  C.passes += 1;
  C.adv = 1;
  V.trace[(C.it - 1) * 4 + 0] = (double)C.it;
  V.trace[(C.it - 1) * 4 + 1] = Fn;
  V.trace[(C.it - 1) * 4 + 2] = sqrt(rs[0]);
  V.trace[(C.it - 1) * 4 + 3] = 0.0;
  C.pending = 1;
  C.lam_used = C.lam_k;
  C.cut = 1e-10 * pymax(p[3], 1.0);
  C.hist = C.hist + 1 < 2 ? C.hist + 1 : 2;
  const bool fires = C.stop_kind != ELL1_STOP_KKT &&
                     stop_fires(C.stop_kind, C.stop_thr, C.hist, Fn, C.F_prev, p[4], p[5], p[6], C.gt_norm, 0.0);
  const double t_new = fista_t_next(C.tc);     // the t computed at the top of this iteration
  C.tp = C.tc;
  C.tc = t_new;
  C.f_y = 0.5 * rs[1];
  C.F_prev = Fn;
  if (fires) C.converged = 1;
  if (fires || C.it >= C.max_iter) {
    C.state = ELL1_SF_FINAL;                   // one more round carries the KKT count
    C.run_trial = 0;
    return;
  }
  C.lam_k = pymax(C.beta * C.lam_k, C.lam_bar);
  // momentum of the next iteration and of its residual (shrinkage.py:266-272)
  C.m = (C.tp - 1.0) / C.tc;
  C.mn = (C.tc - 1.0) / fista_t_next(C.tc);
}

// K6: rotate (x_prev <- x <- x_n, g likewise, r <- r_n) and the KKT partials
// of the accepted iterate into the rank's slot (model.py:160-173, support
// cut 1e-10 max(max|x|, 1), model.py:227-233).
__global__ void __launch_bounds__(NTHR) sf_advance_kernel(const ell1_shard_ctl_t* __restrict__ ctl, int64_t n,
                                                          int64_t d, int64_t ld, ell1_sfista_bufs_t V, SfWs w) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (!ctl->adv) return;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  const double lam = ctl->lam_used, cut = ctl->cut;
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = V.xn[k], gk = V.gn[k];
    V.xp[k] = V.x[k];
    V.x[k] = xk;
    V.gp[k] = V.g[k];
    V.g[k] = gk;
    const double c = -gk;
    if (xk != 0.0) { s[0] = nmax(s[0], fabs(c - lam * sgn(xk))); s[2] = 1.0; }
    else { s[1] = nmax(s[1], fabs(c)); s[3] = 1.0; }
    if (fabs(xk) > cut) s[4] += 1.0;
  }
  for (int64_t i = (int64_t)blockIdx.x * NTHR + threadIdx.x; i < d; i += (int64_t)gridDim.x * NTHR) V.r[i] = V.rn[i];
  block_reduce<SP>(E, s, 0xFu);
  if (threadIdx.x < SP) w.part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
  if (last_cta(w.ticket + 2)) {
    double* slots = V.xchg + ld;
    if (threadIdx.x < SP)
      slots[ctl->rank * SLOT + SP + threadIdx.x] = fold_parts(w.part, gridDim.x, threadIdx.x, threadIdx.x < 4);
    if (threadIdx.x == 0) w.ticket[2] = 0u;
  }
}

}  // namespace ell1

using namespace ell1;

static int launch_gemv(const ell1_dict_t* D, const double* x, double* y, void* ws, size_t wsb, cudaStream_t s,
                       const int* gate) {
  const int nb = pick_blocks(D->n, 0);
  if (gemv_t_stream_ok(D) && D->d * D->n >= (int64_t(1) << 32) && !getenv("ELL1_GEMV_PANEL")) {
    // long fp32 columns of a >= 16 GiB dictionary: the bulk-copy ring (the
    // partial layout is the engine's).  64 GiB: 7.2 vs 6.36-6.74 TB/s for the
    // panel pass; at <= 8 GiB the panel pass is as fast or faster
    // (tools/gemv_bench.py, ELL1_GEMV_PANEL=1 forces the panel pass).
    GridBufs g;
    Carve cv(ws, wsb);
    if (!carve_grid(cv, g, nb, D->d, 1)) return ELL1_ERR_ARG;
    static unsigned attr = 0;                              // per-device bit
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr >> (dev & 31) & 1u)) {
      if (cudaFuncSetAttribute(gemv_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gvs::SMEM) !=
          cudaSuccess)
        return ELL1_ERR_CUDA;
      attr |= 1u << (dev & 31);
    }
    gemv_stream_kernel<<<nb, gvs::THREADS, gvs::SMEM, s>>>((const float*)D->A, D->ld, D->d, D->n, x, g.part, g.rp,
                                                           gate);
    gemv_reduce_kernel<<<nb, NTHR, 0, s>>>(g.part, g.rp, nb, D->d, y, gate);
    return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  }
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = x; a.y = y;
  a.gate = gate;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_partial_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_partial_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  gemv_reduce_kernel<<<nb, NTHR, 0, s>>>(a.g.part, a.g.rp, nb, D->d, y, gate);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

static int launch_gemv_t(const ell1_dict_t* D, const double* r, double* g, void* ws, size_t wsb, cudaStream_t s,
                         const int* gate) {
  if (gemv_t_stream_ok(D)) {
    static unsigned attr = 0;                              // per-device bit
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (!(attr >> (dev & 31) & 1u)) {
      if (cudaFuncSetAttribute(gemv_t_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gts::SMEM) !=
          cudaSuccess)
        return ELL1_ERR_CUDA;
      attr |= 1u << (dev & 31);
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gemv_t_stream_kernel<<<sms, gts::THREADS, gts::SMEM, s>>>((const float*)D->A, D->ld, D->d, D->n, r, g, gate);
    return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  }
  const int nb = pick_blocks(D->n, 0);
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = r; a.y = g;
  a.gate = gate;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_t_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_t_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" size_t ell1_gemv_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, D->d, 1) + (size_t)EW_BLOCKS * SP * 8 + 4096;
}

extern "C" int ell1_gemv(const ell1_dict_t* D, const double* x, double* y, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !x || !y) return ELL1_ERR_ARG;
  return launch_gemv(D, x, y, ws, wsb, (cudaStream_t)stream, nullptr);
}

extern "C" int ell1_gemv_t(const ell1_dict_t* D, const double* r, double* g, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !r || !g) return ELL1_ERR_ARG;
  return launch_gemv_t(D, r, g, ws, wsb, (cudaStream_t)stream, nullptr);
}

static int ew_blocks(int64_t n) {
  int64_t b = (n + NTHR - 1) / NTHR;
  if (b > EW_BLOCKS) b = EW_BLOCKS;
  return b < 1 ? 1 : (int)b;
}

extern "C" int ell1_shard_kkt(int64_t n, const double* x, const double* g, double lam, double cut,
                              double* out8, void* ws, void* stream) {
  if (n < 0 || !out8 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(n);
  double* part = (double*)ws;
  shard_kkt_kernel<<<nb, NTHR, 0, s>>>(n, x, g, lam, cut, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 0xFu, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_shard_resid(int64_t d, const double* ax, const double* b, const double* rx, double mn,
                                double* rn, double* out8, void* ws, void* stream) {
  if (d < 0 || !out8 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(d);
  double* part = (double*)ws;
  shard_resid_kernel<<<nb, NTHR, 0, s>>>(d, ax, b, rx, mn, rn, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 0u, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

// ---- device-controlled rounds
// workspace: [gemv grid scratch | EW_BLOCKS x SP partials | NTICKET tickets]
extern "C" size_t ell1_sfista_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  return ell1_gemv_workspace(D) + (size_t)EW_BLOCKS * SP * 8 + 256;
}

static bool sf_carve(const ell1_dict_t* D, void* ws, size_t wsb, SfWs& w, size_t& gws) {
  gws = ell1_gemv_workspace(D);
  if (!ws || wsb < ell1_sfista_workspace(D)) return false;
  w.part = (double*)((char*)ws + gws);
  w.ticket = (unsigned*)((char*)ws + gws + (size_t)EW_BLOCKS * SP * 8);
  return true;
}

static bool sf_bufs_ok(const ell1_sfista_bufs_t* V) {
  return V && V->x && V->xp && V->xn && V->g && V->gp && V->gn && V->r && V->rn && V->b && V->xchg && V->trace;
}

extern "C" int ell1_sfista_pre(const ell1_dict_t* D, ell1_shard_ctl_t* ctl, const ell1_sfista_bufs_t* V,
                               void* ws, size_t wsb, void* stream) {
  SfWs w;
  size_t gws;
  if (!dict_ok(D) || D->ext || !ctl || !sf_bufs_ok(V) || !sf_carve(D, ws, wsb, w, gws)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ell1_sfista_bufs_t P = *V;
  P.xchg = V->xchg + D->ld;                    // the prox kernel addresses the slot region
  sf_prox_kernel<<<ew_blocks(D->n), NTHR, 0, s>>>(ctl, D->n, P, w);
  if (cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
  return launch_gemv(D, V->xn, V->xchg, ws, gws, s, &ctl->run_trial);
}

extern "C" int ell1_sfista_post(const ell1_dict_t* D, ell1_shard_ctl_t* ctl, const ell1_sfista_bufs_t* V,
                                void* ws, size_t wsb, void* stream) {
  SfWs w;
  size_t gws;
  if (!dict_ok(D) || D->ext || !ctl || !sf_bufs_ok(V) || !sf_carve(D, ws, wsb, w, gws)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  sf_decide_kernel<<<ew_blocks(D->d), NTHR, 0, s>>>(ctl, D->d, D->ld, *V, w);
  if (cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
  const int rc = launch_gemv_t(D, V->rn, V->gn, ws, gws, s, &ctl->adv);
  if (rc != ELL1_OK) return rc;
  sf_advance_kernel<<<ew_blocks(D->n > D->d ? D->n : D->d), NTHR, 0, s>>>(ctl, D->n, D->d, D->ld, *V, w);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
