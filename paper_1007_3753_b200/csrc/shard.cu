// shard.cu — device primitives of the column-sharded single-instance FISTA
// (BASELINE config 4: A = [A_0 ... A_{G-1}] by columns, one rank per GPU, one
// NCCL allreduce of the d-length partial A x per iteration).
//
//   ell1_gemv        y = A x          (panel partials + fixed-order row reduction)
//   ell1_gemv_t      g = A^T r        (panel GEMV^T, local to each column)
//   ell1_shard_prox  x_next = soft(y - g_y/L, lam/L) over the local columns with
//                    the backtracking / stopping partial sums (shrinkage.py:199-213)
//   ell1_shard_resid r_next = (A x_next) - b, ||r||^2, ||r_y'||^2 (replicated d side)
//   ell1_shard_kkt   KKT / support partials of the local columns (model.py:160-173, 227-233)
// All reductions are deterministic (fixed order); scalar partials are
// returned per rank for the host driver to combine across ranks.
#include <cstdlib>
#include "solvers_common.cuh"

namespace ell1 {

struct GvArgs {
  DictRaw D;
  const double* x;
  double* y;
  GridBufs g;
};

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) gemv_partial_kernel(const __grid_constant__ GvArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
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
                                                           double* y) {
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
// deterministic.  3 stages x (16 columns x 1024 rows) = 192 KB of A in flight
// per SM keeps HBM busy: 7.1 TB/s at d = 65536 (the register-staged engine
// path holds ~32 KB per SM and reached 4.8 TB/s; 8-column x 4-stage 5.9,
// 16 x 512-row stages 4.2 — measured with tools/gemv_bench.py).
namespace gts {
#ifndef ELL1_GTS_CB
#define ELL1_GTS_CB 16
#endif
#ifndef ELL1_GTS_RC
#define ELL1_GTS_RC 1024
#endif
constexpr int CB = ELL1_GTS_CB;           // columns per block
constexpr int RC = ELL1_GTS_RC;           // rows per chunk (2 per consumer thread)
#ifndef ELL1_GTS_ST
#define ELL1_GTS_ST 3
#endif
constexpr int ST = ELL1_GTS_ST;           // ring depth
constexpr int CW = 16;                    // consumer warps
constexpr int THREADS = (CW + 1) * 32;    // + producer warp
constexpr int A_BYTES = CB * RC * 4;
constexpr int R_BYTES = RC * 8;
constexpr int STAGE = A_BYTES + R_BYTES;
constexpr int SMEM = ST * STAGE + 2 * ST * 8 + CW * CB * 8 + 64;
}  // namespace gts

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(gts::THREADS, 1)
    gemv_t_stream_kernel(const float* __restrict__ A, int64_t ld, int64_t d, int64_t n, const double* __restrict__ r,
                         double* __restrict__ g) {
  using namespace gts;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + ST * STAGE);
  uint64_t* empty = full + ST;
  double* red = (double*)(empty + ST);                  // [CW][CB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // balanced contiguous column ranges per CTA, in blocks of CB
  const int64_t nblk = (n + CB - 1) / CB;
  const int64_t b0 = nblk * blockIdx.x / gridDim.x, b1 = nblk * (blockIdx.x + 1) / gridDim.x;
  const int nch = (int)((d + RC - 1) / RC);
  const int64_t total = (b1 - b0) * nch;                  // (block, chunk) steps of this CTA
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + s)), "r"(CW));
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
      for (int64_t t = 0; t < total; ++t) {
        const int s = (int)(t % ST);
        const int64_t u = t / ST;
        if (u > 0) wait(empty + s, (unsigned)((u - 1) & 1));
        const int64_t blk = b0 + t / nch;
        const int ch = (int)(t % nch);
        const int64_t row0 = (int64_t)ch * RC;
        const int rows = (int)((d - row0) < RC ? (d - row0) : RC);
        const int64_t c0 = blk * CB;
        const int cols = (int)((n - c0) < CB ? (n - c0) : CB);
        unsigned char* st = sm + (size_t)s * STAGE;
        const unsigned bytes = (unsigned)(cols * rows * 4 + rows * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(bytes)
                     : "memory");
        for (int c = 0; c < cols; ++c)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(st + (size_t)c * RC * 4)),
              "l"(A + (c0 + c) * ld + row0), "r"(rows * 4), "r"(su32(full + s))
              : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(st + A_BYTES)),
                     "l"(r + row0), "r"(rows * 8), "r"(su32(full + s))
                     : "memory");
      }
    }
    return;
  }
  // ---- consumers: thread t owns rows 2t, 2t+1 of every chunk
  const int tc = threadIdx.x;                           // 0 .. CW*32-1
  double acc[CB];
  for (int64_t t = 0; t < total; ++t) {
    const int s = (int)(t % ST);
    const int64_t u = t / ST;
    const int ch = (int)(t % nch);
    const int64_t blk = b0 + t / nch;
    const int64_t row0 = (int64_t)ch * RC;
    const int rows = (int)((d - row0) < RC ? (d - row0) : RC);
    const int64_t c0 = blk * CB;
    const int cols = (int)((n - c0) < CB ? (n - c0) : CB);
    if (ch == 0)
#pragma unroll
      for (int c = 0; c < CB; ++c) acc[c] = 0.0;
    wait(full + s, (unsigned)(u & 1));
    const unsigned char* st = sm + (size_t)s * STAGE;
    for (int i = 2 * tc; i < rows; i += 2 * CW * 32) {
      const double2 rv = *reinterpret_cast<const double2*>(st + A_BYTES + (size_t)i * 8);
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        if (c < cols) {
          const float2 av = *reinterpret_cast<const float2*>(st + ((size_t)c * RC + i) * 4);
          acc[c] = fma((double)av.x, rv.x, acc[c]);
          acc[c] = fma((double)av.y, rv.y, acc[c]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
    if (ch == nch - 1) {
      // column block done: fixed-order reduction (lanes -> xor tree, then warps in order)
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        double v = acc[c];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp * CB + c] = v;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
      if (tc < cols) {
        double v = red[tc];
        for (int w = 1; w < CW; ++w) v += red[w * CB + tc];
        g[c0 + tc] = v;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
    }
  }
}

static bool gemv_t_stream_ok(const ell1_dict_t* D) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("ELL1_GEMVT_STREAM");
    off = e && e[0] == '0';
  }
  return !off && D->dtype == ELL1_F32 && !D->ext && D->d >= 4096 && D->d % 32 == 0 && D->ld % 4 == 0;
}

// ---- elementwise + partial-sum kernels (grid-stride, CTA partials, then one CTA folds)
constexpr int SP = 8;

__global__ void __launch_bounds__(NTHR) shard_prox_kernel(int64_t n, const double* x, const double* xp,
                                                          const double* gx, const double* gxp, double* xn,
                                                          double m, double L, double thr, const double* gt,
                                                          double* part) {
  __shared__ double sh[NWARP * SP + SP];
  __shared__ Ctx E;
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double s[SP] = {0, 0, 0, 0, 0, 0, 0, 0};   // |xn|, gy.dl, dl.dl, max|xn|, (xn-x)^2, x^2, (xn-gt)^2, -
  for (int64_t k = (int64_t)blockIdx.x * NTHR + threadIdx.x; k < n; k += (int64_t)gridDim.x * NTHR) {
    const double xk = x[k];
    const double yk = xk + m * (xk - xp[k]);
    const double gk = (1.0 + m) * gx[k] - m * gxp[k];
    const double u = soft1(yk - gk / L, thr);
    xn[k] = u;
    const double dl = u - yk;
    s[0] += fabs(u);
    s[1] += gk * dl;
    s[2] += dl * dl;
    s[3] = nmax(s[3], fabs(u));
    const double dd = u - xk;
    s[4] += dd * dd;
    s[5] += xk * xk;
    if (gt) { const double e = u - gt[k]; s[6] += e * e; }
  }
  block_reduce<SP>(E, s, 1u << 3);
  if (threadIdx.x < SP) part[(int64_t)blockIdx.x * SP + threadIdx.x] = s[threadIdx.x];
}

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

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_gemv_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, 0);
  return grid_bytes(nb, D->d, 1) + (size_t)EW_BLOCKS * SP * 8 + 4096;
}

extern "C" int ell1_gemv(const ell1_dict_t* D, const double* x, double* y, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !x || !y) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, 0);
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = x; a.y = y;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_partial_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_partial_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_partial_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  gemv_reduce_kernel<<<nb, NTHR, 0, s>>>(a.g.part, a.g.rp, nb, D->d, y);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_gemv_t(const ell1_dict_t* D, const double* r, double* g, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !r || !g) return ELL1_ERR_ARG;
  if (gemv_t_stream_ok(D)) {
    cudaStream_t s = (cudaStream_t)stream;
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
    gemv_t_stream_kernel<<<sms, gts::THREADS, gts::SMEM, s>>>((const float*)D->A, D->ld, D->d, D->n, r, g);
    return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  }
  const int nb = pick_blocks(D->n, 0);
  GvArgs a;
  a.D = to_raw(D);
  a.D.ext = 0;
  a.x = r; a.y = g;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  const SmemPlan sp = plan_smem(a.D, nb, 0, 2, false);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (D->dtype == ELL1_F64) {
    cudaFuncSetAttribute(gemv_t_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<double><<<nb, NTHR, sp.bytes, s>>>(a);
  } else {
    cudaFuncSetAttribute(gemv_t_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    gemv_t_kernel<float><<<nb, NTHR, sp.bytes, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

static int ew_blocks(int64_t n) {
  int64_t b = (n + NTHR - 1) / NTHR;
  if (b > EW_BLOCKS) b = EW_BLOCKS;
  return b < 1 ? 1 : (int)b;
}

extern "C" int ell1_shard_prox(int64_t n, const double* x, const double* xp, const double* gx,
                               const double* gxp, double* xn, double m, double L, double lam,
                               const double* gt, double* out8, void* ws, void* stream) {
  if (n < 0 || !out8 || !ws || !(L > 0)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = ew_blocks(n);
  double* part = (double*)ws;
  shard_prox_kernel<<<nb, NTHR, 0, s>>>(n, x, xp, gx, gxp, xn, m, L, lam / L, gt, part);
  fold_kernel<<<1, 32, 0, s>>>(part, nb, 1u << 3, out8);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
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
