// engine.cuh — persistent-grid machinery shared by every single-instance solver.
//
// Execution model: one cooperative launch runs a whole solve.
// Each CTA owns
//   * a contiguous panel of dictionary columns  [c0, c1)   (w = c1 - c0)
//   * a contiguous slice of rows                 [r0, r1)   (d-side reductions)
//   * for the [A, sI] extension, the identity columns n + [r0, r1).
// Owned n-side vectors (x, g, ...) live in SHARED memory, indexed by a local
// column index k in [0, W): k < w is dictionary column c0 + k, k >= w is the
// identity column n + r0 + (k - w).  The first `rc` panel columns are
// resident in shared memory for the whole launch, the rest are streamed
// from global memory (L2 / HBM).
// D v is computed as per-CTA partial d-vectors (panel GEMV) reduced
// slice-by-slice after a grid barrier; D^T r is local to each panel.
// Every scalar decision is computed redundantly and bit-identically by all
// CTAs from deterministic fixed-order reductions — no broadcast needed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/ell1_b200.h"

#ifndef ELL1_GT_QU32
#define ELL1_GT_QU32 2    // fp32 long-column GEMV^T: row steps per lane in flight (2: +2% on a 4 GiB stream vs 1, 4 no better)
#endif

namespace ell1 {

constexpr int NTHR = 512;
constexpr int NWARP = NTHR / 32;
constexpr int SCAL = 32;                  // scalar slots per CTA per buffer
constexpr long long SPIN_LIMIT = 1LL << 26;

// ------------------------------------------------------------------ memory
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// E.sh (and everything carved from it) lives in shared memory; telling the
// compiler lets it emit LDS/STS instead of generic LD/ST, which it cannot
// infer through the pointer stored in the shared Ctx.
__device__ __forceinline__ double* shmem(double* p) {
  __builtin_assume(__isShared(p));
  return p;
}

__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// Per-CTA stride of K published scalars: a power of two >= 2.
__host__ __device__ constexpr int kpad(int K) {
  return K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32;
}

// Row-slice stride of the partial regions: the largest slice (ceil(d / nb)
// rows) padded to a power of two (<= 32 rows) or to an even count.
__host__ __device__ inline int rpad(int64_t d, int nb) {
  const int64_t rows = (d + nb - 1) / nb;
  if (rows <= 32) {
    int p = 2;
    while (p < rows) p <<= 1;
    return p;
  }
  return (int)((rows + 1) / 2 * 2);
}

// NaN-propagating max (np.max semantics)
__device__ __forceinline__ double nmax(double a, double b) { return (a > b || a != a) ? a : b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------ dictionary
template <class TA>
struct DictV {
  const TA* A;
  int64_t d, n, ld;   // ld == padded row count
  int ext;
  double s;
};

template <class TA>
struct VecOf { static constexpr int VW = 16 / (int)sizeof(TA); };

// ------------------------------------------------------------------ grid context
struct Ctx {            // lives in shared memory; written by thread 0 only
  int nb, b;
  int ok;             // result of the last grid barrier
  int64_t c0, c1;     // owned dictionary-column panel
  int64_t r0, r1;     // owned row slice
  int w, W;           // panel width, owned local columns (w + slice for ext)
  unsigned long long* bar;
  int* abort;
  unsigned long long epoch;
  unsigned nbar;      // barriers passed (selects scalar double-buffer)
  double* part;       // d-vector partials, slice-major (see panel_gemv)
  int64_t pvec;       // doubles per vector slot of `part` (nb * nb * rp)
  int rp;             // padded row-slice stride (rpad(d, nb))
  double* scal;       // [2][nb][SCAL]
  double* sh;         // shared scratch
  int64_t shcap;      // its capacity in doubles
  unsigned long long* prof;   // optional per-CTA phase timers [nb][16]
  unsigned long long tmark;
  unsigned long long pacc[16];  // phase accumulators (flushed to prof at mark(-1))
};

__device__ __forceinline__ int tix() { return (int)threadIdx.x; }
__device__ __forceinline__ int lnx() { return (int)(threadIdx.x & 31); }
__device__ __forceinline__ int wpx() { return (int)(threadIdx.x >> 5); }

// thread 0 only (Ctx is a __shared__ object); callers __syncthreads afterwards
// nb: CTAs cooperating on this solve (gridDim.x for a single-solve launch,
// the team size for a group launch, whose teams are consecutive CTAs).
__device__ __forceinline__ void ctx_init(Ctx& E, int64_t d, int64_t n, int ext, int nb) {
  E.nb = nb;
  E.b = (int)(blockIdx.x % (unsigned)nb);
  E.ok = 1;
  E.c0 = (n * E.b) / E.nb;
  E.c1 = (n * (E.b + 1)) / E.nb;
  E.r0 = (d * E.b) / E.nb;
  E.r1 = (d * (E.b + 1)) / E.nb;
  E.w = (int)(E.c1 - E.c0);
  E.W = E.w + (ext ? (int)(E.r1 - E.r0) : 0);
  E.epoch = 0;
  E.nbar = 0;
  E.prof = nullptr;
  E.tmark = 0;
  for (int k = 0; k < 16; ++k) E.pacc[k] = 0;
}

// global column index of local owned column k
__device__ __forceinline__ int64_t gcol(const Ctx& E, int64_t n, int k) {
  return k < E.w ? E.c0 + k : n + E.r0 + (k - E.w);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// accumulate the time since the previous mark into phase k (thread 0 of each
// CTA) in shared memory; mark(E, -1) (iteration start) stores the running
// totals to prof with plain stores, so no L2 round trip sits inside a phase.
__device__ __forceinline__ void mark(Ctx& E, int k) {
  if (tix() == 0 && E.prof != nullptr) {
    const unsigned long long t = gtimer();
    if (k >= 0) {
      E.pacc[k] += t - E.tmark;
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) E.prof[(size_t)E.b * 16 + q] = E.pacc[q];
    }
    E.tmark = t;
  }
}

// Software grid barrier: release-add on a monotone counter, acquire-poll
// until every CTA of this epoch arrived.  The acquire load orders (and
// invalidates L1 for) everything read after the barrier.  Returns false
// when a peer aborted or the wait timed out; callers unwind cleanly.
__device__ __forceinline__ bool grid_sync(Ctx& E) {
  __syncthreads();
  if (E.nb == 1) {                       // one-CTA team: a block barrier suffices
    if (tix() == 0) E.nbar++;
    __syncthreads();
    return true;
  }
  if (tix() == 0) {
    E.epoch += (unsigned long long)E.nb;
    E.nbar++;
    red_release_add(E.bar, 1ULL);        // MEMBAR.ALL.GPU + REDG: publishes the CTA's writes
    long long spins = 0;
    int ok = 1;
    const unsigned long long target = E.epoch;
    while (ld_acquire(E.bar) < target) {  // each acquire poll is LDG.STRONG.GPU + CCTL.IVALL
      if (((++spins) & 1023) == 0) {
        if (*(volatile int*)E.abort) { ok = 0; break; }
        if (spins > SPIN_LIMIT) { atomicExch(E.abort, 1); ok = 0; break; }
      }
    }
    E.ok = ok;
  }
  __syncthreads();
  return E.ok != 0;
}

// Split-phase form of grid_sync: arrive publishes this CTA's writes and
// counts it in; work placed between arrive and wait (by any thread) must not
// read data other CTAs write before the barrier — it overlaps the barrier's
// latency (thread-0 scalar bookkeeping, mostly).  No publish/gather between
// the two (the scalar double-buffer flips at arrive).
__device__ __forceinline__ void grid_arrive(Ctx& E) {
  __syncthreads();
  if (tix() == 0) {
    E.epoch += (unsigned long long)E.nb;
    E.nbar++;
    if (E.nb > 1) red_release_add(E.bar, 1ULL);
  }
}
__device__ __forceinline__ bool grid_wait(Ctx& E) {
  if (E.nb == 1) {
    __syncthreads();
    return true;
  }
  if (tix() == 0) {
    long long spins = 0;
    int ok = 1;
    const unsigned long long target = E.epoch;
    while (ld_acquire(E.bar) < target) {
      if (((++spins) & 1023) == 0) {
        if (*(volatile int*)E.abort) { ok = 0; break; }
        if (spins > SPIN_LIMIT) { atomicExch(E.abort, 1); ok = 0; break; }
      }
    }
    E.ok = ok;
  }
  __syncthreads();
  return E.ok != 0;
}

// ------------------------------------------------------------------ block reductions
// K values reduced across the CTA in a fixed order; every thread gets the result.
// Warp stage: a transpose-reduction over P = pow2 >= K slots costs
// (P - 1) + (5 - log2 P) shuffles instead of 5K (shuffle throughput is the
// limit with 16 warps); lane 4v.. then holds value v (P = 8).
template <int K>
__device__ __forceinline__ void block_reduce(const Ctx& E, double (&v)[K], unsigned maxmask) {
  constexpr int P = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
  constexpr int LOGP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : 4;
  static_assert(K <= 16, "block_reduce supports up to 16 values");
  double p[P];
#pragma unroll
  for (int k = 0; k < P; ++k) p[k] = k < K ? v[k] : (((maxmask >> k) & 1u) ? -INFINITY : 0.0);
  const int l = lnx();
  int base = 0;                                  // value index held in slot 0
#pragma unroll
  for (int r = 0; r < LOGP; ++r) {
    const int o = 16 >> r;                       // lane offset of this round
    const int h = P >> (r + 1);                  // slots kept after the round
    const bool upper = (l & o) != 0;
    if (upper) base += h;
#pragma unroll
    for (int u = 0; u < h; ++u) {
      const double send = upper ? p[u] : p[u + h];
      const double keep = upper ? p[u + h] : p[u];
      const double got = __shfl_xor_sync(0xffffffffu, send, o);
      p[u] = ((maxmask >> (base + u)) & 1u) ? nmax(keep, got) : keep + got;
    }
  }
  const bool mxf = (maxmask >> base) & 1u;
#pragma unroll
  for (int o = 16 >> LOGP; o > 0; o >>= 1) {
    const double got = __shfl_xor_sync(0xffffffffu, p[0], o);
    p[0] = mxf ? nmax(p[0], got) : p[0] + got;
  }
  double* sh = shmem(E.sh);
  // lane l holds value `base` iff l's low (5 - LOGP) bits are zero
  if ((l & ((32 >> LOGP) - 1)) == 0 && base < K) sh[wpx() * K + base] = p[0];
  __syncthreads();
  if (tix() < K) {
    const int k = tix();
    const bool mx = (maxmask >> k) & 1u;
    double t[NWARP];
#pragma unroll
    for (int w = 0; w < NWARP; ++w) t[w] = sh[w * K + k];
    double s = t[0];
#pragma unroll
    for (int w = 1; w < NWARP; ++w) s = mx ? nmax(s, t[w]) : s + t[w];
    sh[NWARP * K + k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sh[NWARP * K + k];
  __syncthreads();
}

// block_reduce whose results land in warp 0 only (thread 0 publishes them):
// one __syncthreads instead of three.  The caller must __syncthreads before
// E.sh is written again (panel_gemv / panel_gemv_t start with one).
template <int K>
__device__ __forceinline__ void block_reduce_w0(const Ctx& E, double (&v)[K], unsigned maxmask) {
  constexpr int P = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
  constexpr int LOGP = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : 4;
  static_assert(K <= 16, "block_reduce supports up to 16 values");
  double p[P];
#pragma unroll
  for (int k = 0; k < P; ++k) p[k] = k < K ? v[k] : (((maxmask >> k) & 1u) ? -INFINITY : 0.0);
  const int l = lnx();
  int base = 0;
#pragma unroll
  for (int r = 0; r < LOGP; ++r) {
    const int o = 16 >> r;
    const int h = P >> (r + 1);
    const bool upper = (l & o) != 0;
    if (upper) base += h;
#pragma unroll
    for (int u = 0; u < h; ++u) {
      const double send = upper ? p[u] : p[u + h];
      const double keep = upper ? p[u + h] : p[u];
      const double got = __shfl_xor_sync(0xffffffffu, send, o);
      p[u] = ((maxmask >> (base + u)) & 1u) ? nmax(keep, got) : keep + got;
    }
  }
  const bool mxf = (maxmask >> base) & 1u;
#pragma unroll
  for (int o = 16 >> LOGP; o > 0; o >>= 1) {
    const double got = __shfl_xor_sync(0xffffffffu, p[0], o);
    p[0] = mxf ? nmax(p[0], got) : p[0] + got;
  }
  double* sh = shmem(E.sh);
  if ((l & ((32 >> LOGP) - 1)) == 0 && base < K) sh[wpx() * K + base] = p[0];
  __syncthreads();
  if (wpx() == 0) {
    double s = 0.0;
    if (l < K) {
      const bool mx = (maxmask >> l) & 1u;
      double t[NWARP];
#pragma unroll
      for (int w = 0; w < NWARP; ++w) t[w] = sh[w * K + l];
      s = t[0];
#pragma unroll
      for (int w = 1; w < NWARP; ++w) s = mx ? nmax(s, t[w]) : s + t[w];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __shfl_sync(0xffffffffu, s, k);
  }
}

// Publish this CTA's K partial scalars into the buffer the next barrier
// selects: scal[buf][b * kpad(K) + k] (pad slots zero).
template <int K>
__device__ __forceinline__ void publish(const Ctx& E, const double (&v)[K]) {
  constexpr int KP = kpad(K);
  if (tix() == 0) {
    double* dst = E.scal + (size_t)((E.nbar + 1) & 1u) * E.nb * SCAL + (size_t)E.b * KP;
#pragma unroll
    for (int k = 0; k < KP; ++k) dst[k] = k < K ? v[k] : 0.0;
  }
}

// Published scalar k of CTA q (K published per CTA) in the current buffer.
__device__ __forceinline__ const double* published(const Ctx& E, int K, int q, int k) {
  return E.scal + (size_t)(E.nbar & 1u) * E.nb * SCAL + (size_t)q * kpad(K) + k;
}

// ----------------------------------------------------------------------------
// Cross-CTA reductions over "regions": nb rows (one per CTA) of RP doubles
// (RP a power of two in [2, 32]); entry j of the result = op over rows c of
// R[c * RP + j], op = max where maxmask bit j is set, else +.
// Every warp-wide load covers 64 consecutive doubles (16 B per lane, 4 L2
// lines), so a region of nb rows costs ceil(nb * RP / 64) warp loads — the
// loads of a warp are issued back to back (one L2 round trip).
// region_partial: warps wr in [0, nw) each fold a fixed subset of rows into
// lanes, reduce lanes holding the same entries, and leave entry j of their
// partial in red_row[j] (j < RP).  region_fold combines the nw partials in
// warp order.  The order of every combine is fixed, so results are
// bit-identical in every CTA.
constexpr int RU = 6;   // warp loads in flight per round

__device__ __forceinline__ double rop(bool mx, double a, double b) { return mx ? nmax(a, b) : a + b; }

__device__ __forceinline__ void region_partial(const double* R, int nb, int RP, unsigned maxmask,
                                               int wr, int nw, double* red_row) {
  const int l = lnx();
  const int G = 64 / RP;                      // rows per warp load
  const int j = (2 * l) & (RP - 1);
  const int cl = (2 * l) / RP;
  const bool m0 = (maxmask >> j) & 1u, m1 = (maxmask >> (j + 1)) & 1u;
  const double i0 = m0 ? -INFINITY : 0.0, i1 = m1 ? -INFINITY : 0.0;
  double a0 = i0, a1 = i1;
  const int ninstr = (nb + G - 1) / G;
  for (int u0 = wr; u0 < ninstr; u0 += nw * RU) {
    double2 t[RU];
#pragma unroll
    for (int uu = 0; uu < RU; ++uu) {
      const int u = u0 + uu * nw;
      const int c = u * G + cl;
      if (u < ninstr && c < nb) t[uu] = ldcg2(R + (size_t)c * RP + j);
      else t[uu] = make_double2(i0, i1);
    }
#pragma unroll
    for (int uu = 0; uu < RU; ++uu) { a0 = rop(m0, a0, t[uu].x); a1 = rop(m1, a1, t[uu].y); }
  }
  for (int o = RP / 2; o < 32; o <<= 1) {
    const double b0 = __shfl_xor_sync(0xffffffffu, a0, o);
    const double b1 = __shfl_xor_sync(0xffffffffu, a1, o);
    a0 = rop(m0, a0, b0);
    a1 = rop(m1, a1, b1);
  }
  if (2 * l < RP) { red_row[2 * l] = a0; red_row[2 * l + 1] = a1; }
}

__device__ __forceinline__ double region_fold(const double* red, int wl, int nw, int j, bool mx) {
  double s = red[wl * 32 + j];
  for (int w = 1; w < nw; ++w) s = rop(mx, s, red[(wl + w) * 32 + j]);
  return s;
}

// After a barrier: reduce the K published scalars over all CTAs (identical
// in every CTA).  maxmask bit k selects max instead of sum.
template <int K>
__device__ __forceinline__ void gather(const Ctx& E, double (&out)[K], unsigned maxmask) {
  static_assert(K <= 16, "up to 16 scalars");
  constexpr int KP = kpad(K);
  double* red = shmem(E.sh);                  // [NWARP][32]; results at red[16 + k]
  const double* src = E.scal + (size_t)(E.nbar & 1u) * E.nb * SCAL;
  region_partial(src, E.nb, KP, maxmask, wpx(), NWARP, red + wpx() * 32);
  __syncthreads();
  if (tix() < K) {
    const double r = region_fold(red, 0, NWARP, tix(), (maxmask >> tix()) & 1u);
    red[16 + tix()] = r;                      // row 0 upper half: never read by the folds
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = red[16 + k];
  __syncthreads();
}

// Grid-wide reduction of K per-thread values in one barrier (block reduce,
// publish, barrier, fixed-order gather).  Returns false on barrier failure.
template <int K>
__device__ __forceinline__ bool allreduce(Ctx& E, double (&v)[K], unsigned maxmask) {
  block_reduce<K>(E, v, maxmask);
  publish<K>(E, v);
  if (!grid_sync(E)) return false;
  gather<K>(E, v, maxmask);
  return true;
}

// Fused phase after the barrier that follows panel_gemv: the K scalar
// gathers and, for every owned row i, sums[v] = sum_c part_v[c][i] (fixed
// order), then f(i, sums, aux) with aux[a] = auxv[a][i] prefetched
// alongside the partial loads.  f runs on one thread per row; its
// per-thread accumulations are the caller's business.
// Small slices (rp <= 32): the scalar region and the NV partial regions are
// reduced concurrently by disjoint warp groups (one L2 round trip).  Large
// slices: one warp per 64-row chunk walks the nb partials with 16-byte loads.
// SHOUT: `out` is a shared-memory array written by the folding threads and
// valid for every thread on return (saves the broadcast round).
template <int K, int NV, int NA, bool SHOUT = false, class F>
__device__ void gather_slice(const Ctx& E, double* out, unsigned maxmask, int64_t /*ld*/,
                             const double* const (&auxv)[NA > 0 ? NA : 1], F&& f) {
  static_assert(K <= 16, "up to 16 scalars");
  constexpr int KP = kpad(K);
  double* red = shmem(E.sh);
  const int rows = (int)(E.r1 - E.r0);
  const int RP = E.rp;
  const int nb = E.nb;
  const double* own = E.part + (size_t)E.b * nb * RP;     // this CTA's region in slot 0
  if (RP <= 32) {
    constexpr int R = (K > 0 ? 1 : 0) + NV;
    double au[NA > 0 ? NA : 1];
    const int jt = tix();
    if (jt < rows) {
#pragma unroll
      for (int a = 0; a < NA; ++a) au[a] = ldcg(auxv[a] + E.r0 + jt);
    }
    const int w = wpx();
    const int r = ((w + 1) * R - 1) / NWARP;
    const int wl = (NWARP * r) / R, nw = (NWARP * (r + 1)) / R - wl;
    if (K > 0 && r == 0) {
      region_partial(E.scal + (size_t)(E.nbar & 1u) * nb * SCAL, nb, KP, maxmask, w - wl, nw,
                     red + w * 32);
    } else {
      const int v = r - (K > 0 ? 1 : 0);
      region_partial(own + (size_t)v * E.pvec, nb, RP, 0u, w - wl, nw, red + w * 32);
    }
    __syncthreads();
    if (jt < rows) {
      double sums[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int rr = v + (K > 0 ? 1 : 0);
        const int l0 = (NWARP * rr) / R, n0 = (NWARP * (rr + 1)) / R - l0;
        sums[v] = region_fold(red, l0, n0, jt, false);
      }
      f(E.r0 + jt, sums, au);
    }
    if (K > 0) {
      const int k = jt - 32;
      const int n0 = NWARP / R;                 // scalar region: warps [0, NWARP / R)
      double sk = 0.0;
      if (k >= 0 && k < K) sk = region_fold(red, 0, n0, k, (maxmask >> k) & 1u);
      // red[16 + k] lies in warp 0's row, upper half: no fold reads it
      if (k >= 0 && k < K) {
        if (SHOUT) out[k] = sk;
        else red[16 + k] = sk;
      }
      __syncthreads();
      if (!SHOUT) {
        for (int q = 0; q < K; ++q) out[q] = red[16 + q];
        __syncthreads();
      }
    } else {
      __syncthreads();
    }
  } else {
    if (K > 0) {
      double tmp[K > 0 ? K : 1];
      gather<(K > 0 ? K : 1)>(E, *reinterpret_cast<double(*)[K > 0 ? K : 1]>(tmp), maxmask);
      if (SHOUT) {
        if (tix() == 0)
          for (int q = 0; q < K; ++q) out[q] = tmp[q];
      } else {
        for (int q = 0; q < K; ++q) out[q] = tmp[q];
      }
    }
    for (int h = wpx(); h * 64 < rows; h += NWARP) {
      const int j = h * 64 + 2 * lnx();
      if (j < rows) {
        double acc[NV][2];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double* Rv = own + (size_t)v * E.pvec + j;
          double s0 = 0.0, s1 = 0.0;
          int c = 0;
          for (; c + 4 <= nb; c += 4) {
            double2 t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = ldcg2(Rv + (size_t)(c + u) * RP);
#pragma unroll
            for (int u = 0; u < 4; ++u) { s0 += t[u].x; s1 += t[u].y; }
          }
          for (; c < nb; ++c) {
            const double2 t = ldcg2(Rv + (size_t)c * RP);
            s0 += t.x; s1 += t.y;
          }
          acc[v][0] = s0; acc[v][1] = s1;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (j + e < rows) {
            const int64_t i = E.r0 + j + e;
            double au[NA > 0 ? NA : 1];
#pragma unroll
            for (int a = 0; a < NA; ++a) au[a] = ldcg(auxv[a] + i);
            double sums[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) sums[v] = acc[v][e];
            f(i, sums, au);
          }
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ panel
// Column jl of the CTA panel: resident in shared memory when jl < rc,
// streamed from global otherwise.
template <class TA>
struct Panel {
  const TA* sm;    // resident columns (rc of them)
  const TA* gl;    // global column c0
  int rc;
  int w;
  int oqv;         // 1: oq holds this thread's slice-major output offsets (ld / VW <= NTHR)
  int oq[VecOf<TA>::VW];   // offset of row tix() * VW + e in the partial slot (-1: padding row)
};

template <class TA>
__device__ __forceinline__ void ld16_sa(unsigned addr, TA (&a)[VecOf<TA>::VW]) {
  if constexpr (sizeof(TA) == 8) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a[0]), "=d"(a[1]) : "r"(addr));
  } else {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]) : "r"(addr));
  }
}
template <class TA>
__device__ __forceinline__ void ld16_s(const TA* p, TA (&a)[VecOf<TA>::VW]) {
  ld16_sa<TA>((unsigned)__cvta_generic_to_shared(p), a);
}
template <class TA>
__device__ __forceinline__ void ld16_g(const TA* p, TA (&a)[VecOf<TA>::VW]) {
  if constexpr (sizeof(TA) == 8) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    a[0] = t.x; a[1] = t.y;
  } else {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    a[0] = t.x; a[1] = t.y; a[2] = t.z; a[3] = t.w;
  }
}

// Panel over columns [c0, c0 + w) of an arbitrary column-major matrix
// (ld rows), first rc columns resident at dst.
template <class TA>
__device__ Panel<TA> setup_panel_at(const TA* Abase, int64_t ld, int64_t c0, int w, TA* dst, int rc) {
  Panel<TA> P;
  P.gl = Abase + c0 * ld;
  P.w = w;
  P.rc = rc < w ? rc : w;
  P.sm = dst;
  P.oqv = 0;
  const int64_t n4 = (int64_t)P.rc * ld * (int64_t)sizeof(TA) / 16;
  const int4* src = reinterpret_cast<const int4*>(P.gl);
  int4* d4 = reinterpret_cast<int4*>(dst);
  for (int64_t k = tix(); k < n4; k += NTHR) d4[k] = __ldg(src + k);
  __syncthreads();
  return P;
}

template <class TA>
__device__ __forceinline__ void panel_offsets_impl(const Ctx& E, const DictV<TA>& D, Panel<TA>& P);

// Copy the first rc panel columns (contiguous in the column-major layout)
// into shared memory.
template <class TA>
__device__ Panel<TA> setup_panel(const Ctx& E, const DictV<TA>& D, TA* dst, int rc) {
  Panel<TA> P;
  P.gl = D.A + E.c0 * D.ld;
  P.w = E.w;
  P.rc = rc < E.w ? rc : E.w;
  P.sm = dst;
  panel_offsets_impl<TA>(E, D, P);
  const int64_t n4 = (int64_t)P.rc * D.ld * (int64_t)sizeof(TA) / 16;
  const int4* src = reinterpret_cast<const int4*>(P.gl);
  int4* d4 = reinterpret_cast<int4*>(dst);
  for (int64_t k = tix(); k < n4; k += NTHR) d4[k] = __ldg(src + k);
  __syncthreads();
  return P;
}

// ------------------------------------------------------------------ panel GEMV
// Partial of CTA b for row i of vector slot s:  sum_{jl < w} A[i, c0 + jl] xs[v][jl]
// stored slice-major — in the region of the row's owner o (the CTA whose
// row slice holds i):  part[s * pvec + o * (nb * rp) + b * rp + (i - r0(o))].
// The owner then reads its nb x rp region with fully coalesced loads.
// xs: owned local vectors in shared memory.
// (32-bit arithmetic when d * nb fits, which covers every practical shape)
__device__ __forceinline__ int64_t slice_r0(int64_t d, int nb, int64_t o) {
  if (d * nb < 0xFFFFFFFFLL) return (int64_t)((unsigned)d * (unsigned)o / (unsigned)nb);
  return (d * o) / nb;
}
__device__ __forceinline__ int64_t slice_owner(int64_t d, int nb, int64_t i) {
  if (d * nb < 0xFFFFFFFFLL) return (int64_t)((((unsigned)i + 1u) * (unsigned)nb - 1u) / (unsigned)d);
  return ((i + 1) * nb - 1) / d;
}
// this thread's output offsets for its row vector (rows tix() * VW + e)
template <class TA>
__device__ __forceinline__ void panel_offsets_impl(const Ctx& E, const DictV<TA>& D, Panel<TA>& P) {
  constexpr int VW = VecOf<TA>::VW;
  const int64_t nvec = D.ld / VW;
  P.oqv = nvec <= NTHR ? 1 : 0;
  const int64_t reg = (int64_t)E.nb * E.rp;
  const int64_t i0 = (int64_t)tix() * VW;
  int64_t ow = i0 < D.d ? slice_owner(D.d, E.nb, i0) : 0;
  int64_t r0 = slice_r0(D.d, E.nb, ow), r1 = slice_r0(D.d, E.nb, ow + 1);
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    const int64_t i = i0 + e;
    P.oq[e] = -1;
    if (i < D.d) {
      while (i >= r1) { ++ow; r0 = r1; r1 = slice_r0(D.d, E.nb, ow + 1); }
      P.oq[e] = (int)(ow * reg + (i - r0));
    }
  }
}

template <class TA, int NV>
__device__ void panel_gemv(const Ctx& E, const DictV<TA>& D, const Panel<TA>& P,
                           const double* const (&xs)[NV], bool accumulate = false, int slot0 = 0) {
  constexpr int VW = VecOf<TA>::VW;
  constexpr int PF = 4;                            // streamed columns prefetched per group
  const int64_t nvec = D.ld / VW;
  const int w = P.w, rc = P.rc;
  double* out = E.part + (size_t)slot0 * E.pvec + (size_t)E.b * E.rp;
  const int64_t reg = (int64_t)E.nb * E.rp;      // region stride (one owner)
  __syncthreads();
  {
    // Short panels with many columns (small problems, group launches): KG
    // column groups of wgr warps each cover all rows; group g sums its column
    // range, the KG partials are added in group order through E.sh (first
    // NWARP * 32 doubles only).
    const int wgr = (int)((nvec + 31) >> 5);
    int KG = NWARP / wgr;
    const int64_t per = (int64_t)wgr * 32 * VW * NV;          // doubles per group partial
    while (KG > 1 && KG * per > NWARP * 32) --KG;
    if (KG > 1 && w >= 8 * KG) {
      const int grp = wpx() / wgr;
      const int64_t q = (int64_t)(wpx() - grp * wgr) * 32 + lnx();
      const bool act = grp < KG && q < nvec;
      double acc[NV][VW];
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[v][e] = 0.0;
      if (act) {
        const int ja = (int)(((int64_t)w * grp) / KG), jb = (int)(((int64_t)w * (grp + 1)) / KG);
        const unsigned p = (unsigned)__cvta_generic_to_shared(P.sm + q * VW);
        const unsigned cst = (unsigned)(D.ld * sizeof(TA));
        const TA* pg = P.gl + q * VW;
        int j = ja;
        for (; j + 4 <= jb; j += 4) {
          TA a[4][VW];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (j + u < rc) ld16_sa<TA>(p + (unsigned)(j + u) * cst, a[u]);
            else ld16_g<TA>(pg + (int64_t)(j + u) * D.ld, a[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double xv = xs[v][j + u];
#pragma unroll
              for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[u][e], xv, acc[v][e]);
            }
        }
        for (; j < jb; ++j) {
          TA a[VW];
          if (j < rc) ld16_sa<TA>(p + (unsigned)j * cst, a);
          else ld16_g<TA>(pg + (int64_t)j * D.ld, a);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double xv = xs[v][j];
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[e], xv, acc[v][e]);
          }
        }
      }
      double* st = shmem(E.sh);                                 // [KG][NV][rows]
      const int64_t rows = (int64_t)wgr * 32 * VW;
      if (act && grp > 0)
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < VW; ++e) st[(grp * NV + v) * rows + q * VW + e] = acc[v][e];
      __syncthreads();
      if (act && grp == 0) {
        for (int g = 1; g < KG; ++g)
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[v][e] += st[(g * NV + v) * rows + q * VW + e];
        const int64_t i0 = q * VW;
        int64_t ow = i0 < D.d ? slice_owner(D.d, E.nb, i0) : 0;
        int64_t r0 = slice_r0(D.d, E.nb, ow), r1 = slice_r0(D.d, E.nb, ow + 1);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          const int64_t i = i0 + e;
          if (i < D.d) {
            while (i >= r1) { ++ow; r0 = r1; r1 = slice_r0(D.d, E.nb, ow + 1); }
            double* o = out + ow * reg + (i - r0);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double* ov = o + (size_t)v * E.pvec;
              *ov = accumulate ? *ov + acc[v][e] : acc[v][e];
            }
          }
        }
      }
      __syncthreads();                                          // E.sh free again for the caller
      return;
    }
  }
  if (nvec >= 2 * NTHR && w - rc >= 8) {
    // Long mostly-streamed columns: each thread takes two consecutive row
    // vectors, so the CTA reads 2 x 8 KB-per-column runs as one contiguous
    // 16 KB run (HBM streams these faster than scattered 8 KB pieces).  The
    // per-row sum runs over the columns in the same order as below: the
    // result bits do not change.
    for (int64_t q0 = 2 * (int64_t)tix(); q0 < nvec; q0 += 2 * NTHR) {
      const bool has1 = q0 + 1 < nvec;
      double acc[2][NV][VW];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[h][v][e] = 0.0;
      const unsigned p = (unsigned)__cvta_generic_to_shared(P.sm + q0 * VW);
      const unsigned cst = (unsigned)(D.ld * sizeof(TA));
      const TA* pg = P.gl + q0 * VW;
      int j = 0;
      for (; j < rc; ++j) {
        TA a[2][VW];
        ld16_sa<TA>(p + (unsigned)j * cst, a[0]);
        if (has1) ld16_sa<TA>(p + (unsigned)j * cst + 16u, a[1]);
        else {
#pragma unroll
          for (int e = 0; e < VW; ++e) a[1][e] = (TA)0;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xs[v][j];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[h][v][e] = fma((double)a[h][e], xv, acc[h][v][e]);
        }
      }
      for (; j + 4 <= w; j += 4) {
        TA a[4][2][VW];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ld16_g<TA>(pg + (int64_t)(j + u) * D.ld, a[u][0]);
          if (has1) ld16_g<TA>(pg + (int64_t)(j + u) * D.ld + VW, a[u][1]);
          else {
#pragma unroll
            for (int e = 0; e < VW; ++e) a[u][1][e] = (TA)0;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double xv = xs[v][j + u];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int e = 0; e < VW; ++e) acc[h][v][e] = fma((double)a[u][h][e], xv, acc[h][v][e]);
          }
      }
      for (; j < w; ++j) {
        TA a[2][VW];
        ld16_g<TA>(pg + (int64_t)j * D.ld, a[0]);
        if (has1) ld16_g<TA>(pg + (int64_t)j * D.ld + VW, a[1]);
        else {
#pragma unroll
          for (int e = 0; e < VW; ++e) a[1][e] = (TA)0;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xs[v][j];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[h][v][e] = fma((double)a[h][e], xv, acc[h][v][e]);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i0 = (q0 + h) * VW;
        if (h == 1 && !has1) break;
        int64_t ow = i0 < D.d ? slice_owner(D.d, E.nb, i0) : 0;
        int64_t r0 = slice_r0(D.d, E.nb, ow), r1 = slice_r0(D.d, E.nb, ow + 1);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          const int64_t i = i0 + e;
          if (i < D.d) {
            while (i >= r1) { ++ow; r0 = r1; r1 = slice_r0(D.d, E.nb, ow + 1); }
            double* o = out + ow * reg + (i - r0);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double* ov = o + (size_t)v * E.pvec;
              *ov = accumulate ? *ov + acc[h][v][e] : acc[h][v][e];
            }
          }
        }
      }
    }
    return;
  }
  for (int64_t q = tix(); q < nvec; q += NTHR) {
    double acc[NV][VW];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[v][e] = 0.0;
    int j = rc;
    // streamed columns: a prefetched group overlaps the resident sweep below
    TA g[PF][VW];
    const int ng = (w - rc) < PF ? (w - rc) : PF;
#pragma unroll
    for (int u = 0; u < PF; ++u)
      if (u < ng) ld16_g<TA>(P.gl + (int64_t)(rc + u) * D.ld + q * VW, g[u]);
    // resident columns
    {
      const unsigned p = (unsigned)__cvta_generic_to_shared(P.sm + q * VW);
      const unsigned cst = (unsigned)(D.ld * sizeof(TA));
      int jj = 0;
      for (; jj + 4 <= rc; jj += 4) {
        TA a[4][VW];
#pragma unroll
        for (int u = 0; u < 4; ++u) ld16_sa<TA>(p + (unsigned)(jj + u) * cst, a[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double xv = xs[v][jj + u];
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[u][e], xv, acc[v][e]);
          }
      }
      for (; jj < rc; ++jj) {
        TA a[VW];
        ld16_sa<TA>(p + (unsigned)jj * cst, a);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xs[v][jj];
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[e], xv, acc[v][e]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < PF; ++u)
      if (u < ng) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xs[v][rc + u];
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)g[u][e], xv, acc[v][e]);
        }
      }
    j = rc + ng;
    // remaining streamed columns (large panels): unrolled by 8 for MLP
    const TA* pg = P.gl + q * VW;
    for (; j + 8 <= w; j += 8) {
      TA a[8][VW];
#pragma unroll
      for (int u = 0; u < 8; ++u) ld16_g<TA>(pg + (int64_t)(j + u) * D.ld, a[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xs[v][j + u];
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[u][e], xv, acc[v][e]);
        }
    }
    for (; j < w; ++j) {
      TA a[VW];
      ld16_g<TA>(pg + (int64_t)j * D.ld, a);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double xv = xs[v][j];
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[v][e] = fma((double)a[e], xv, acc[v][e]);
      }
    }
    if (P.oqv) {                                  // q == tix(): offsets precomputed
#pragma unroll
      for (int e = 0; e < VW; ++e)
        if (P.oq[e] >= 0) {
          double* o = out + P.oq[e];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            double* ov = o + (size_t)v * E.pvec;
            *ov = accumulate ? *ov + acc[v][e] : acc[v][e];
          }
        }
    } else {
      const int64_t i0 = q * VW;
      int64_t ow = i0 < D.d ? slice_owner(D.d, E.nb, i0) : 0;
      int64_t r0 = slice_r0(D.d, E.nb, ow), r1 = slice_r0(D.d, E.nb, ow + 1);
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        const int64_t i = i0 + e;
        if (i < D.d) {
          while (i >= r1) { ++ow; r0 = r1; r1 = slice_r0(D.d, E.nb, ow + 1); }
          double* o = out + ow * reg + (i - r0);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            double* ov = o + (size_t)v * E.pvec;
            *ov = accumulate ? *ov + acc[v][e] : acc[v][e];
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ panel GEMV^T
// outs[v][jl] = sum_i A[i, c0 + jl] * rs[v][i] for jl < w (A columns only;
// outs are owned local vectors).  rs are replicated d-vectors in global
// memory, read after the grid barrier.
//
// Short columns (ld/VW <= NTHR): thread q keeps row-vector q of r in
// registers, forms per-column partials for a chunk of 32 columns, and a
// warp transpose-reduction (31 shuffles / 32 columns) + a 16-way fixed-order
// cross-warp sum finish them.  Long columns: warp per (column, segment).
// Operands of the short-column GEMV^T that can be loaded ahead of time
// (before the decision that needs them is known): thread q's slice of r and
// the first streamed (non-resident) panel column.  Issuing these loads early
// overlaps their L2 latency with other work.
// Short-column GEMV^T thread map: a column is covered by wg = ceil(nvec / 32)
// warps; the CTA's warps form NWARP / wg column groups, each walking its own
// column chunks.  Returns this thread's row vector (-1: idle warp).
__device__ __forceinline__ int64_t gt_row(int64_t nvec) {
  const int wg = (int)((nvec + 31) >> 5);
  const int grp = wpx() / wg;
  if (grp >= NWARP / wg) return -1;
  return (int64_t)(wpx() - grp * wg) * 32 + lnx();
}

template <class TA, int NV>
struct GtPre {
  double rq[NV][VecOf<TA>::VW];
  TA g[VecOf<TA>::VW];
};

template <class TA, int NV>
__device__ __forceinline__ void gemv_t_prefetch(const DictV<TA>& D, const Panel<TA>& P,
                                                const double* const (&rs)[NV], GtPre<TA, NV>& pre) {
  constexpr int VW = VecOf<TA>::VW;
  const int64_t nvec = D.ld / VW;
  if (nvec > NTHR) return;                          // long columns stage r themselves
  const int64_t q = gt_row(nvec);
  const bool act = q >= 0 && q < nvec;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VW; ++e) pre.rq[v][e] = act ? ldcg(rs[v] + q * VW + e) : 0.0;
  if (act && P.rc < P.w) ld16_g<TA>(P.gl + (int64_t)P.rc * D.ld + q * VW, pre.g);
  else {
#pragma unroll
    for (int e = 0; e < VW; ++e) pre.g[e] = (TA)0;
  }
}

template <class TA, int NV>
__device__ void panel_gemv_t_pre(const Ctx& E, const DictV<TA>& D, const Panel<TA>& P,
                                 const GtPre<TA, NV>& pre, const double* const (&rs)[NV],
                                 double* const (&outs)[NV]);

template <class TA, int NV>
__device__ void panel_gemv_t(const Ctx& E, const DictV<TA>& D, const Panel<TA>& P,
                             const double* const (&rs)[NV], double* const (&outs)[NV]) {
  GtPre<TA, NV> pre;
  gemv_t_prefetch<TA, NV>(D, P, rs, pre);
  panel_gemv_t_pre<TA, NV>(E, D, P, pre, rs, outs);
}

template <class TA, int NV>
__device__ void panel_gemv_t_pre(const Ctx& E, const DictV<TA>& D, const Panel<TA>& P,
                                 const GtPre<TA, NV>& pre, const double* const (&rs)[NV],
                                 double* const (&outs)[NV]) {
  constexpr int VW = VecOf<TA>::VW;
  const int64_t nvec = D.ld / VW;
  const int w = P.w, rc = P.rc;
  double* red = shmem(E.sh);                        // [NWARP][CW] per v pass
  __syncthreads();
  if (nvec <= NTHR) {
    // column groups of wg warps (gt_row); per chunk of CW columns each warp
    // transpose-reduces its rows, then (wg > 1) the group's warps are summed
    // in warp order through shared memory — the same order, and so the same
    // bits, as one group spanning the whole CTA.
    const int wg = (int)((nvec + 31) >> 5);
    const int G = NWARP / wg;
    const int grp = wpx() / wg;
    const int64_t q = gt_row(nvec);
    const bool act = q >= 0 && q < nvec;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(P.sm + (act ? q : 0) * VW);
    const unsigned cst = (unsigned)(D.ld * sizeof(TA));
    constexpr int CW = 16;                          // columns per transpose-reduce chunk
    const int nchunk = (w + CW - 1) / CW;
    int cb = 0;                                     // staging buffer (double-buffered: one sync per round)
    for (int r0 = 0; r0 < nchunk; r0 += G) {
      const int j0 = (r0 + grp) * CW;
      const int cnt = (grp < G && j0 < w) ? ((w - j0) < CW ? (w - j0) : CW) : 0;
#pragma unroll
      for (int v = 0; v < NV; ++v, cb ^= 1) {
        double* rb = red + cb * (NWARP * CW);
        double p[CW];
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          TA a[VW];
          const int j = j0 + u;
          if (u < cnt && act) {
            if (j < rc) ld16_sa<TA>(sbase + (unsigned)j * cst, a);
            else if (j == rc) {
#pragma unroll
              for (int e = 0; e < VW; ++e) a[e] = pre.g[e];
            } else ld16_g<TA>(P.gl + (int64_t)j * D.ld + q * VW, a);
          } else {
#pragma unroll
            for (int e = 0; e < VW; ++e) a[e] = (TA)0;
          }
          double s = 0.0;
#pragma unroll
          for (int e = 0; e < VW; ++e) s = fma((double)a[e], pre.rq[v][e], s);
          p[u] = s;
        }
        // transpose-reduce: afterwards lane l (and l^16) holds the warp sum of column j0 + (l & 15)
#pragma unroll
        for (int o = CW / 2; o >= 1; o >>= 1) {
          const bool upper = (lnx() & o) != 0;
#pragma unroll
          for (int u = 0; u < o; ++u) {
            const double send = upper ? p[u] : p[u + o];
            const double keep = upper ? p[u + o] : p[u];
            p[u] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        p[0] += __shfl_xor_sync(0xffffffffu, p[0], 16);
        if (wg == 1) {
          if (lnx() < cnt) outs[v][j0 + lnx()] = p[0];
        } else {
          if (lnx() < CW) rb[wpx() * CW + lnx()] = p[0];
          __syncthreads();
          const int g2 = tix() / CW, c = tix() - (tix() / CW) * CW;
          if (g2 < G) {
            const int jj = (r0 + g2) * CW + c;
            if (jj < w && c < CW) {
              const double* t = rb + (g2 * wg) * CW + c;
              double s2 = t[0];
              for (int ww = 1; ww < wg; ++ww) s2 += t[ww * CW];
              outs[v][jj] = s2;
            }
          }
        }
      }
    }
    __syncthreads();
  } else {
    // Long columns: column groups of NWARP x CPW (a warp per CPW columns, lanes
    // over rows).  r is staged through shared memory in row chunks shared by
    // every warp of the group, double-buffered: the next chunk's loads are in
    // flight (registers) while the current one is consumed, one __syncthreads
    // per chunk.  The CPW columns of a warp are walked together, so each lane
    // keeps CPW independent 16-byte loads of A in flight.
    constexpr int CPW = sizeof(TA) == 8 ? 2 : 4;        // columns per warp
    constexpr int QU = sizeof(TA) == 8 ? 2 : ELL1_GT_QU32;  // row steps per lane in flight
    constexpr int SPT = 4;                              // staged doubles per thread per chunk
    int64_t rch = (int64_t)NTHR * SPT / (VW * NV);      // row vectors per chunk
    while (rch * VW * NV * 2 > E.shcap && rch > 32) rch /= 2;
    rch = rch / 32 * 32;
    double* const stg0 = shmem(E.sh);
    double* const stg1 = stg0 + rch * VW * NV;
    const int64_t nch = (nvec + rch - 1) / rch;
    const int64_t sdbl = rch * VW;                      // staged doubles per vector per chunk
    // staging: thread t moves doubles t, t + NTHR, ... of the chunk (all vectors)
#define ELL1_STAGE_LOAD(ch, buf)                                                     \
  do {                                                                              \
    const int64_t rb_ = (ch) * rch;                                                 \
    const int64_t cnt_ = min(rch, nvec - rb_) * VW;                                 \
    _Pragma("unroll") for (int u = 0; u < SPT; ++u) {                               \
      const int64_t t = tix() + (int64_t)u * NTHR;                                  \
      double val_ = 0.0;                                                            \
      _Pragma("unroll") for (int v = 0; v < NV; ++v) {                              \
        const int64_t o = t - (int64_t)v * sdbl;                                    \
        if (o >= 0 && o < cnt_) val_ = ldcg(rs[v] + rb_ * VW + o);                  \
      }                                                                             \
      buf[u] = val_;                                                                \
    }                                                                               \
  } while (0)
#define ELL1_STAGE_STORE(dst, buf)                                                   \
  do {                                                                              \
    _Pragma("unroll") for (int u = 0; u < SPT; ++u) {                               \
      const int64_t t = tix() + (int64_t)u * NTHR;                                  \
      if (t < NV * sdbl) (dst)[t] = buf[u];                                         \
    }                                                                               \
  } while (0)
    for (int jg = 0; jg < w; jg += NWARP * CPW) {
      double acc[CPW][NV];
#pragma unroll
      for (int c = 0; c < CPW; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[c][v] = 0.0;
      const TA* colp[CPW];
      bool resc[CPW], live[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int jl = jg + wpx() * CPW + c;
        live[c] = jl < w;
        resc[c] = jl < rc;
        colp[c] = (resc[c] ? P.sm : P.gl) + (int64_t)(live[c] ? jl : 0) * D.ld;
      }
      double buf[SPT];
      ELL1_STAGE_LOAD(0, buf);
      ELL1_STAGE_STORE(stg0, buf);
      __syncthreads();
      for (int64_t ch = 0; ch < nch; ++ch) {
        const bool more = ch + 1 < nch;
        if (more) ELL1_STAGE_LOAD(ch + 1, buf);          // in flight during the sweep
        const double* cur = (ch & 1) ? stg1 : stg0;
        const int64_t rb = ch * rch;
        const int64_t rcnt = min(rch, nvec - rb);
        for (int64_t q0 = lnx(); q0 < rcnt; q0 += 32 * QU) {
          TA a[QU][CPW][VW];
#pragma unroll
          for (int h = 0; h < QU; ++h) {
            const int64_t q = q0 + 32 * h;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
              if (live[c] && q < rcnt) {
                const TA* pa = colp[c] + (rb + q) * VW;
                if (resc[c]) ld16_s<TA>(pa, a[h][c]);
                else ld16_g<TA>(pa, a[h][c]);
              } else {
#pragma unroll
                for (int e = 0; e < VW; ++e) a[h][c][e] = (TA)0;
              }
            }
          }
#pragma unroll
          for (int h = 0; h < QU; ++h) {
            const int64_t q = q0 + 32 * h;
            if (q < rcnt) {
#pragma unroll
              for (int v = 0; v < NV; ++v) {
                const double2* rv = reinterpret_cast<const double2*>(cur + v * sdbl + q * VW);
#pragma unroll
                for (int e2 = 0; e2 < VW / 2; ++e2) {
                  const double2 t = rv[e2];
#pragma unroll
                  for (int c = 0; c < CPW; ++c) {
                    acc[c][v] = fma((double)a[h][c][2 * e2], t.x, acc[c][v]);
                    acc[c][v] = fma((double)a[h][c][2 * e2 + 1], t.y, acc[c][v]);
                  }
                }
              }
            }
          }
        }
        if (more) ELL1_STAGE_STORE(((ch + 1) & 1) ? stg1 : stg0, buf);
        __syncthreads();
      }
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int jl = jg + wpx() * CPW + c;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double s = warp_sum(acc[c][v]);
          if (jl < w && lnx() == 0) outs[v][jl] = s;
        }
      }
    }
#undef ELL1_STAGE_LOAD
#undef ELL1_STAGE_STORE
    __syncthreads();
  }
}

// ------------------------------------------------------------------ owned-column loop
// f(k) for every owned local column k in [0, W)
template <class F>
__device__ __forceinline__ void for_owned(const Ctx& E, F&& f) {
  for (int k = tix(); k < E.W; k += NTHR) f(k);
}

// shared-memory scratch (doubles) the engine needs next to the panel / owned vectors
__host__ __device__ inline int64_t engine_scratch_doubles(int kmax) {
  int64_t s = NWARP * 32;                   // GEMV^T / gather cross-warp staging
  if (s < NWARP * kmax + kmax) s = NWARP * kmax + kmax;
  if (s < 16 * 2) s = 32;
  return (s + 31) / 32 * 32;
}

}  // namespace ell1
