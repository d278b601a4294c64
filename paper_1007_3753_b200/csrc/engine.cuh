// engine.cuh — persistent-grid machinery shared by every single-instance solver.
//
// Execution model: one cooperative launch runs a whole solve.
// Each CTA owns
//   * a contiguous panel of dictionary columns  [c0, c1)   (n-side vectors x, y, g ...)
//   * a contiguous slice of rows                 [r0, r1)   (d-side reductions)
//   * for the [A, sI] extension, the identity columns n + [r0, r1).
// A matvec D v is computed as per-CTA partial d-vectors (panel GEMV) that are
// reduced slice-by-slice after a grid barrier; D^T r is local to each panel.
// Every scalar decision (backtracking accept, step sizes, stop rules) is
// computed redundantly and bit-identically by all CTAs from deterministic
// fixed-order reductions, so control flow needs no broadcast.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/ell1_b200.h"

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

// NaN-propagating max (np.max semantics)
__device__ __forceinline__ double nmax(double a, double b) {
  return (a > b || a != a) ? a : b;
}

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
  int64_t d, n, ld;   // ld == padded row count (dpad)
  int ext;
  double s;
  __device__ __forceinline__ int64_t ncols() const { return n + (ext ? d : 0); }
};

// ------------------------------------------------------------------ grid context
struct Ctx {
  int nb, b, tid, lane, warp;
  int64_t c0, c1;     // owned dictionary-column panel
  int64_t r0, r1;     // owned row slice
  unsigned long long* bar;
  int* abort;
  unsigned long long epoch;
  unsigned nbar;      // barriers passed (selects scalar double-buffer)
  double* part;       // [nb][pstride] d-vector partials
  int64_t pstride;
  double* scal;       // [2][nb][SCAL]
  double* sh;         // shared scratch
  int64_t shcap;      // its capacity in doubles
};

__device__ __forceinline__ void ctx_init(Ctx& E, int64_t d, int64_t n) {
  E.nb = gridDim.x;
  E.b = blockIdx.x;
  E.tid = threadIdx.x;
  E.lane = threadIdx.x & 31;
  E.warp = threadIdx.x >> 5;
  E.c0 = (n * E.b) / E.nb;
  E.c1 = (n * (E.b + 1)) / E.nb;
  E.r0 = (d * E.b) / E.nb;
  E.r1 = (d * (E.b + 1)) / E.nb;
  E.epoch = 0;
  E.nbar = 0;
}

// Software grid barrier (sense-free monotone counter).  Returns false when a
// peer CTA aborted or the wait timed out; callers then unwind cleanly.
__device__ bool grid_sync(Ctx& E) {
  __shared__ int s_ok;
  __syncthreads();
  E.epoch += (unsigned long long)E.nb;
  E.nbar++;
  if (E.tid == 0) {
    __threadfence();
    atomicAdd(E.bar, 1ULL);
    long long spins = 0;
    int ok = 1;
    while (ld_acquire(E.bar) < E.epoch) {
      if (((++spins) & 255) == 0) {
        if (*(volatile int*)E.abort) { ok = 0; break; }
        if (spins > SPIN_LIMIT) { atomicExch(E.abort, 1); ok = 0; break; }
        __nanosleep(64);
      }
    }
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// ------------------------------------------------------------------ block reductions
// K values reduced across the CTA in a fixed order; every thread gets the result.
template <int K>
__device__ __forceinline__ void block_reduce(const Ctx& E, double (&v)[K], unsigned maxmask) {
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = ((maxmask >> k) & 1u) ? warp_max(v[k]) : warp_sum(v[k]);
  double* sh = E.sh;
  if (E.lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[E.warp * K + k] = v[k];
  }
  __syncthreads();
  if (E.tid < K) {
    const int k = E.tid;
    const bool mx = (maxmask >> k) & 1u;
    double s = sh[k];
    for (int w = 1; w < NWARP; ++w) s = mx ? nmax(s, sh[w * K + k]) : s + sh[w * K + k];
    sh[NWARP * K + k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sh[NWARP * K + k];
  __syncthreads();
}

// Publish this CTA's K partial scalars into the buffer the next barrier selects.
template <int K>
__device__ __forceinline__ void publish(const Ctx& E, const double (&v)[K], int slot0 = 0) {
  if (E.tid < K) {
    double* dst = E.scal + ((size_t)((E.nbar + 1) & 1u) * E.nb + E.b) * SCAL + slot0;
    dst[E.tid] = v[E.tid];
  }
}

// After a barrier: reduce the K published scalars over all CTAs (fixed order,
// identical in every CTA).  maxmask bit k selects max instead of sum.
template <int K>
__device__ __forceinline__ void gather(const Ctx& E, double (&out)[K], unsigned maxmask, int slot0 = 0) {
  static_assert(K <= NWARP, "one warp per scalar");
  const double* src = E.scal + (size_t)(E.nbar & 1u) * E.nb * SCAL + slot0;
  double* sh = E.sh;
  if (E.warp < K) {
    const int k = E.warp;
    const bool mx = (maxmask >> k) & 1u;
    double s = mx ? -INFINITY : 0.0;
    for (int q = E.lane; q < E.nb; q += 32) {
      const double t = ldcg(src + (size_t)q * SCAL + k);
      s = mx ? nmax(s, t) : s + t;
    }
    s = mx ? warp_max(s) : warp_sum(s);
    if (E.lane == 0) sh[k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = sh[k];
  __syncthreads();
}

// ------------------------------------------------------------------ panel source
// Where a CTA reads its dictionary panel from: global memory (streamed through
// L2 with ld.global.nc) or a copy resident in shared memory for the whole
// launch (when the panel fits next to the scratch area).
template <class TA, bool SM>
struct Src {
  const TA* p;      // column c0 of the panel; column j at p + (j - c0) * ld
};

template <class TA>
struct VecOf { static constexpr int VW = 16 / (int)sizeof(TA); };

// 16-byte load of VW consecutive rows, widened to double
template <class TA, bool SM>
__device__ __forceinline__ void ld16(const TA* p, double (&a)[VecOf<TA>::VW]) {
  if constexpr (SM) {
    const unsigned addr = (unsigned)__cvta_generic_to_shared(p);
    if constexpr (sizeof(TA) == 8) {
      double x, y;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
      a[0] = x; a[1] = y;
    } else {
      float x, y, z, w;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(addr));
      a[0] = x; a[1] = y; a[2] = z; a[3] = w;
    }
  } else {
    if constexpr (sizeof(TA) == 8) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p));
      a[0] = t.x; a[1] = t.y;
    } else {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p));
      a[0] = t.x; a[1] = t.y; a[2] = t.z; a[3] = t.w;
    }
  }
}

// Copy this CTA's panel (columns [c0, c1), contiguous in the column-major
// layout) into shared memory.  Returns the smem source.
template <class TA>
__device__ Src<TA, true> load_panel(const Ctx& E, const DictV<TA>& D, TA* dst) {
  const int64_t cnt = (E.c1 - E.c0) * D.ld;              // multiple of 32 elements
  const int4* src = reinterpret_cast<const int4*>(D.A + E.c0 * D.ld);
  int4* d4 = reinterpret_cast<int4*>(dst);
  const int64_t n4 = cnt * (int64_t)sizeof(TA) / 16;
  for (int64_t k = E.tid; k < n4; k += NTHR) d4[k] = __ldg(src + k);
  __syncthreads();
  return Src<TA, true>{dst};
}

template <class TA>
__device__ __forceinline__ Src<TA, false> global_panel(const Ctx& E, const DictV<TA>& D) {
  return Src<TA, false>{D.A + E.c0 * D.ld};
}

// ------------------------------------------------------------------ panel GEMV
// part[b][v * ld + i] = sum_{j in panel} A[i, j] * xs[v][j]   (all rows, all v < NV)
template <class TA, bool SM, int NV>
__device__ void panel_gemv(const Ctx& E, const DictV<TA>& D, Src<TA, SM> S, const double* const (&xs)[NV]) {
  constexpr int VW = VecOf<TA>::VW;
  constexpr int U = SM ? 4 : 8;                    // columns per unrolled group (loads in flight)
  const int64_t w = E.c1 - E.c0;
  double* xsm = E.sh;                              // staged x panel: NV * w
  __syncthreads();
  for (int64_t k = E.tid; k < w; k += NTHR) {
#pragma unroll
    for (int v = 0; v < NV; ++v) xsm[v * w + k] = ldcg(xs[v] + E.c0 + k);
  }
  __syncthreads();
  const int64_t nvec = D.ld / VW;                  // row-vectors per column
  double* out = E.part + (size_t)E.b * E.pstride;
  for (int64_t q = E.tid; q < nvec; q += NTHR) {
    double acc[NV][VW];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[v][e] = 0.0;
    const TA* p = S.p + q * VW;
    int64_t j = 0;
    for (; j + U <= w; j += U) {
      double a[U][VW];
#pragma unroll
      for (int u = 0; u < U; ++u) ld16<TA, SM>(p + (j + u) * D.ld, a[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double xv = xsm[v * w + j + u];
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[v][e] = fma(a[u][e], xv, acc[v][e]);
        }
    }
    for (; j < w; ++j) {
      double a[VW];
      ld16<TA, SM>(p + j * D.ld, a);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double xv = xsm[v * w + j];
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[v][e] = fma(a[e], xv, acc[v][e]);
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VW; ++e) out[v * D.ld + q * VW + e] = acc[v][e];
  }
  __syncthreads();
}

// ------------------------------------------------------------------ panel GEMV^T
// outs[v][j] = sum_i A[i, j] * rs[v][i] for j in the panel (A-columns only).
// Work unit = (column, row segment); segments balance narrow panels over the
// 16 warps and are summed in a fixed order.  rs are replicated d-vectors
// written during this launch; they are read through L1 after the grid
// barrier's fence (which invalidates L1).
template <class TA, bool SM, int NV>
__device__ void panel_gemv_t(const Ctx& E, const DictV<TA>& D, Src<TA, SM> S,
                             const double* const (&rs)[NV], double* const (&outs)[NV]) {
  constexpr int VW = VecOf<TA>::VW;
  const int64_t w = E.c1 - E.c0;
  const int64_t nvec = D.ld / VW;
  int64_t seg = (2 * NWARP + w - 1) / (w > 0 ? w : 1);
  const int64_t maxseg = nvec / 32 > 0 ? nvec / 32 : 1;
  if (seg > maxseg) seg = maxseg;
  if (seg < 1) seg = 1;
  if (seg * w * NV > E.shcap) seg = 1;
  const int64_t seglen = (nvec + seg - 1) / seg;
  const int64_t units = w * seg;
  double* stage = E.sh;
  __syncthreads();
  for (int64_t u = E.warp; u < units; u += NWARP) {
    const int64_t jl = u / seg, sg = u - jl * seg;
    const TA* col = S.p + jl * D.ld;
    const int64_t q0 = sg * seglen;
    const int64_t q1 = min(nvec, q0 + seglen);
    double acc[NV][2];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v][0] = acc[v][1] = 0.0;
    int64_t q = q0 + E.lane;
    for (; q + 96 < q1; q += 128) {
      double a[4][VW];
#pragma unroll
      for (int k = 0; k < 4; ++k) ld16<TA, SM>(col + (q + 32 * k) * VW, a[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double* rv = rs[v] + (q + 32 * k) * VW;
#pragma unroll
          for (int e = 0; e < VW; ++e) acc[v][k & 1] = fma(a[k][e], rv[e], acc[v][k & 1]);
        }
    }
    for (; q < q1; q += 32) {
      double a[VW];
      ld16<TA, SM>(col + q * VW, a);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double* rv = rs[v] + q * VW;
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[v][0] = fma(a[e], rv[e], acc[v][0]);
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double s = warp_sum(acc[v][0] + acc[v][1]);
      if (E.lane == 0) {
        if (seg == 1) outs[v][E.c0 + jl] = s;
        else stage[(v * w + jl) * seg + sg] = s;
      }
    }
  }
  __syncthreads();
  if (seg > 1) {
    for (int64_t t = E.tid; t < w * NV; t += NTHR) {
      const int v = (int)(t / w);
      const int64_t jl = t - (int64_t)v * w;
      const double* st = stage + (v * w + jl) * seg;
      double s = st[0];
      for (int64_t k = 1; k < seg; ++k) s += st[k];
#pragma unroll
      for (int vv = 0; vv < NV; ++vv)
        if (vv == v) outs[vv][E.c0 + jl] = s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ slice reduction
// After the barrier that follows panel_gemv: for each owned row i,
//   sums[v] = sum over CTAs of part[c][v * ld + i]   (fixed order)
// then f(i, sums) runs once per row (thread-parallel over rows).
template <int NV, class F>
__device__ void slice_reduce(const Ctx& E, int64_t ld, F&& f) {
  int64_t CH = E.shcap / NV;                        // rows per chunk (NV*CH doubles of smem)
  if (CH > 256) CH = 256;
  double* stage = E.sh;
  for (int64_t base = E.r0; base < E.r1; base += CH) {
    const int rows = (int)min(CH, E.r1 - base);
    const int items = rows * NV;
    for (int it = E.warp; it < items; it += NWARP) {
      const int v = it / rows, rr = it - v * rows;
      const double* src = E.part + (size_t)v * ld + base + rr;
      double s = 0.0;
      for (int c = E.lane; c < E.nb; c += 32) s += ldcg(src + (size_t)c * E.pstride);
      s = warp_sum(s);
      if (E.lane == 0) stage[it] = s;
    }
    __syncthreads();
    for (int rr = E.tid; rr < rows; rr += NTHR) {
      double sums[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) sums[v] = stage[v * rows + rr];
      f(base + rr, sums);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ owned-column loop
// f(j) for every owned column of D: the A panel and (extension) the identity
// columns n + [r0, r1).
template <class TA, class F>
__device__ __forceinline__ void for_owned(const Ctx& E, const DictV<TA>& D, F&& f) {
  for (int64_t j = E.c0 + E.tid; j < E.c1; j += NTHR) f(j);
  if (D.ext)
    for (int64_t i = E.r0 + E.tid; i < E.r1; i += NTHR) f(D.n + i);
}

// shared-memory scratch (doubles) the engine needs next to an optional panel
__host__ __device__ inline int64_t engine_scratch_doubles(int64_t n, int nb, int nv, int kmax) {
  const int64_t w = (n + nb - 1) / nb + 1;
  int64_t s = w * nv * 2;                   // x staging / GEMV^T segment partials (>= 2 segs)
  if (s < 64 * nv) s = 64 * nv;             // slice staging
  if (s < NWARP * kmax + kmax) s = NWARP * kmax + kmax;   // block reductions of kmax scalars
  return (s + 31) / 32 * 32;
}

}  // namespace ell1
