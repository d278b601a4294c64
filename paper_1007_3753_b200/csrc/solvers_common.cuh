// solvers_common.cuh — launch plumbing + scalar helpers shared by the solver kernels.
#pragma once
#include "engine.cuh"
#include <math.h>

namespace ell1 {

// Raw (type-erased) dictionary as the C ABI carries it.
struct DictRaw {
  const void* A;
  int dtype, ext;
  int64_t d, n, ld;
  double s;
};

// Grid-shared scratch common to every persistent solver.
struct GridBufs {
  double* part;               // nv slots of pvec doubles (slice-major partials)
  int64_t pvec;
  int rp;
  double* scal;               // [2][nb][SCAL]
  unsigned long long* bar;
  int* abort;
  int64_t shcap;              // shared-memory scratch doubles per CTA
  size_t panel_bytes;         // resident dictionary panel bytes (0: streamed)
};

template <class TA>
__device__ __forceinline__ DictV<TA> dict_view(const DictRaw& R) {
  DictV<TA> D;
  D.A = reinterpret_cast<const TA*>(R.A);
  D.d = R.d; D.n = R.n; D.ld = R.ld; D.ext = R.ext; D.s = R.s;
  return D;
}

// thread 0 only
__device__ __forceinline__ void ctx_bind(Ctx& E, const GridBufs& g, double* smem) {
  E.bar = g.bar; E.abort = g.abort; E.part = g.part; E.pvec = g.pvec; E.rp = g.rp;
  E.scal = g.scal; E.sh = smem; E.shcap = g.shcap;
}

// shrinkage.py:184-196 — t' = (1 + sqrt(4t^2 + 1)) / 2, nudged down by ulps
// until t'^2 - t' <= t^2 (the file is built with -fmad=false so this matches numpy).
__device__ __forceinline__ double fista_t_next(double t) {
  double tn = 0.5 * (1.0 + sqrt(4.0 * t * t + 1.0));
  while (tn * tn - tn > t * t) tn = nextafter(tn, 1.0);
  return tn;
}

// _fastkernels.pyx:14-27 (u > a -> u - a; u < -a -> u + a; else +0)
__device__ __forceinline__ double soft1(double u, double a) {
  return u > a ? u - a : (u < -a ? u + a : 0.0);
}

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// Python max(a, b) for floats (first argument wins ties / NaN in b).
__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }

// user stopping rule test (model.py:176-224) from reduced quantities
__device__ __forceinline__ bool stop_fires(int kind, double thr, int hist, double F, double F_prev,
                                           double dx2, double xp2, double gt2, double gtn, double kkt) {
  switch (kind) {
    case ELL1_STOP_REL_OBJECTIVE: return hist >= 2 && fabs(F - F_prev) <= thr * fabs(F_prev);
    case ELL1_STOP_REL_ESTIMATE: return hist >= 2 && sqrt(dx2) <= thr * sqrt(xp2);
    case ELL1_STOP_GROUND_TRUTH: return sqrt(gt2) <= thr * gtn;
    case ELL1_STOP_KKT: return kkt <= thr;
    default: return false;
  }
}

}  // namespace ell1

// ---------------------------------------------------------------- host side
#include <cstdio>
namespace ell1 {

inline int sm_count(int dev) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return v;
}

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Grid size: one CTA per SM at most, at least ~16 columns per CTA.
inline int pick_blocks(int64_t n, int requested) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = sm_count(dev);
  if (sms <= 0) sms = 148;
  int nb = requested > 0 ? requested : sms;
  if (nb > sms) nb = sms;
  int64_t by_cols = (n + 15) / 16;
  if (by_cols < 1) by_cols = 1;
  if (nb > by_cols) nb = (int)by_cols;
  return nb < 1 ? 1 : nb;
}

// Bump allocator over a caller workspace (256-byte aligned pieces).
struct Carve {
  char* base;
  size_t off, cap;
  bool ok;
  Carve(void* p, size_t c) : base((char*)p), off(0), cap(c), ok(true) {}
  template <class T>
  T* take(size_t count) {
    size_t bytes = align_up((int64_t)(count * sizeof(T)), 256);
    if (off + bytes > cap) { ok = false; return nullptr; }
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

// Grid scratch for nv partial d-vectors of a d-row operator over nb CTAs.
inline size_t grid_bytes(int nb, int64_t d, int nv) {
  const int64_t pvec = (int64_t)nb * nb * rpad(d, nb);
  return align_up((int64_t)(nv > 0 ? nv : 1) * pvec * 8, 256) + align_up((int64_t)2 * nb * SCAL * 8, 256) +
         512;
}

inline bool carve_grid(Carve& cv, GridBufs& g, int nb, int64_t d, int nv) {
  g.rp = rpad(d, nb);
  g.pvec = (int64_t)nb * nb * g.rp;
  g.part = cv.take<double>((size_t)(nv > 0 ? nv : 1) * g.pvec);
  g.scal = cv.take<double>((size_t)2 * nb * SCAL);
  g.bar = cv.take<unsigned long long>(4);
  g.abort = reinterpret_cast<int*>(g.bar + 2);
  return cv.ok;
}

// Cooperative launch with the requested dynamic shared memory.
template <class K, class Arg>
inline int coop_launch(K kernel, int nb, size_t smem, cudaStream_t s, Arg& arg, unsigned long long* bar) {
  if (cudaMemsetAsync(bar, 0, 4 * sizeof(unsigned long long), s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return ELL1_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NTHR, smem) != cudaSuccess) return ELL1_ERR_CUDA;
  int dev = 0;
  cudaGetDevice(&dev);
  if (per_sm < 1 || nb > per_sm * sm_count(dev)) return ELL1_ERR_NOCOOP;
  void* args[] = {(void*)&arg};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kernel, dim3(nb), dim3(NTHR), args, smem, s);
  if (e != cudaSuccess) {
    fprintf(stderr, "ell1_b200: cooperative launch failed: %s\n", cudaGetErrorString(e));
    return ELL1_ERR_CUDA;
  }
  return ELL1_OK;
}

// Shared-memory plan for a persistent solver:
//   [resident panel: rc columns][owned vectors: nov x wmax doubles][scratch]
struct SmemPlan {
  int rc;                // resident panel columns
  int wmax;              // owned-vector stride (max owned local columns over CTAs)
  size_t panel_bytes;
  size_t bytes;          // total dynamic smem
  int64_t scratch;       // scratch doubles
};

inline int max_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 48 * 1024;
  return v - 128;      // static __shared__ (grid_sync flag) + slack
}

inline SmemPlan plan_smem(const DictRaw& D, int nb, int nov, int kmax, bool allow_resident,
                          int64_t min_scratch = 0) {
  SmemPlan p;
  const int64_t wcols = (D.n + nb - 1) / nb;
  const int64_t wrows = D.ext ? (D.d + nb - 1) / nb : 0;
  p.wmax = (int)align_up(wcols + wrows, 2);
  p.scratch = engine_scratch_doubles(kmax);
  if (p.scratch < min_scratch) p.scratch = align_up(min_scratch, 32);
  const int64_t esz = D.dtype == ELL1_F64 ? 8 : 4;
  // long columns (GEMV^T row chunks of r staged in shared memory, NV <= 2)
  const int64_t vw = 16 / esz;
  if (D.ld / vw > NTHR) {
    int64_t want = 2 * 1024 * vw;
    if (want > 16384) want = 16384;
    if (p.scratch < want) p.scratch = want;
  }
  const int64_t fixed = ((int64_t)nov * p.wmax + p.scratch) * 8;
  const int64_t cap = max_smem_optin();
  int64_t rc = 0;
  if (allow_resident) {
    rc = (cap - fixed) / (D.ld * esz);
    if (rc < 0) rc = 0;
    if (rc > wcols) rc = wcols;
  }
  p.rc = (int)rc;
  p.panel_bytes = (size_t)align_up(rc * D.ld * esz, 16);
  p.bytes = p.panel_bytes + (size_t)fixed;
  return p;
}

inline DictRaw to_raw(const ell1_dict_t* D) {
  DictRaw r;
  r.A = D->A; r.dtype = D->dtype; r.ext = D->ext; r.d = D->d; r.n = D->n; r.ld = D->ld;
  r.s = D->ext_scale;
  return r;
}

inline bool dict_ok(const ell1_dict_t* D) {
  return D && D->A && D->d >= 1 && D->n >= 1 && D->ld >= D->d && D->ld % 32 == 0 &&
         (D->dtype == ELL1_F64 || D->dtype == ELL1_F32);
}

inline int64_t ncols_of(const ell1_dict_t* D) { return D->n + (D->ext ? D->d : 0); }

}  // namespace ell1
