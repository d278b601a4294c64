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
  int nb;                     // CTAs cooperating on the solve
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


// ---------------------------------------------------------------- groups
// A group launch runs `count` independent solves — each with its own Args
// (dictionary, b, controls, workspace, outputs) — on teams of `nb`
// consecutive CTAs of one persistent launch; team t takes solves t,
// t + nteams, ...  Run::run(a) is the solver body (the same code as the
// single-solve kernel), Run::reset(a, lane) prepares one solve's workspace
// (barrier counter, padding rows) with one warp.
template <class Args, class Run>
__global__ void __launch_bounds__(NTHR, 1) group_kernel(const Args* __restrict__ argv, int count, int nb) {
  __shared__ __align__(16) Args sa;
  const int team = (int)(blockIdx.x / (unsigned)nb);
  const int nteams = (int)(gridDim.x / (unsigned)nb);
  static_assert(sizeof(Args) % 4 == 0, "Args must be a whole number of words");
  for (int g = team; g < count; g += nteams) {
    __syncthreads();
    const unsigned* src = reinterpret_cast<const unsigned*>(argv + g);
    unsigned* dst = reinterpret_cast<unsigned*>(&sa);
    for (int i = (int)threadIdx.x; i < (int)(sizeof(Args) / 4); i += NTHR) dst[i] = src[i];
    __syncthreads();
    Run::run(sa);
  }
}

template <class Args, class Run>
__global__ void group_reset_kernel(const Args* __restrict__ argv, int count) {
  const int g = (int)(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32);
  if (g < count) Run::reset(argv[g], (int)(threadIdx.x & 31));
}

// zero the 4-word barrier block and the rows [d, ld) of k vectors (one warp)
__device__ __forceinline__ void reset_bar(unsigned long long* bar, int lane) {
  if (lane < 4) bar[lane] = 0ULL;
}
__device__ __forceinline__ void zero_pad_rows(double* v, int64_t d, int64_t ld, int lane) {
  for (int64_t i = d + lane; i < ld; i += 32) v[i] = 0.0;
}

}  // namespace ell1

// ---------------------------------------------------------------- host side
#include <cstdio>
#include <vector>
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
  g.nb = nb;
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


// Team size for a group launch: the fewest CTAs (<= 32, >= 16 columns each)
// whose shared memory holds the whole dictionary panel; 0 when even 32 do not.
inline int group_team_for(const DictRaw& D, int nov, int kmax, int64_t min_scratch = 0) {
  const int64_t wcols_1 = D.n;
  for (int nb = 1; nb <= 32; ++nb) {
    if (nb > 1 && (wcols_1 + nb - 1) / nb < 16) break;
    const SmemPlan p = plan_smem(D, nb, nov, kmax, true, min_scratch);
    if ((int64_t)p.rc >= (D.n + nb - 1) / nb) return nb;
  }
  return 0;
}

// Launch a group: copy the per-solve Args to the device (args_ws), reset
// each solve's workspace, then one persistent launch of teams of nb CTAs
// (cooperative when nb > 1, so every team's CTAs are co-resident).
template <class Args, class Run>
inline int group_launch(const std::vector<Args>& av, int nb, size_t smem, void* args_ws, size_t args_bytes,
                        cudaStream_t s) {
  const int count = (int)av.size();
  if (count == 0) return ELL1_OK;
  if (nb < 1) return ELL1_ERR_ARG;
  const size_t bytes = av.size() * sizeof(Args);
  if (!args_ws || args_bytes < bytes) return ELL1_ERR_ARG;
  if (cudaMemcpyAsync(args_ws, av.data(), bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) return ELL1_ERR_CUDA;
  const Args* dargs = reinterpret_cast<const Args*>(args_ws);
  group_reset_kernel<Args, Run><<<(count + 7) / 8, 256, 0, s>>>(dargs, count);
  if (cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
  auto kernel = group_kernel<Args, Run>;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return ELL1_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NTHR, smem) != cudaSuccess) return ELL1_ERR_CUDA;
  int dev = 0;
  cudaGetDevice(&dev);
  int teams = per_sm * sm_count(dev) / nb;
  if (teams < 1) return ELL1_ERR_NOCOOP;
  if (teams > count) teams = count;
  int cnt = count, team = nb;
  void* kargs[] = {(void*)&dargs, (void*)&cnt, (void*)&team};
  cudaError_t e = nb > 1 ? cudaLaunchCooperativeKernel((const void*)kernel, dim3(teams * nb), dim3(NTHR), kargs, smem, s)
                         : cudaLaunchKernel((const void*)kernel, dim3(teams * nb), dim3(NTHR), kargs, smem, s);
  if (e != cudaSuccess) {
    fprintf(stderr, "ell1_b200: group launch failed: %s\n", cudaGetErrorString(e));
    return ELL1_ERR_CUDA;
  }
  return ELL1_OK;
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

// Auto team size: group_team_for, or (dictionary too large for 32 CTAs'
// shared memory) the streamed single-solve grid capped at 32.
inline int group_team(const DictRaw& D, int nov, int kmax, int64_t min_scratch) {
  const int t = group_team_for(D, nov, kmax, min_scratch);
  return t > 0 ? t : pick_blocks(D.n, 32);
}

// Shared group driver: per-solve setup at the team size, then one launch
// per storage dtype present (a group normally holds one dtype).
template <class Args, template <class> class Run, class Setup>
inline int run_group(const ell1_group_t* G, int nov, int kmax, int64_t min_scratch, Setup setup, void* stream) {
  if (!G || G->count < 0 || (G->count > 0 && (!G->dicts || !G->io))) return ELL1_ERR_ARG;
  if (G->count == 0) return ELL1_OK;
  int nb = G->team;
  for (int i = 0; i < G->count; ++i)
    if (!dict_ok(&G->dicts[i])) return ELL1_ERR_ARG;
  if (nb <= 0) {
    nb = 1;
    for (int i = 0; i < G->count; ++i) {
      const int t = group_team(to_raw(&G->dicts[i]), nov, kmax, min_scratch);
      if (t > nb) nb = t;
    }
  }
  std::vector<Args> av64, av32;
  size_t smem64 = 0, smem32 = 0;
  for (int i = 0; i < G->count; ++i) {
    if (G->io[i].max_steps > 0) return ELL1_ERR_ARG;
    Args a;
    SmemPlan sp;
    const int rc = setup(i, nb, a, sp);
    if (rc != ELL1_OK) return rc;
    if (G->dicts[i].dtype == ELL1_F64) { av64.push_back(a); if (sp.bytes > smem64) smem64 = sp.bytes; }
    else { av32.push_back(a); if (sp.bytes > smem32) smem32 = sp.bytes; }
  }
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)G->args_ws;
  size_t wsb = G->args_ws_bytes;
  int rc = group_launch<Args, Run<double>>(av64, nb, smem64, ws, wsb, s);
  if (rc != ELL1_OK) return rc;
  const size_t used = align_up((int64_t)(av64.size() * sizeof(Args)), 256);
  if (av32.empty()) return ELL1_OK;
  if (wsb < used) return ELL1_ERR_ARG;
  return group_launch<Args, Run<float>>(av32, nb, smem32, ws + used, wsb - used, s);
}

}  // namespace ell1
