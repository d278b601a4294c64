// batch_homotopy.cu — LASSO paths (homotopy.solve_path, homotopy.py:128-244)
// for B right-hand sides sharing one dictionary (BASELINE config 5,
// "batched Homotopy").  Element j equals homotopy_solve on (A, b_j).
//
// One host round = one breakpoint of every active instance:
//   hb_dir   (CTA per instance)  finalise the previous breakpoint from the
//            fresh correlations c = A^T r (lambda repair, trace, stop), then
//            d_I = (A_I^T A_I)^{-1} sgn(c_I) from the instance's upper factor
//            (blocked triangular solves) and v = A_I d_I
//   GEMM     W = A^T V                      (all active instances, cuBLAS DGEMM)
//   hb_step  (CTA per instance)  drift check ||w_I - sgn|| (dense / ridge
//            refactorisation on failure, homotopy.py:53-64,118-125), the step
//            lengths gamma+/gamma- (homotopy.py:78-105), the add / remove event
//            with chol_append / chol_delete, and r = b - A_I x_I
//   GEMM     C = A^T R
// Finished instances are compacted out of the GEMM operands every round.
// fp32 dictionaries are widened once to fp64 (the path's breakpoint tests
// are exact comparisons; every product runs in fp64).
#include <algorithm>
#include <cstdlib>
#include <vector>
#include "batched.cuh"
#include "factor.cuh"

#define T0 if (threadIdx.x == 0)

// resident threads per SM the direction / step kernels are compiled for (register cap 65536 / HB_TPSM)
#ifndef HB_TPSM
#define HB_TPSM 1024
#endif

namespace ell1 {

// Threads per instance CTA (NT, picked per round by hb_threads).  Measured at config 5 (B=256): 512 beats 128 —
// the row / column sweeps of an instance dominate its dependent chains, and
// two 512-thread CTAs per SM already hold every instance of a 296-wide wave.

// fixed-order CTA reduction of K values (sum / max by mask); all threads get them
template <int K, int NT>
__device__ __forceinline__ void hb_reduce(double (&v)[K], unsigned maxmask, double* sh) {
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = ((maxmask >> k) & 1u) ? warp_max(v[k]) : warp_sum(v[k]);
  if (lnx() == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[wpx() * K + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool mx = (maxmask >> k) & 1u;
    double s = sh[k];
    for (int w = 1; w < (NT / 32); ++w) s = mx ? nmax(s, sh[w * K + k]) : s + sh[w * K + k];
    v[k] = s;
  }
  __syncthreads();
}

struct HI {                 // per-instance state (instance-indexed)
  double lam, lam0, floor, gamma, rr, l1, top, cnt;
  int it, m, status, conv, note, done, ridge, pend, redo, finish;
};

struct HB {
  const double* A;          // fp64, column-major ld x n
  int64_t d, n, ld;
  const double* Bm;         // ld x B (instance-indexed right-hand sides)
  int mmax;
  double target;
  int max_iter;
  HI* st;
  double* X;                // [B][n]
  double* Cin;              // [B][n] correlations of the current iterate
  double* R;                // [B][mmax * mmax] upper factor (row-major)
  int* sup;                 // [B][mmax]
  int* posof;               // [B][n]  support position or -1
  double* dI;               // [B][mmax]
  const int* act;           // slot -> instance
  double* V;                // ld x nact (slot-indexed)   v = A_I d_I
  double* W;                // n x nact                   A^T v
  double* Rr;               // ld x nact                  r = b - A_I x_I
  double* C;                // n x nact                   A^T r
  double* trace;            // [B][max_iter][4] or null
  double* lam_out;          // [B] or null
};

constexpr int HB_SMEM_FIXED = 32 * 32;    // triangular-solve tile

__device__ __forceinline__ void argmin_pair(double& v, int& i, double v2, int i2) {
  if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// CTA argmin of (value, index): smallest value, lowest index among ties
template <int NT>
__device__ void cta_argmin(double& v, int& i, double* shv, int* shi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmin_pair(v, i, v2, i2);
  }
  if (lnx() == 0) { shv[wpx()] = v; shi[wpx()] = i; }
  __syncthreads();
  v = shv[0]; i = shi[0];
  for (int w = 1; w < (NT / 32); ++w) argmin_pair(v, i, shv[w], shi[w]);
  __syncthreads();
}

// Dense upper Cholesky of A_I^T A_I (+ shift I) with the Gram rows formed on
// the fly (row k: one warp per column, lanes over the d rows): no m x m
// scratch.  numpy.linalg.cholesky semantics; false when not PD.
template <int NT>
__device__ bool gram_chol(const HB& a, const int* sup, int m, double shift, double* R, int ldr,
                          double* row, double* sc) {
  for (int k = 0; k < m; ++k) {
    const double* ak = a.A + (int64_t)sup[k] * a.ld;
    for (int j = k + wpx(); j < m; j += (NT / 32)) {
      const double* aj = a.A + (int64_t)sup[j] * a.ld;
      double acc = 0.0;
      for (int64_t i = lnx(); i < a.d; i += 32) acc = fma(ak[i], aj[i], acc);
      acc = warp_sum(acc);
      if (lnx() == 0) row[j] = acc + (j == k ? shift : 0.0);
    }
    __syncthreads();
    if (tix() == 0) {
      double s = row[k];
      for (int i = 0; i < k; ++i) s -= R[(size_t)i * ldr + k] * R[(size_t)i * ldr + k];
      sc[0] = s;
    }
    __syncthreads();
    if (!(sc[0] > 0.0)) return false;
    const double rkk = sqrt(sc[0]);
    for (int j = k + tix(); j < m; j += NT) {
      if (j == k) { R[(size_t)k * ldr + k] = rkk; continue; }
      double s = row[j];
      for (int i = 0; i < k; ++i) s -= R[(size_t)i * ldr + k] * R[(size_t)i * ldr + j];
      R[(size_t)k * ldr + j] = s / rkk;
    }
    __syncthreads();
  }
  return true;
}

// ridge factor (homotopy.py:118-125): G + 1e-12 max(tr G, 1) I
template <int NT>
__device__ bool ridge_chol(const HB& a, const int* sup, int m, double* R, int ldr, double* row, double* sc) {
  double tr[1] = {0.0};
  for (int p = wpx(); p < m; p += (NT / 32)) {
    const double* ap = a.A + (int64_t)sup[p] * a.ld;
    double acc = 0.0;
    for (int64_t i = lnx(); i < a.d; i += 32) acc = fma(ap[i], ap[i], acc);
    acc = warp_sum(acc);
    if (lnx() == 0) row[p] = acc;
  }
  __syncthreads();
  T0 {
    double t = 0.0;
    for (int p = 0; p < m; ++p) t += row[p];
    sc[3] = 1e-12 * pymax(t, 1.0);
  }
  __syncthreads();
  (void)tr;
  return gram_chol<NT>(a, sup, m, sc[3], R, ldr, row, sc);
}

// sum_p A[sup[p], i] * w[p] in support order (same rounding as the plain
// loop), 16 column loads in flight per thread
__device__ __forceinline__ double sup_dot(const double* A, int64_t ld, const int* sup, int m, int64_t i,
                                          const double* w) {
  double acc = 0.0;
  int p = 0;
  for (; p + 16 <= m; p += 16) {
    double av[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) av[u] = A[(int64_t)sup[p + u] * ld + i];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = fma(av[u], w[p + u], acc);
  }
  for (; p < m; ++p) acc = fma(A[(int64_t)sup[p] * ld + i], w[p], acc);
  return acc;
}

// ---- setup: lambda0, first atom (homotopy.py:142-177); C holds A^T b (slot = instance)
template <int NT>
__global__ void __launch_bounds__(NT) hb_init(HB a, int B) {
  const int j = blockIdx.x;
  if (j >= B) return;
  __shared__ double sh[(NT / 32) * 4 + 8];
  __shared__ double shv[(NT / 32)];
  __shared__ int shi[(NT / 32)];
  HI& S = a.st[j];
  const double* c = a.C + (int64_t)j * a.n;
  double* X = a.X + (int64_t)j * a.n;
  double* Ci = a.Cin + (int64_t)j * a.n;
  int* pos = a.posof + (int64_t)j * a.n;
  const double* b = a.Bm + (int64_t)j * a.ld;
  double v[2] = {0.0, 0.0};
  for (int64_t k = tix(); k < a.n; k += NT) {
    const double ck = c[k];
    Ci[k] = ck; X[k] = 0.0; pos[k] = -1;
    v[0] = nmax(v[0], fabs(ck));
  }
  for (int64_t i = tix(); i < a.d; i += NT) v[1] += b[i] * b[i];
  hb_reduce<2, NT>(v, 1u, sh);
  const double lam0 = v[0];
  double bv = INFINITY;
  int bi = 0x7fffffff;
  for (int64_t k = tix(); k < a.n; k += NT)
    if (fabs(c[k]) == lam0) argmin_pair(bv, bi, 0.0, (int)k);
  cta_argmin<NT>(bv, bi, shv, shi);
  const double bn = sqrt(v[1]);
  if (lam0 <= a.target || lam0 == 0.0) {                 // homotopy.py:161-166
    T0 {
      const double lamr = pymax(lam0, a.target);
      if (a.trace) {
        double* tr = a.trace + (size_t)j * (a.max_iter > 0 ? a.max_iter : 1) * 4;
        tr[0] = 0.0; tr[1] = 0.5 * bn * bn; tr[2] = bn; tr[3] = 0.0;
      }
      S.lam = lamr; S.lam0 = lam0; S.it = 0; S.m = 0; S.status = ELL1_ZERO_DATA; S.conv = 1; S.done = 1;
      S.note = 0; S.pend = 0; S.redo = 0; S.ridge = 0; S.finish = 0;
    }
    return;
  }
  // first atom: R = [||a_j0||]
  const double* col = a.A + (int64_t)bi * a.ld;
  double q[1] = {0.0};
  for (int64_t i = tix(); i < a.d; i += NT) q[0] += col[i] * col[i];
  hb_reduce<1, NT>(q, 0u, sh);
  T0 {
    S.lam = lam0; S.lam0 = lam0; S.floor = pymax(a.target, 1e-12 * lam0);
    S.it = 0; S.m = 1; S.conv = 0; S.done = 0; S.note = 0; S.pend = 0; S.redo = 0; S.ridge = 0;
    S.finish = 0;
    S.status = q[0] > 0.0 ? ELL1_OK : ELL1_NOT_PD;
    if (!(q[0] > 0.0)) S.done = 1;
    a.R[(size_t)j * a.mmax * a.mmax] = sqrt(q[0]);
    a.sup[(size_t)j * a.mmax] = bi;
    pos[bi] = 0;
  }
}

// ---- finalise the previous breakpoint, then the direction of the next one
template <int NT>
__global__ void __launch_bounds__(NT, HB_TPSM / NT) hb_dir(HB a, int nact) {
  const int s = blockIdx.x;
  if (s >= nact) return;
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sh[(NT / 32) * 4 + 8];
  __shared__ int flag;
  const int j = a.act[s];
  HI& S = a.st[j];
  const int ldr = a.mmax;
  double* tile = dsm;                          // 32 x 32
  double* zs = dsm + HB_SMEM_FIXED;            // mmax
  double* Vs = a.V + (int64_t)s * a.ld;
  double* Ci = a.Cin + (int64_t)j * a.n;
  if (S.pend) {
    // fresh correlations (homotopy.py:224-234)
    const double* c = a.C + (int64_t)s * a.n;
    double v[1] = {0.0};
    for (int64_t k = tix(); k < a.n; k += NT) {
      const double ck = c[k];
      Ci[k] = ck;
      v[0] = nmax(v[0], fabs(ck));
    }
    hb_reduce<1, NT>(v, 1u, sh);
    T0 {
      double lam;
      if (S.finish) lam = a.target;
      else {
        const double lam_step = S.lam - S.gamma;
        const double lam_emp = v[0];
        if (fabs(lam_emp - lam_step) <= 1e-9 * pymax(lam_step, 1e-30) || S.m == 0) lam = lam_step;
        else lam = lam_emp;
      }
      S.lam = lam;
      const double rn = sqrt(S.rr);
      if (a.trace) {
        double* tr = a.trace + ((size_t)j * (a.max_iter > 0 ? a.max_iter : 1) + (S.it - 1)) * 4;
        tr[0] = (double)S.it; tr[1] = 0.5 * rn * rn + lam * S.l1; tr[2] = rn; tr[3] = S.cnt;
      }
      if (S.finish || lam <= S.floor) { S.conv = 1; S.done = 1; }
      S.pend = 0;
    }
    __syncthreads();
  }
  T0 {
    flag = 0;
    if (!S.done && !S.redo && S.it >= a.max_iter) S.done = 1;       // budget exhausted
    if (S.done) flag = 1;
    else if (S.redo) S.redo = 0;                                    // retry of the same breakpoint
    else { S.it++; S.ridge = 0; }
  }
  __syncthreads();
  if (flag) {
    for (int64_t i = tix(); i < a.ld; i += NT) Vs[i] = 0.0;
    return;
  }
  const int m = S.m;
  const int* sup = a.sup + (size_t)j * a.mmax;
  const double* R = a.R + (size_t)j * a.mmax * a.mmax;
  double* dI = a.dI + (size_t)j * a.mmax;
  for (int p = tix(); p < m; p += NT) zs[p] = sgn(Ci[sup[p]]);
  __syncthreads();
  trsv_RT<NT>(R, ldr, m, zs, tile);
  trsv_R<NT>(R, ldr, m, zs, tile);
  for (int p = tix(); p < m; p += NT) dI[p] = zs[p];
  // v = A_I d_I (rows over threads, support columns in order)
  for (int64_t i = tix(); i < a.ld; i += NT) {
    double acc = 0.0;
    if (i < a.d)
      acc = sup_dot(a.A, a.ld, sup, m, i, zs);
    Vs[i] = acc;
  }
}

// ---- drift check, step lengths, event, factor update, residual
template <int NT>
__global__ void __launch_bounds__(NT, HB_TPSM / NT) hb_step(HB a, int nact) {
  const int s = blockIdx.x;
  if (s >= nact) return;
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sh[(NT / 32) * 8 + 16];
  __shared__ double shv[(NT / 32)];
  __shared__ int shi[(NT / 32)];
  __shared__ double sc[4];
  __shared__ int dec[4];               // 0: refactor, 1: event(0 add / 1 remove / 2 finish), 2: ip, 3: im
  const int j = a.act[s];
  HI& S = a.st[j];
  const int ldr = a.mmax;
  double* tile = dsm;
  double* zs = dsm + HB_SMEM_FIXED;            // mmax
  double* row = zs + a.mmax;                   // mmax (Gram rows / x_I)
  double* Rs = a.Rr + (int64_t)s * a.ld;
  const double* w = a.W + (int64_t)s * a.n;
  double* X = a.X + (int64_t)j * a.n;
  const double* Ci = a.Cin + (int64_t)j * a.n;
  int* pos = a.posof + (int64_t)j * a.n;
  int* sup = a.sup + (size_t)j * a.mmax;
  double* R = a.R + (size_t)j * a.mmax * a.mmax;
  const double* dI = a.dI + (size_t)j * a.mmax;
  const double* b = a.Bm + (int64_t)j * a.ld;
  if (S.done) {
    for (int64_t i = tix(); i < a.ld; i += NT) Rs[i] = 0.0;
    return;
  }
  const int m = S.m;
  const double lam = S.lam;
  // drift ||w_I - sgn||, ||sgn|| (homotopy.py:48-52; w_I == A_I^T v)
  {
    double q[2] = {0.0, 0.0};
    for (int p = tix(); p < m; p += NT) {
      const double sg = sgn(Ci[sup[p]]);
      const double e = w[sup[p]] - sg;
      q[0] += e * e;
      q[1] += sg * sg;
    }
    hb_reduce<2, NT>(q, 0u, sh);
    T0 {
      const double tol = 1e-6 * pymax(1.0, sqrt(q[1]));
      dec[0] = (!(sqrt(q[0]) <= tol) && S.ridge != 2) ? 1 : 0;
    }
    __syncthreads();
  }
  if (dec[0]) {
    // dense refactorisation; a second failure (or a singular Gram) -> ridge
    bool ok = false;
    if (S.ridge == 0) ok = gram_chol<NT>(a, sup, m, 0.0, R, ldr, row, sc);
    if (ok) {
      T0 S.ridge = 1;
    } else {
      const bool ok2 = ridge_chol<NT>(a, sup, m, R, ldr, row, sc);
      T0 {
        S.ridge = 2; S.note = 1;
        if (!ok2) { S.status = ELL1_NOT_PD; S.done = 1; }
      }
    }
    T0 S.redo = 1;
    for (int64_t i = tix(); i < a.ld; i += NT) Rs[i] = 0.0;
    return;
  }
  // step lengths (homotopy.py:78-105): gamma+ over the inactive set, gamma- over the support
  {
    const double floor = 1e-10 * pymax(lam, 1e-30);
    double v1 = INFINITY, v2 = INFINITY, vm = INFINITY;
    int i1 = 0x7fffffff, i2 = 0x7fffffff, im = 0x7fffffff;
    for (int64_t k = tix(); k < a.n; k += NT) {
      const int p = pos[k];
      const double wk = w[k];
      if (p >= 0) {
        const double r = -X[k] / dI[p];
        if (isfinite(r) && r > 0.0) argmin_pair(vm, im, r, (int)k);
      } else {
        const double ck = Ci[k];
        const double r1 = (lam - ck) / (1.0 - wk);
        const double r2 = (lam + ck) / (1.0 + wk);
        if (isfinite(r1) && r1 > floor) argmin_pair(v1, i1, r1, (int)k);
        if (isfinite(r2) && r2 > floor) argmin_pair(v2, i2, r2, (int)k);
      }
    }
    cta_argmin<NT>(v1, i1, shv, shi);
    cta_argmin<NT>(v2, i2, shv, shi);
    cta_argmin<NT>(vm, im, shv, shi);
    T0 {
      double gp = v1;
      int ip = isfinite(v1) ? i1 : -1;
      if (v2 < gp) { gp = v2; ip = i2; }
      const double gm = vm;
      const int imm = isfinite(gm) ? im : -1;
      const double ge = fmin(gp, gm);
      const double cap = lam - a.target;
      if (cap <= ge) { dec[1] = 2; sc[0] = cap; }
      else {
        const bool remove = gm <= gp + 1e-12;
        dec[1] = remove ? 1 : 0;
        sc[0] = remove ? gm : gp;
      }
      dec[2] = ip; dec[3] = imm;
      S.gamma = sc[0];
      S.finish = dec[1] == 2;
    }
    __syncthreads();
  }
  const double gamma = sc[0];
  const int ev = dec[1];
  for (int p = tix(); p < m; p += NT) X[sup[p]] = X[sup[p]] + gamma * dI[p];
  __syncthreads();
  int mn = m;
  if (ev == 1) {
    // remove im: chol_delete(pos) (numerics.py:140-158)
    const int im = dec[3];
    const int p0 = pos[im];
    T0 X[im] = 0.0;
    // rows above: shift columns > p0 left — a warp per row, each 32-column
    // chunk read before any lane writes (row-local, so rows run in parallel)
    for (int i = wpx(); i < p0; i += (NT / 32)) {
      double* Ri = R + (size_t)i * ldr;
      for (int j0 = p0 + 1; j0 < m; j0 += 32) {
        const int jj = j0 + lnx();
        const double v = jj < m ? Ri[jj] : 0.0;
        __syncwarp();
        if (jj < m) Ri[jj - 1] = v;
        __syncwarp();
      }
    }
    __syncthreads();
    if (p0 < m - 1) {
      const int mt = m - p0 - 1;
      for (int jj = tix(); jj < mt; jj += NT) zs[jj] = R[(size_t)p0 * ldr + p0 + 1 + jj];
      __syncthreads();
      chol_update_shift<NT>(R, ldr, p0 + 1, p0, mt, zs, sc);
    }
    T0 {
      for (int p = p0; p < m - 1; ++p) { const int c = sup[p + 1]; sup[p] = c; pos[c] = p; }
      pos[im] = -1;
    }
    mn = m - 1;
  } else if (ev == 0) {
    // add ip: chol_append (numerics.py:115-137); NotPD -> ridge over the grown support
    const int ip = dec[2];
    const double* acol = a.A + (int64_t)ip * a.ld;
    for (int p = wpx(); p < m; p += (NT / 32)) {
      const double* ap = a.A + (int64_t)sup[p] * a.ld;
      double acc = 0.0;
      for (int64_t i = lnx(); i < a.d; i += 32) acc = fma(ap[i], acol[i], acc);
      acc = warp_sum(acc);
      if (lnx() == 0) zs[p] = acc;
    }
    double q[1] = {0.0};
    for (int64_t i = tix(); i < a.d; i += NT) q[0] += acol[i] * acol[i];
    hb_reduce<1, NT>(q, 0u, sh);
    trsv_RT<NT>(R, ldr, m, zs, tile);
    double uu[1] = {0.0};
    for (int p = tix(); p < m; p += NT) uu[0] += zs[p] * zs[p];
    hb_reduce<1, NT>(uu, 0u, sh);
    const double d2 = q[0] - uu[0];
    const bool fits = m < ldr;
    if (d2 > 0.0 && fits) {
      for (int p = tix(); p < m; p += NT) R[(size_t)p * ldr + m] = zs[p];
      T0 {
        R[(size_t)m * ldr + m] = sqrt(d2);
        sup[m] = ip; pos[ip] = m;
      }
      __syncthreads();
    } else if (!fits) {
      T0 { S.status = ELL1_DEGENERATE; S.done = 1; }
      __syncthreads();
    } else {
      T0 { sup[m] = ip; pos[ip] = m; }
      __syncthreads();
      const bool ok2 = ridge_chol<NT>(a, sup, m + 1, R, ldr, row, sc);
      T0 { S.note = 1; if (!ok2) { S.status = ELL1_NOT_PD; S.done = 1; } }
    }
    if (fits) mn = m + 1;
  }
  __syncthreads();
  T0 S.m = mn;
  // r = b - A_I x_I, ||r||^2, ||x||_1, max|x|, support count (homotopy.py:224-226)
  for (int p = tix(); p < mn; p += NT) row[p] = X[sup[p]];
  __syncthreads();
  double q3[3] = {0.0, 0.0, 0.0};
  for (int64_t i = tix(); i < a.ld; i += NT) {
    double r = 0.0;
    if (i < a.d) {
      double acc = 0.0;
      acc = sup_dot(a.A, a.ld, sup, mn, i, row);
      r = b[i] - acc;
      q3[0] += r * r;
    }
    Rs[i] = r;
  }
  for (int64_t k = tix(); k < a.n; k += NT) { const double xk = fabs(X[k]); q3[1] += xk; q3[2] = nmax(q3[2], xk); }
  hb_reduce<3, NT>(q3, 0x4u, sh);
  const double cut = 1e-10 * pymax(q3[2], 1.0);
  double c1[1] = {0.0};
  for (int64_t k = tix(); k < a.n; k += NT) if (fabs(X[k]) > cut) c1[0] += 1.0;
  hb_reduce<1, NT>(c1, 0u, sh);
  T0 { S.rr = q3[0]; S.l1 = q3[1]; S.top = q3[2]; S.cnt = c1[0]; S.pend = 1; }
}

__global__ void hb_scan(const HI* st, const int* act, int nact, int* perm, int* newn) {
  __shared__ int base;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nact; c0 += blockDim.x) {
    const int s = c0 + threadIdx.x;
    const int live = (s < nact) ? !st[act[s]].done : 0;
    const unsigned msk = __ballot_sync(0xffffffffu, live);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) wsum[w] = __popc(msk);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = base;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { const int t = wsum[k]; wsum[k] = acc; acc += t; }
      base = acc;
    }
    __syncthreads();
    if (live) perm[wsum[w] + __popc(msk & ((1u << l) - 1))] = s;
    __syncthreads();
  }
  if (threadIdx.x == 0) *newn = base;
}

__global__ void hb_permute(const int* act, const int* perm, int nn, int* act2, const double* V, double* V2,
                           int64_t ld) {
  const int k = blockIdx.y;
  if (k >= nn) return;
  const int s = perm[k];
  if (blockIdx.x == 0 && threadIdx.x == 0) act2[k] = act[s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += (int64_t)gridDim.x * blockDim.x)
    V2[(int64_t)k * ld + i] = V[(int64_t)s * ld + i];
}

__global__ void hb_out(HB a, int B, double* x, int32_t* its, int32_t* conv, int32_t* status, int32_t* notes) {
  const int j = blockIdx.x;
  if (j >= B) return;
  const HI& S = a.st[j];
  for (int64_t k = threadIdx.x; k < a.n; k += blockDim.x) x[(int64_t)j * a.n + k] = a.X[(int64_t)j * a.n + k];
  if (threadIdx.x == 0) {
    its[j] = S.it;
    conv[j] = S.conv;
    status[j] = S.status;
    if (notes) notes[j] = S.note;
    if (a.lam_out) a.lam_out[j] = S.lam;
  }
}

__global__ void widen_kernel(const float* src, double* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

template <int NT>
bool hb_smem_attr(size_t smem) {
  return cudaFuncSetAttribute(hb_dir<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
         cudaFuncSetAttribute(hb_step<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
}

// threads per instance for a round of nact instances
int hb_threads(int nact) {
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("ELL1_HB_NT");                  // diagnostics: 128 / 256 / 512
    force = e ? atoi(e) : 0;
  }
  if (force == 128 || force == 256 || force == 512) return force;
  // few instances: wide CTAs shorten each instance's sweeps; many: narrow CTAs
  // keep more instances resident so their dependent chains overlap
  // (tools/hb_nt_ab.py: B=256 512 > 256 > 128; B=4096 128 > 256 > 512)
  return nact > 2048 ? 128 : nact > 512 ? 256 : 512;
}

void hb_launch(int which, int nt, int nact, size_t smem, cudaStream_t s, const HB& a) {
  if (nt == 128) {
    if (which == 0) hb_dir<128><<<nact, 128, smem, s>>>(a, nact);
    else hb_step<128><<<nact, 128, smem, s>>>(a, nact);
  } else if (nt == 256) {
    if (which == 0) hb_dir<256><<<nact, 256, smem, s>>>(a, nact);
    else hb_step<256><<<nact, 256, smem, s>>>(a, nact);
  } else {
    if (which == 0) hb_dir<512><<<nact, 512, smem, s>>>(a, nact);
    else hb_step<512><<<nact, 512, smem, s>>>(a, nact);
  }
}

inline bool dgemm_AtX(cudaStream_t st, const HB& a, const double* X, double* Y, int B) {
  if (B <= 0) return true;
  // Y (n x B) = A^T (n x d) X (d x B) on the DMMA path (dmma_gemm.cu)
  return dgemm(1, 0, a.n, B, a.d, a.A, a.ld, X, a.ld, Y, a.n, st);
}

}  // namespace ell1

using namespace ell1;

static int hb_mmax(const ell1_dict_t* D) {
  int64_t m = D->d + 32;
  if (m > D->n) m = D->n;
  return (int)m;
}

extern "C" int ell1_batch_homotopy_capacity(const ell1_dict_t* D) { return dict_ok(D) ? hb_mmax(D) : 0; }

extern "C" size_t ell1_batch_homotopy_workspace(const ell1_dict_t* D, int32_t B) {
  if (!dict_ok(D) || B < 1 || D->ext) return 0;
  const int64_t n = D->n, ld = D->ld, mm = hb_mmax(D);
  size_t s = 0;
  if (D->dtype == ELL1_F32) s += align_up(n * ld * 8, 256);           // widened A
  s += align_up(ld * B * 8, 256);                                      // Bm
  s += align_up((int64_t)sizeof(HI) * B, 256);
  s += 2 * align_up(n * B * 8, 256);                                   // X, Cin
  s += align_up(mm * mm * B * 8, 256);                                 // R
  s += align_up(mm * B * 4, 256) + align_up(n * B * 4, 256);           // sup, posof
  s += align_up(mm * B * 8, 256);                                      // dI
  s += 3 * align_up(ld * B * 8, 256) + 2 * align_up(n * B * 8, 256);   // V, V2, Rr, W, C
  s += 3 * align_up(B * 4, 256) + 4096;                                // act, act2, perm, counters
  return s;
}

extern "C" int ell1_batch_homotopy(const ell1_dict_t* D, const double* Bmat, int32_t B, double target,
                                   int32_t max_iter, const ell1_batch_out_t* out, double* lam_out,
                                   int32_t* notes, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || D->ext || !Bmat || B < 1 || !out || !out->x || !out->iterations || !out->converged ||
      !out->status || max_iter < 0 || !(target >= 0.0))
    return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = D->n, ld = D->ld;
  HB a;
  a.d = D->d; a.n = n; a.ld = ld; a.mmax = hb_mmax(D); a.target = target; a.max_iter = max_iter;
  Carve cv(ws, wsb);
  if (D->dtype == ELL1_F32) {
    double* A64 = cv.take<double>(n * ld);
    if (!cv.ok) return ELL1_ERR_ARG;
    widen_kernel<<<148 * 8, 256, 0, s>>>((const float*)D->A, A64, n * ld);
    a.A = A64;
  } else {
    a.A = (const double*)D->A;
  }
  const int64_t mm = a.mmax;
  double* Bm = cv.take<double>(ld * B);
  a.st = cv.take<HI>(B);
  a.X = cv.take<double>(n * B);
  a.Cin = cv.take<double>(n * B);
  a.R = cv.take<double>(mm * mm * B);
  a.sup = cv.take<int>(mm * B);
  a.posof = cv.take<int>(n * B);
  a.dI = cv.take<double>(mm * B);
  double* V1 = cv.take<double>(ld * B);
  double* V2 = cv.take<double>(ld * B);
  a.Rr = cv.take<double>(ld * B);
  a.W = cv.take<double>(n * B);
  a.C = cv.take<double>(n * B);
  int* act1 = cv.take<int>(B);
  int* act2 = cv.take<int>(B);
  int* perm = cv.take<int>(B);
  int* ctr = cv.take<int>(8);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.Bm = Bm;
  a.trace = out->trace;
  a.lam_out = lam_out;
  a.V = V1;
  if (cudaMemcpyAsync(Bm, Bmat, ld * B * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return ELL1_ERR_CUDA;
  // c = A^T b for every instance, then lambda0 / first atom
  if (!dgemm_AtX(s, a, Bm, a.C, B)) return ELL1_ERR_CUDA;
  hb_init<512><<<B, 512, 0, s>>>(a, B);
  // identity active list
  {
    std::vector<int> ident(B);
    for (int k = 0; k < B; ++k) ident[k] = k;
    if (cudaMemcpyAsync(act1, ident.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return ELL1_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
  }
  const size_t smem = (size_t)(HB_SMEM_FIXED + 2 * mm) * 8;
  if (!hb_smem_attr<128>(smem) || !hb_smem_attr<256>(smem) || !hb_smem_attr<512>(smem)) return ELL1_ERR_CUDA;
  int nact = B;
  int* act = act1;
  int* actn = act2;
  double* Vcur = V1;
  double* Valt = V2;
  while (nact > 0) {
    a.act = act;
    a.V = Vcur;
    hb_launch(0, hb_threads(nact), nact, smem, s, a);
    // drop finished instances from the GEMM operands
    hb_scan<<<1, 1024, 0, s>>>(a.st, act, nact, perm, ctr);
    int* box = host_mailbox();
    if (cudaMemcpyAsync(box, ctr, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
    const int nn = box[0];
    if (nn == 0) break;
    if (nn < nact) {
      dim3 g((unsigned)std::min<int64_t>((ld + 255) / 256, 8), (unsigned)nn);
      hb_permute<<<g, 256, 0, s>>>(act, perm, nn, actn, Vcur, Valt, ld);
      std::swap(act, actn);
      std::swap(Vcur, Valt);
      nact = nn;
      a.act = act;
      a.V = Vcur;
    }
    if (!dgemm_AtX(s, a, a.V, a.W, nact)) return ELL1_ERR_CUDA;
    hb_launch(1, hb_threads(nact), nact, smem, s, a);
    if (!dgemm_AtX(s, a, a.Rr, a.C, nact)) return ELL1_ERR_CUDA;
  }
  hb_out<<<B, 256, 0, s>>>(a, B, out->x, out->iterations, out->converged, out->status, notes);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
