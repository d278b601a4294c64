// linalg.cu — device versions of the reference's numerics / operator
// utilities that sit on the hot path's boundary:
//
//   ell1_chol_factor      dense upper Cholesky         numerics.chol_factor    (numerics.py:75-87)
//   ell1_chol_solve       (R^T R) x = rhs               CholFactor.solve        (numerics.py:62-65)
//   ell1_chol_append      factor of [[G, g], [g^T, s]]  numerics.chol_append    (numerics.py:115-137)
//   ell1_column_norms_sq  sum_i A_ij^2                  DenseDictionary.column_norms_sq (operators.py:44-45)
//   ell1_gram_dd          A diag(w) A^T  (cuBLAS)       DenseDictionary.(weighted_)gram_dd (operators.py:53-58)
//   ell1_pcg_dense        Jacobi-PCG on a dense SPD M   numerics.pcg_solve      (numerics.py:164-221)
//
// The factor routines run on one CTA (O(m^2) / O(m^3) with m = |support| or
// d); the PCG is a persistent grid over column panels of M (symmetric, so
// M p for owned columns is the local panel GEMV^T of the replicated p).
#include "solvers_common.cuh"
#include "factor.cuh"
#include "batched.cuh"

#define T0 if (threadIdx.x == 0)

namespace ell1 {

__global__ void __launch_bounds__(NTHR) chol_factor_kernel(const double* G, double* R, int m, int32_t* status) {
  __shared__ double sc[4];
  for (int64_t t = tix(); t < (int64_t)m * m; t += NTHR) R[t] = 0.0;
  __syncthreads();
  const bool ok = dense_chol(G, R, m, m, sc);
  if (tix() == 0) *status = ok ? 0 : 1;
}

__global__ void __launch_bounds__(NTHR) chol_solve_kernel(const double* R, const double* rhs, double* z, int m) {
  __shared__ double tile[32 * 32];
  for (int t = tix(); t < m; t += NTHR) z[t] = rhs[t];
  __syncthreads();
  trsv_RT(R, m, m, z, tile);
  trsv_R(R, m, m, z, tile);
}

// Rout (m+1 x m+1) = [[R, u], [0, sqrt(diag - u.u)]], u = R^{-T} g
__global__ void __launch_bounds__(NTHR) chol_append_kernel(const double* R, int m, const double* g, double diag,
                                                           double* Rout, double* u, int32_t* status) {
  __shared__ double tile[32 * 32];
  __shared__ double red[NWARP];
  const int m1 = m + 1;
  for (int64_t t = tix(); t < (int64_t)m1 * m1; t += NTHR) {
    const int i = (int)(t / m1), j = (int)(t % m1);
    Rout[t] = (i < m && j < m) ? R[(size_t)i * m + j] : 0.0;
  }
  for (int t = tix(); t < m; t += NTHR) u[t] = g[t];
  __syncthreads();
  double d2 = diag;
  if (m > 0) {
    trsv_RT(R, m, m, u, tile);
    double s = 0.0;
    for (int t = tix(); t < m; t += NTHR) s += u[t] * u[t];
    s = warp_sum(s);
    if (lnx() == 0) red[wpx()] = s;
    __syncthreads();
    double uu = 0.0;
    for (int w = 0; w < NWARP; ++w) uu += red[w];
    d2 = diag - uu;
    for (int t = tix(); t < m; t += NTHR) Rout[(size_t)t * m1 + m] = u[t];
  }
  if (tix() == 0) {
    if (d2 <= 0.0) *status = 1;
    else { *status = 0; Rout[(size_t)m * m1 + m] = sqrt(d2); }
  }
}

template <class TA>
__global__ void colnorm_kernel(const TA* A, int64_t d, int64_t n, int64_t ld, double* out) {
  const int64_t j = (int64_t)blockIdx.x * NWARP + wpx();
  if (j >= n) return;
  const TA* c = A + j * ld;
  double s = 0.0;
  for (int64_t i = lnx(); i < d; i += 32) { const double v = (double)c[i]; s = fma(v, v, s); }
  s = warp_sum(s);
  if (lnx() == 0) out[j] = s;
}

// AW[:, j] = w_j A[:, j] (fp64), A64 = A (fp64) — operands of the Gram GEMM
template <class TA>
__global__ void scale_cols_kernel(const TA* A, int64_t ld, int64_t n, const double* w, double* AW, double* A64) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * ld; t += (int64_t)gridDim.x * blockDim.x) {
    const double a = (double)A[t];
    if (A64) A64[t] = a;
    AW[t] = w ? a * w[t / ld] : a;
  }
}

// ---------------------------------------------------------------- dense PCG
struct PcgArgs {
  DictRaw D;                // M (m x m symmetric), column panels
  const double* rhs;
  const double* diag;       // Jacobi preconditioner (nullptr: identity)
  double tol;
  int max_iter;
  double* P;                // replicated p (ld)
  double* x_out;
  double* out;              // {converged, iterations, residual, status}
  GridBufs g;
  int wmax, rc;
};

constexpr int PCG_OV = 5;   // x, r, p, Ap, best_x

struct PcgV {
  double bn, rz, best, res;
  int k, done, conv, status, use_best;
};

// a grid barrier timed out (the kernel aborts cleanly): status ELL1_ERR_TIMEOUT in out[3]
__device__ __forceinline__ void pcg_timeout(const Ctx& E, double* out) {
  if (E.b == 0 && threadIdx.x == 0) { out[0] = 0.0; out[1] = 0.0; out[2] = NAN; out[3] = (double)ELL1_ERR_TIMEOUT; }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) pcg_kernel(const __grid_constant__ PcgArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ PcgV V;
  DictV<TA> D = dict_view<TA>(a.D);
  D.ext = 0;
  TA* panel = reinterpret_cast<TA*>(smem);
  double* ov = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + a.g.panel_bytes);
  if (tix() == 0) {
    ctx_init(E, D.d, D.n, 0, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.sh = ov + PCG_OV * a.wmax;
  }
  __syncthreads();
  double* X = ov;
  double* Rv = ov + a.wmax;
  double* Pv = ov + 2 * a.wmax;
  double* AP = ov + 3 * a.wmax;
  double* BX = ov + 4 * a.wmax;
  const Panel<TA> PN = setup_panel<TA>(E, D, panel, a.rc);
  const double* dg = a.diag;
  // r = rhs, z = M^-1 r, p = z, ||rhs||, r.z
  double s2[2] = {0.0, 0.0};
  for_owned(E, [&](int k) {
    const int64_t j = E.c0 + k;
    const double r = a.rhs[j];
    const double z = dg ? r / dg[j] : r;
    X[k] = 0.0; BX[k] = 0.0; Rv[k] = r; Pv[k] = z;
    a.P[j] = z;
    s2[0] += r * r;
    s2[1] += r * z;
  });
  if (!allreduce<2>(E, s2, 0u)) { pcg_timeout(E, a.out); return; }
  if (tix() == 0) {
    V.bn = sqrt(s2[0]); V.rz = s2[1]; V.best = V.bn; V.res = 0.0;
    V.k = 0; V.done = 0; V.conv = 0; V.status = 0; V.use_best = 0;
    if (V.bn == 0.0) { V.done = 1; V.conv = 1; }
  }
  __syncthreads();
  while (!V.done) {
    // every thread reads the budget before thread 0 advances V.k (a warp that
    // read the incremented count would leave the loop alone and write the
    // current iterate for its columns while the others go on)
    const bool over = V.k >= a.max_iter;
    __syncthreads();
    if (over) {                                      // budget: best iterate, not converged
      T0 { V.done = 1; V.use_best = 1; V.res = V.best; V.k = a.max_iter; }
      __syncthreads();
      break;
    }
    T0 V.k++;
    {
      const double* rs[1] = {a.P};
      double* os[1] = {AP};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);        // (M p)_own (M symmetric)
    }
    double q[1] = {0.0};
    for_owned(E, [&](int k) { q[0] += Pv[k] * AP[k]; });
    if (!allreduce<1>(E, q, 0u)) { pcg_timeout(E, a.out); return; }
    const double pAp = q[0];
    if (!isfinite(pAp)) { T0 { V.status = ELL1_BREAKDOWN; V.done = 1; } __syncthreads(); break; }
    if (pAp <= 0.0) { T0 { V.done = 1; V.use_best = 1; V.res = V.best; } __syncthreads(); break; }
    const double alpha = V.rz / pAp;
    double s[2] = {0.0, 0.0};
    for_owned(E, [&](int k) {
      X[k] = X[k] + alpha * Pv[k];
      const double r = Rv[k] - alpha * AP[k];
      Rv[k] = r;
      s[0] += r * r;
    });
    if (!allreduce<1>(E, *reinterpret_cast<double(*)[1]>(s), 0u)) { pcg_timeout(E, a.out); return; }
    const double res = sqrt(s[0]);
    if (!isfinite(res)) { T0 { V.status = ELL1_BREAKDOWN; V.done = 1; } __syncthreads(); break; }
    const bool better = res < V.best;
    if (better) for_owned(E, [&](int k) { BX[k] = X[k]; });
    __syncthreads();
    T0 { if (better) V.best = res; }
    if (res <= a.tol * V.bn) { T0 { V.done = 1; V.conv = 1; V.res = res; } __syncthreads(); break; }
    double rz1[1] = {0.0};
    for_owned(E, [&](int k) {
      const double z = dg ? Rv[k] / dg[E.c0 + k] : Rv[k];
      rz1[0] += Rv[k] * z;
    });
    if (!allreduce<1>(E, rz1, 0u)) { pcg_timeout(E, a.out); return; }
    const double beta = rz1[0] / V.rz;
    for_owned(E, [&](int k) {
      const double z = dg ? Rv[k] / dg[E.c0 + k] : Rv[k];
      const double p = z + beta * Pv[k];
      Pv[k] = p;
      a.P[E.c0 + k] = p;
    });
    __syncthreads();
    T0 V.rz = rz1[0];
    if (!grid_sync(E)) { pcg_timeout(E, a.out); return; }   // p complete before the next GEMV^T
  }
  __syncthreads();
  const bool ub = V.use_best;
  for_owned(E, [&](int k) { a.x_out[E.c0 + k] = ub ? BX[k] : X[k]; });
  if (E.b == 0 && tix() == 0) {
    a.out[0] = V.conv ? 1.0 : 0.0;
    a.out[1] = (double)V.k;
    a.out[2] = V.bn == 0.0 ? 0.0 : V.res / V.bn;
    a.out[3] = (double)V.status;
  }
}

}  // namespace ell1

using namespace ell1;

extern "C" int ell1_chol_factor(const double* G, double* R, int64_t m, int32_t* status, void* stream) {
  if (!G || !R || !status || m < 0 || m > (1 << 20)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (m == 0) return cudaMemsetAsync(status, 0, 4, s) == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  chol_factor_kernel<<<1, NTHR, 0, s>>>(G, R, (int)m, status);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_chol_solve(const double* R, const double* rhs, double* out, int64_t m, void* stream) {
  if (!R || !rhs || !out || m < 0 || m > (1 << 20)) return ELL1_ERR_ARG;
  if (m == 0) return ELL1_OK;
  chol_solve_kernel<<<1, NTHR, 0, (cudaStream_t)stream>>>(R, rhs, out, (int)m);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_chol_append(const double* R, int64_t m, const double* g, double diag, double* Rout,
                                double* work, int32_t* status, void* stream) {
  if ((m > 0 && (!R || !g || !work)) || !Rout || !status || m < 0 || m > (1 << 20)) return ELL1_ERR_ARG;
  chol_append_kernel<<<1, NTHR, 0, (cudaStream_t)stream>>>(R, (int)m, g, diag, Rout, work, status);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_column_norms_sq(const ell1_dict_t* D, double* out, void* stream) {
  if (!dict_ok(D) || !out) return ELL1_ERR_ARG;
  const unsigned nbk = (unsigned)((D->n + NWARP - 1) / NWARP);
  cudaStream_t s = (cudaStream_t)stream;
  if (D->dtype == ELL1_F64) colnorm_kernel<double><<<nbk, NTHR, 0, s>>>((const double*)D->A, D->d, D->n, D->ld, out);
  else colnorm_kernel<float><<<nbk, NTHR, 0, s>>>((const float*)D->A, D->d, D->n, D->ld, out);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" size_t ell1_gram_dd_workspace(const ell1_dict_t* D) {
  if (!dict_ok(D)) return 0;
  return (size_t)2 * D->n * D->ld * 8 + 512;
}

extern "C" int ell1_gram_dd(const ell1_dict_t* D, const double* w, double* G, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !G || !ws || wsb < ell1_gram_dd_workspace(D)) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  double* AW = (double*)ws;
  double* A64 = D->dtype == ELL1_F64 ? (double*)D->A : AW + D->n * D->ld;
  const int64_t tot = D->n * D->ld;
  const unsigned g = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16);
  if (D->dtype == ELL1_F64) scale_cols_kernel<double><<<g, 256, 0, s>>>((const double*)D->A, D->ld, D->n, w, AW, nullptr);
  else scale_cols_kernel<float><<<g, 256, 0, s>>>((const float*)D->A, D->ld, D->n, w, AW, A64);
  if (cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
  // G (d x d, ld d) = AW (d x n, ld) * A64^T on the DMMA path (dmma_gemm.cu)
  return dgemm(0, 1, D->d, D->d, D->n, AW, D->ld, A64, D->ld, G, D->d, s) ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" size_t ell1_pcg_workspace(const ell1_dict_t* M) {
  if (!dict_ok(M)) return 0;
  const int nb = pick_blocks(M->n, 0);
  return grid_bytes(nb, M->d, 0) + align_up(M->ld * 8, 256) + 1024;
}

extern "C" int ell1_pcg_dense(const ell1_dict_t* M, const double* rhs, const double* diag, double tol,
                              int32_t max_iter, double* x, double* out4, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(M) || M->d != M->n || M->ext || !rhs || !x || !out4 || max_iter < 0) return ELL1_ERR_ARG;
  const int nb = pick_blocks(M->n, 0);
  PcgArgs a;
  a.D = to_raw(M);
  a.rhs = rhs; a.diag = diag; a.tol = tol; a.max_iter = max_iter; a.x_out = x; a.out = out4;
  Carve cv(ws, wsb);
  if (!carve_grid(cv, a.g, nb, M->d, 0)) return ELL1_ERR_ARG;
  a.P = cv.take<double>(M->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(a.P, 0, M->ld * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  const SmemPlan sp = plan_smem(a.D, nb, PCG_OV, 2, true);
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = sp.panel_bytes;
  a.rc = sp.rc;
  a.wmax = sp.wmax;
  return (M->dtype == ELL1_F64) ? coop_launch(pcg_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(pcg_kernel<float>, nb, sp.bytes, s, a, a.g.bar);
}
