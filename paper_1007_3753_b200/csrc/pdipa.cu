// pdipa.cu — fused vector kernels of the primal-dual interior-point solver
// (pdipa.py:1-185).  The split LP
//   min 1'v  s.t.  [A, -A] v = b,  v >= 0        (v = [x+; x-], length 2n)
// needs, per Newton step, two dictionary products (panel GEMV / GEMV^T of
// libell1b200), the weighted row Gram A diag(w+ + w-) A^T (cuBLAS DGEMM via
// ell1_gram_dd), one d x d Cholesky solve, and the elementwise / reduction
// work below.  "split" = 1 folds the [A, -A] structure (vectors of length 2n
// against an n-column A); split = 0 runs the same formulas on an explicit
// A_ext with N columns (newton_kkt_step, pdipa.py:65-94).
// Every reduction is fixed order: per-CTA partials, then one CTA folds.
#include "solvers_common.cuh"

namespace ell1 {

constexpr int PB = 296;          // CTAs for the elementwise passes (2 per SM)
constexpr int PK = 4;            // scalars per pass

__global__ void __launch_bounds__(NTHR) pd_fold(const double* part, int nb, unsigned maxmask, unsigned minmask,
                                                double* out) {
  const int k = threadIdx.x;
  if (k >= PK) return;
  const bool mx = (maxmask >> k) & 1u, mn = (minmask >> k) & 1u;
  double s = mx ? -INFINITY : (mn ? INFINITY : 0.0);
  for (int c = 0; c < nb; ++c) {
    const double t = part[c * PK + k];
    s = mx ? nmax(s, t) : (mn ? ((t < s || t != t) ? t : s) : s + t);
  }
  out[k] = s;
}

// per-CTA fixed-order reduction of PK values into part[blockIdx.x][PK]
__device__ __forceinline__ void pd_cta(double (&v)[PK], unsigned maxmask, unsigned minmask, double* part) {
  __shared__ double sh[NWARP * PK];
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    const bool mx = (maxmask >> k) & 1u, mn = (minmask >> k) & 1u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = mx ? nmax(v[k], t) : (mn ? ((t < v[k] || t != t) ? t : v[k]) : v[k] + t);
    }
  }
  if (lnx() == 0)
#pragma unroll
    for (int k = 0; k < PK; ++k) sh[wpx() * PK + k] = v[k];
  __syncthreads();
  if (tix() < PK) {
    const int k = tix();
    const bool mx = (maxmask >> k) & 1u, mn = (minmask >> k) & 1u;
    double s = sh[k];
    for (int w = 1; w < NWARP; ++w) {
      const double t = sh[w * PK + k];
      s = mx ? nmax(s, t) : (mn ? ((t < s || t != t) ? t : s) : s + t);
    }
    part[blockIdx.x * PK + k] = s;
  }
}

__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * NTHR; }
__device__ __forceinline__ int64_t gidx() { return (int64_t)blockIdx.x * NTHR + threadIdx.x; }

// u = x[:n] - x[n:] (split) or u = x; out: max|u|
__global__ void __launch_bounds__(NTHR) pd_split_kernel(int64_t n, int split, const double* x, double* u,
                                                        double* part) {
  double v[PK] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k = gidx(); k < n; k += gstride()) {
    const double t = split ? x[k] - x[n + k] : x[k];
    u[k] = t;
    v[0] = nmax(v[0], fabs(t));
  }
  pd_cta(v, 1u, 0u, part);
}

// rp = b - Ax (d), rd = c - [Aty; -Aty] - z (N2): {sum rp^2, b.y, sum rd^2, c.x}
__global__ void __launch_bounds__(NTHR) pd_resid_kernel(int64_t d, int64_t n, int split, const double* Ax,
                                                        const double* b, const double* y, const double* Aty,
                                                        const double* x, const double* z, const double* c,
                                                        double* rp, double* rd, double* part) {
  double v[PK] = {0.0, 0.0, 0.0, 0.0};
  const int64_t N2 = split ? 2 * n : n;
  for (int64_t i = gidx(); i < d; i += gstride()) {
    const double r = b[i] - Ax[i];
    rp[i] = r;
    v[0] += r * r;
    v[1] += b[i] * y[i];
  }
  for (int64_t k = gidx(); k < N2; k += gstride()) {
    const double ck = c ? c[k] : 1.0;
    const double at = split ? (k < n ? Aty[k] : -Aty[k - n]) : Aty[k];
    const double r = ck - at - z[k];
    rd[k] = r;
    v[2] += r * r;
    v[3] += ck * x[k];
  }
  pd_cta(v, 0u, 0u, part);
}

// rc = mu_hat - x z, w = x / z, v = rc / z - w rd; wsum = w+ + w-, vd = v+ - v- (split)
__global__ void __launch_bounds__(NTHR) pd_prep_kernel(int64_t n, int split, const double* x, const double* z,
                                                       const double* rd, double mu_hat, double* rc, double* w,
                                                       double* wsum, double* vd) {
  const int64_t N2 = split ? 2 * n : n;
  for (int64_t k = gidx(); k < N2; k += gstride()) {
    const double zk = z[k];
    const double r = mu_hat - x[k] * zk;
    const double wk = x[k] / zk;
    rc[k] = r;
    w[k] = wk;
  }
  if (split) {
    for (int64_t k = gidx(); k < n; k += gstride()) {
      const double zp = z[k], zm = z[n + k];
      const double xp = x[k], xm = x[n + k];
      const double wp = xp / zp, wm = xm / zm;
      const double rcp = mu_hat - xp * zp, rcm = mu_hat - xm * zm;
      wsum[k] = wp + wm;
      vd[k] = (rcp / zp - wp * rd[k]) - (rcm / zm - wm * rd[n + k]);
    }
  } else {
    for (int64_t k = gidx(); k < n; k += gstride()) {
      const double zk = z[k], xk = x[k];
      const double wk = xk / zk;
      const double r = mu_hat - xk * zk;
      wsum[k] = wk;
      vd[k] = r / zk - wk * rd[k];
    }
  }
}

// dz = rd - [Atdy; -Atdy], dx = rc / z - w dz;
// {min_{dx<0} -x/dx, min_{dz<0} -z/dz, nonfinite(dx, dz, dy), sum (z dx + x dz - rc)^2}
__global__ void __launch_bounds__(NTHR) pd_dir_kernel(int64_t n, int split, int64_t d, const double* Atdy,
                                                      const double* dy, const double* rd, const double* rc,
                                                      const double* x, const double* z, const double* w,
                                                      double* dx, double* dz, double* part) {
  double v[PK] = {INFINITY, INFINITY, 0.0, 0.0};
  const int64_t N2 = split ? 2 * n : n;
  for (int64_t k = gidx(); k < N2; k += gstride()) {
    const double at = split ? (k < n ? Atdy[k] : -Atdy[k - n]) : Atdy[k];
    const double dzk = rd[k] - at;
    const double dxk = rc[k] / z[k] - w[k] * dzk;
    dz[k] = dzk;
    dx[k] = dxk;
    if (dxk < 0.0) { const double t = -x[k] / dxk; v[0] = (t < v[0] || t != t) ? t : v[0]; }
    if (dzk < 0.0) { const double t = -z[k] / dzk; v[1] = (t < v[1] || t != t) ? t : v[1]; }
    if (!isfinite(dxk) || !isfinite(dzk)) v[2] = 1.0;
    const double e = z[k] * dxk + x[k] * dzk - rc[k];
    v[3] += e * e;
  }
  for (int64_t i = gidx(); i < d; i += gstride())
    if (!isfinite(dy[i])) v[2] = 1.0;
  pd_cta(v, 0x4u, 0x3u, part);
}

// sum (x + ap dx)(z + ad dz)
__global__ void __launch_bounds__(NTHR) pd_mu_kernel(int64_t N2, const double* x, const double* dx, double ap,
                                                     const double* z, const double* dz, double ad, double* part) {
  double v[PK] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k = gidx(); k < N2; k += gstride()) {
    const double xn = x[k] + ap * dx[k];
    const double zn = z[k] + ad * dz[k];
    v[0] += xn * zn;
  }
  pd_cta(v, 0u, 0u, part);
}

// x += ap dx, z += ad dz (N2), y += ad dy (d)
__global__ void __launch_bounds__(NTHR) pd_update_kernel(int64_t N2, int64_t d, double* x, const double* dx,
                                                         double ap, double* z, const double* dz, double ad,
                                                         double* y, const double* dy) {
  for (int64_t k = gidx(); k < N2; k += gstride()) {
    x[k] = x[k] + ap * dx[k];
    z[k] = z[k] + ad * dz[k];
  }
  for (int64_t i = gidx(); i < d; i += gstride()) y[i] = y[i] + ad * dy[i];
}

static int pd_blocks(int64_t len) {
  int64_t b = (len + NTHR - 1) / NTHR;
  if (b > PB) b = PB;
  return b < 1 ? 1 : (int)b;
}

}  // namespace ell1

using namespace ell1;

extern "C" size_t ell1_pd_workspace(void) { return (size_t)PB * 8 * 8 + 256; }   // also fits the shard reductions

extern "C" int ell1_pd_split(int64_t n, int32_t split, const double* x, double* u, double* out, void* ws,
                             void* stream) {
  if (n < 1 || !x || !u || !out || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = pd_blocks(n);
  pd_split_kernel<<<nb, NTHR, 0, s>>>(n, split, x, u, (double*)ws);
  pd_fold<<<1, 32, 0, s>>>((const double*)ws, nb, 1u, 0u, out);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_pd_resid(int64_t d, int64_t n, int32_t split, const double* Ax, const double* b,
                             const double* y, const double* Aty, const double* x, const double* z,
                             const double* c, double* rp, double* rd, double* out4, void* ws, void* stream) {
  if (d < 1 || n < 1 || !Ax || !b || !y || !Aty || !x || !z || !rp || !rd || !out4 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = pd_blocks(split ? 2 * n : (n > d ? n : d));
  pd_resid_kernel<<<nb, NTHR, 0, s>>>(d, n, split, Ax, b, y, Aty, x, z, c, rp, rd, (double*)ws);
  pd_fold<<<1, 32, 0, s>>>((const double*)ws, nb, 0u, 0u, out4);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_pd_prep(int64_t n, int32_t split, const double* x, const double* z, const double* rd,
                            double mu_hat, double* rc, double* w, double* wsum, double* vd, void* stream) {
  if (n < 1 || !x || !z || !rd || !rc || !w || !wsum || !vd) return ELL1_ERR_ARG;
  pd_prep_kernel<<<pd_blocks(split ? 2 * n : n), NTHR, 0, (cudaStream_t)stream>>>(n, split, x, z, rd, mu_hat, rc,
                                                                                  w, wsum, vd);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_pd_direction(int64_t n, int32_t split, int64_t d, const double* Atdy, const double* dy,
                                 const double* rd, const double* rc, const double* x, const double* z,
                                 const double* w, double* dx, double* dz, double* out4, void* ws, void* stream) {
  if (n < 1 || !Atdy || !dy || !rd || !rc || !x || !z || !w || !dx || !dz || !out4 || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = pd_blocks(split ? 2 * n : n);
  pd_dir_kernel<<<nb, NTHR, 0, s>>>(n, split, d, Atdy, dy, rd, rc, x, z, w, dx, dz, (double*)ws);
  pd_fold<<<1, 32, 0, s>>>((const double*)ws, nb, 0x4u, 0x3u, out4);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_pd_mu(int64_t N2, const double* x, const double* dx, double ap, const double* z,
                          const double* dz, double ad, double* out, void* ws, void* stream) {
  if (N2 < 1 || !x || !dx || !z || !dz || !out || !ws) return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = pd_blocks(N2);
  pd_mu_kernel<<<nb, NTHR, 0, s>>>(N2, x, dx, ap, z, dz, ad, (double*)ws);
  pd_fold<<<1, 32, 0, s>>>((const double*)ws, nb, 0u, 0u, out);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_pd_update(int64_t N2, int64_t d, double* x, const double* dx, double ap, double* z,
                              const double* dz, double ad, double* y, const double* dy, void* stream) {
  if (N2 < 1 || !x || !dx || !z || !dz || !y || !dy) return ELL1_ERR_ARG;
  pd_update_kernel<<<pd_blocks(N2 > d ? N2 : d), NTHR, 0, (cudaStream_t)stream>>>(N2, d, x, dx, ap, z, dz, ad, y,
                                                                                  dy);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

namespace ell1 {
// M[i][i] += alpha v[i] (v may be null), then *trace = sum_i M[i][i] (fixed order, one CTA)
__global__ void pd_diag_kernel(int64_t d, int64_t ldm, double* M, double alpha, const double* v, double* trace) {
  __shared__ double sh[NWARP];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += NTHR) {
    double m = M[i * ldm + i];
    if (v) { m = m + alpha * v[i]; M[i * ldm + i] = m; }
    s += m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lnx() == 0) sh[wpx()] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NWARP; ++w) t += sh[w];
    *trace = t;
  }
}
}  // namespace ell1

extern "C" int ell1_pd_diag(int64_t d, int64_t ldm, double* M, double alpha, const double* v, double* trace,
                            void* stream) {
  if (d < 1 || ldm < d || !M || !trace) return ELL1_ERR_ARG;
  pd_diag_kernel<<<1, NTHR, 0, (cudaStream_t)stream>>>(d, ldm, M, alpha, v, trace);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
