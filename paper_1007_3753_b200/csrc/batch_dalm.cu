// batch_dalm.cu — dual ALM over a batch of instances sharing one dictionary
// (element j equals alm.dalm_solve on (D, b_j), alm.py:206-272), e.g. the
// cross-and-bouquet face-recognition batch of BASELINE config 3 on [A, sI].
//
// Per iteration (alm.py:172-189, 239-268; Ginv = G^{-1}, G = A A^T (+ s^2 I)):
//   z-kernel  : z = clamp(A^T y + x/beta)
//   float64 storage:
//     GEMM      : A z;  rhs-kernel: rhs = A z - (A x - b)/beta
//     GEMM      : y = Ginv rhs  (d^2 per instance: the reference's cho_solve), y-kernel: b^T y
//   float32 storage (tensor-core GEMMs need the fp32 operands of the precomputed M = Ginv A):
//     v = z - x/beta; GEMMs [M | Ginv] v and A z; y-kernel: y = M v + Ginv b / beta, rhs
//   GEMM      : A^T y
//   x-kernel  : x_new = x - beta (z - A^T y)
//   GEMM      : A [A^T y | x_new]   (one GEMM over 2B columns)
//   c-kernel  : certificate, residual, gap, trace, stopping rules
//   [refinement for instances failing the certificate: Ginv resid GEMM]
#include <cstdio>
#include "batched.cuh"

namespace ell1 {

// min CTAs per SM of the y / x epilogues (88 / 74 registers uncapped: 2-3 CTAs per SM)
#ifndef BD_MINB
#define BD_MINB 4
#endif
#ifndef BD_MINB_ZC
#define BD_MINB_ZC 4
#endif

struct DI {
  double bn, l1_prev, by, rhs2, resid2, rr, l1, maxu;
  double S[6];
  int it, hist, active, status, conv, orig, refine, cnt;
};

struct BDArgs {
  int64_t d, n, N, ld, ldx;
  int ext, f32, cg;
  int vec;                   // fp32 storage with even n, d, ld: paired loads / stores in the epilogues
  int fuse_ext;              // fp32 [A, sI]: [M | Ginv] V as one tensor-core GEMM (no GEXT)
  int gcert;                 // certificate from G y (the opts carry G): P2[:, j] = G y_j already
                             // includes the [A, sI] block, only A x_new needs the s x_e term
  double s, beta, ytol;
  const double* Bm;         // ld x B
  const double* C0;         // ld x B  (Ginv b)
  double* X[2];             // ldx x B
  double* Z;                // ldx x B
  double* UX;               // ldx x 2B : [A^T y | x_new] GEMM operand (fp64)
  double* V;                // ldx x B
  double* Y[2];             // ld x B
  double* AX;               // ld x B (A x of the current x)
  double* RHS;              // ld x B
  double* RES;              // ld x B
  double* P1; double* P2;   // GEMM outputs ld x B / ld x 2B (fp64)
  double* GEXT;             // ld x B (Ginv v_ext)
  float* V32; float* Z32; float* UX32; float* Y32; float* P1f; float* P2f; float* P3f;
  float* V32l; float* Z32l; float* UX32l; float* Y32l;   // pre: lo halves (the arrays above hold rna_tf32 hi)
  int pre;                   // vec path writes the GEMM operands pre-split (3xTF32 hi / lo, no in-GEMM split)
  float* UT32;               // fp32 storage: U = A^T y (n x B, pitch n), the GEMM output itself;
                             // the fp64 copies of U and x_new in UX are then not kept
  DI* inst;
  ell1_ctrl_t C;
  int* counters;            // [0] refine, [1] active
  double* x_out; int* it_out; int* conv_out; int* status_out;
  double* trace;            // [B0][max_iter + 1][4]
  int ix, iy;
};

// paired (16-byte fp64 / 8-byte fp32) accesses of the fp32-storage epilogues
// (BDArgs::vec: n, d, ld even, so no pair straddles a block boundary)
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ float2 ldf2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(double* p, double u, double v) {
  *reinterpret_cast<double2*>(p) = make_double2(u, v);
}
__device__ __forceinline__ void stf2(float* p, double u, double v) {
  *reinterpret_cast<float2*>(p) = make_float2((float)u, (float)v);
}
// GEMM operand pair store: plain fp32, or the 3xTF32 split (hi = rna_tf32(x),
// lo = rna_tf32(x - hi): the same bits as the GEMM's in-kernel split)
__device__ __forceinline__ void stf2s(float* h, float* l, bool pre, double u, double v) {
  const float fu = (float)u, fv = (float)v;
  if (!pre) {
    *reinterpret_cast<float2*>(h) = make_float2(fu, fv);
    return;
  }
  const float hu = tf32_rna(fu), hv = tf32_rna(fv);
  *reinterpret_cast<float2*>(h) = make_float2(hu, hv);
  *reinterpret_cast<float2*>(l) = make_float2(tf32_rna(fu - hu), tf32_rna(fv - hv));
}
__device__ __forceinline__ double clamp1(double t) { return t > 1.0 ? 1.0 : (t < -1.0 ? -1.0 : t); }

__device__ __forceinline__ double bd_rd(const BDArgs& a, const double* p64, const float* p32, int64_t i) {
  return a.f32 ? (double)p32[i] : p64[i];
}

__global__ void __launch_bounds__(BT) bd_init(const BDArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW + 1];
  DI& I = a.inst[j];
  const double* b = a.Bm + (int64_t)j * a.ld;
  double v[1] = {0.0};
  for (int64_t i = threadIdx.x; i < a.ld; i += BT) {
    const double bi = b[i];
    v[0] += bi * bi;
    a.AX[(int64_t)j * a.ld + i] = 0.0;
    a.Y[0][(int64_t)j * a.ld + i] = 0.0;
    a.Y[1][(int64_t)j * a.ld + i] = 0.0;
  }
  for (int64_t k = threadIdx.x; k < a.ldx; k += BT) {
    a.X[0][(int64_t)j * a.ldx + k] = 0.0;
    a.X[1][(int64_t)j * a.ldx + k] = 0.0;
    a.UX[(int64_t)j * a.ldx + k] = 0.0;            // A^T y_0 = 0
  }
  if (a.f32)
    for (int64_t k = threadIdx.x; k < a.n; k += BT) a.UT32[(int64_t)j * a.n + k] = 0.f;
  cta_reduce<1>(v, 0u, sh);
  if (threadIdx.x == 0) {
    I.orig = j; I.it = 0; I.hist = 0; I.conv = 0; I.status = ELL1_OK; I.l1_prev = 0.0; I.refine = 0;
    I.bn = sqrt(v[0]);
    I.active = I.bn != 0.0;
    if (a.trace) {
      double* tr = a.trace + (int64_t)j * (a.C.max_iter + 1) * 4;
      tr[0] = 0.0; tr[1] = 0.0; tr[2] = I.bn; tr[3] = 0.0;   // alm.py:233 (0.0 residual on zero data)
    }
    if (!I.active) {                                         // alm.py:223-226
      I.status = ELL1_ZERO_DATA; I.conv = 1;
      a.it_out[j] = 0; a.conv_out[j] = 1; a.status_out[j] = ELL1_ZERO_DATA;
    } else {
      atomicAdd(a.counters + 1, 1);
    }
  }
  if (!I.active)
    for (int64_t k = threadIdx.x; k < a.N; k += BT) a.x_out[(int64_t)j * a.N + k] = 0.0;
}

// z = clamp(A^T y + x/beta), v = z - x/beta (alm.py:239)
template <bool VEC>
__global__ void __launch_bounds__(BT, BD_MINB_ZC) bd_z(const BDArgs a) {
  const int j = blockIdx.x;
  DI& I = a.inst[j];
  if (!I.active) return;
  if (threadIdx.x == 0) { I.it++; I.refine = 0; }
  if constexpr (VEC) {
    const int64_t o = (int64_t)j * a.ldx;
    const double* __restrict__ x = a.X[a.ix] + o;
    const float* __restrict__ u32 = a.UT32 + (int64_t)j * a.n;
    const double* __restrict__ ycur = a.Y[a.iy] + (int64_t)j * a.ld;
    double* __restrict__ zo = a.Z + o;
    float* __restrict__ v32 = a.V32 + o;
    float* __restrict__ z32 = a.Z32 + o;
    float* __restrict__ v32l = a.V32l + o;
    float* __restrict__ z32l = a.Z32l + o;
    const bool fuse = a.fuse_ext, pre = a.pre;
    const int64_t n = a.n, h = a.N / 2;
    const double beta = a.beta, sc = a.s;
#pragma unroll 4
    for (int64_t t = threadIdx.x; t < h; t += BT) {
      const int64_t k = 2 * t;
      const double2 xx = ld2(x + k);
      double u0, u1;
      if (k < n) {
        const float2 uu = ldf2(u32 + k);
        u0 = uu.x; u1 = uu.y;
      } else {
        const double2 yy = ld2(ycur + (k - n));
        u0 = sc * yy.x; u1 = sc * yy.y;
      }
      const double xb0 = xx.x / beta, xb1 = xx.y / beta;
      const double z0 = clamp1(u0 + xb0), z1 = clamp1(u1 + xb1);
      st2(zo + k, z0, z1);
      if (k < n) {
        stf2s(v32 + k, v32l + k, pre, z0 - xb0, z1 - xb1);
        stf2s(z32 + k, z32l + k, pre, z0, z1);
      } else if (fuse) {
        stf2s(v32 + k, v32l + k, pre, sc * (z0 - xb0), sc * (z1 - xb1));
      }
    }
    return;
  }
  const int64_t o = (int64_t)j * a.ldx;
  const double* __restrict__ x = a.X[a.ix] + o;
  const double* __restrict__ u = a.UX + o;
  const float* __restrict__ u32 = a.UT32 + (int64_t)j * a.n;
  const double* __restrict__ ycur = a.Y[a.iy] + (int64_t)j * a.ld;
  double* __restrict__ zo = a.Z + o;
  double* __restrict__ vo = a.V + o;
  float* __restrict__ v32 = a.V32 + o;
  float* __restrict__ z32 = a.Z32 + o;
  const bool keep_v = false;                                // fp64: y = Ginv rhs needs no v
  const bool f32 = a.f32, fuse = a.fuse_ext;
  const int64_t n = a.n;
  const double beta = a.beta, sc = a.s;
#pragma unroll 4
  for (int64_t k = threadIdx.x; k < a.N; k += BT) {
    const double xb = x[k] / beta;
    // U = A^T y of the current y: fp32 storage reads the GEMM output (+ s y for [A, sI])
    const double uk = !f32 ? u[k] : (k < n ? (double)u32[k] : sc * ycur[k - n]);
    const double t = uk + xb;
    const double z = t > 1.0 ? 1.0 : (t < -1.0 ? -1.0 : t);
    zo[k] = z;
    const double vv = k < n ? z - xb : sc * (z - xb);
    if (keep_v) vo[k] = vv;
    if (f32 && (k < n || fuse)) v32[k] = (float)vv;
    if (f32 && k < n) z32[k] = (float)z;
  }
}

// y = M v + Ginv b / beta; rhs = A z - (A x - b)/beta (alm.py:179-180)
template <bool VEC>
__global__ void __launch_bounds__(BT, BD_MINB) bd_y(const BDArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW * 2 + 2];
  DI& I = a.inst[j];
  if (!I.active) return;
  const int64_t oj = (int64_t)j * a.ld;
  // restrict-qualified views: the four row loads of a thread are independent of
  // its stores, so the unrolled loop keeps them all in flight
  const double* __restrict__ b = a.Bm + oj;
  double* __restrict__ y = a.Y[a.iy ^ 1] + oj;
  const double* __restrict__ zx = a.Z + (int64_t)j * a.ldx + a.n;
  const double* __restrict__ c0 = a.C0 + oj;
  const double* __restrict__ ax = a.AX + oj;
  const double* __restrict__ gx = a.GEXT + oj;
  const float* __restrict__ p1f = a.P1f + oj;
  const float* __restrict__ p2f = a.P2f + oj;
  const double* __restrict__ p1 = a.P1 + oj;
  const double* __restrict__ p2 = a.P2 + oj;
  float* __restrict__ y32 = a.Y32 + oj;
  double* __restrict__ rh = a.RHS + oj;
  const bool f32 = a.f32, addg = a.ext && !a.fuse_ext, ext = a.ext;
  const double beta = a.beta, sc = a.s;
  double q[2] = {0.0, 0.0};
  if constexpr (VEC) {
    const int64_t h = a.d / 2;
#pragma unroll 4
    for (int64_t t = threadIdx.x; t < h; t += BT) {
      const int64_t i = 2 * t;
      const float2 m2 = ldf2(p1f + i);
      double mv0 = m2.x, mv1 = m2.y;
      if (addg) { const double2 g = ld2(gx + i); mv0 = mv0 + g.x; mv1 = mv1 + g.y; }
      const double2 c = ld2(c0 + i);
      const double y0 = mv0 + c.x / beta, y1 = mv1 + c.y / beta;
      const float2 a2 = ldf2(p2f + i);
      double az0 = a2.x, az1 = a2.y;
      if (ext) { const double2 zz = ld2(zx + i); az0 = az0 + sc * zz.x; az1 = az1 + sc * zz.y; }
      const double2 bb = ld2(b + i), xx = ld2(ax + i);
      const double r0 = az0 - (xx.x - bb.x) / beta, r1 = az1 - (xx.y - bb.y) / beta;
      st2(y + i, y0, y1);
      stf2s(y32 + i, a.Y32l + oj + i, a.pre, y0, y1);
      st2(rh + i, r0, r1);
      q[0] += r0 * r0; q[0] += r1 * r1;
      q[1] += bb.x * y0; q[1] += bb.y * y1;
    }
  } else
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < a.d; i += BT) {
    double mv = f32 ? (double)p1f[i] : p1[i];
    if (addg) mv = mv + gx[i];
    const double yi = mv + c0[i] / beta;
    double az = f32 ? (double)p2f[i] : p2[i];
    if (ext) az = az + sc * zx[i];
    const double bi = b[i];
    const double rhs = az - (ax[i] - bi) / beta;
    y[i] = yi;
    if (f32) y32[i] = (float)yi;
    rh[i] = rhs;
    q[0] += rhs * rhs;
    q[1] += bi * yi;
  }
  cta_reduce<2>(q, 0u, sh);
  if (threadIdx.x == 0) { I.rhs2 = q[0]; I.by = q[1]; }
}

// float64 storage: rhs = A z - (A x - b)/beta (alm.py:179), ||rhs||^2
__global__ void __launch_bounds__(BT) bd_rhs(const BDArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW + 1];
  DI& I = a.inst[j];
  if (!I.active) return;
  const int64_t oj = (int64_t)j * a.ld;
  const double* __restrict__ b = a.Bm + oj;
  const double* __restrict__ zx = a.Z + (int64_t)j * a.ldx + a.n;
  const double* __restrict__ ax = a.AX + oj;
  const double* __restrict__ p2 = a.P2 + oj;
  double* __restrict__ rh = a.RHS + oj;
  const bool ext = a.ext;
  const double beta = a.beta, sc = a.s;
  double q[1] = {0.0};
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < a.d; i += BT) {
    double az = p2[i];
    if (ext) az = az + sc * zx[i];
    const double rhs = az - (ax[i] - b[i]) / beta;
    rh[i] = rhs;
    q[0] += rhs * rhs;
  }
  cta_reduce<1>(q, 0u, sh);
  if (threadIdx.x == 0) I.rhs2 = q[0];
}

// float64 storage: y = Ginv rhs (the GEMM output P1), b^T y
__global__ void __launch_bounds__(BT) bd_yg(const BDArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW + 1];
  DI& I = a.inst[j];
  if (!I.active) return;
  const int64_t oj = (int64_t)j * a.ld;
  const double* __restrict__ b = a.Bm + oj;
  double* __restrict__ y = a.Y[a.iy ^ 1] + oj;
  const double* __restrict__ p1 = a.P1 + oj;
  double q[1] = {0.0};
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < a.d; i += BT) {
    const double yi = p1[i];
    y[i] = yi;
    q[0] += b[i] * yi;
  }
  cta_reduce<1>(q, 0u, sh);
  if (threadIdx.x == 0) I.by = q[0];
}

// x_new = x - beta (z - A^T y) (alm.py:245-246); U = A^T y lives in UX[:, j]
template <bool VEC>
__global__ void __launch_bounds__(BT, BD_MINB) bd_x(const BDArgs a, const double* Ut, const float* Ut32, int refine_only) {
  const int j = blockIdx.x;
  __shared__ double sh[BW * 6 + 6];
  DI& I = a.inst[j];
  if (!I.active || (refine_only && !I.refine)) return;
  const int64_t o = (int64_t)j * a.ldx;
  const double* __restrict__ x = a.X[a.ix] + o;
  double* __restrict__ u = a.UX + o;                                   // [A^T y | x_new] block j
  double* __restrict__ xn = a.UX + ((int64_t)gridDim.x + j) * a.ldx;   // second half of UX
  const double* __restrict__ y = a.Y[a.iy ^ 1] + (int64_t)j * a.ld;
  const double* __restrict__ zz = a.Z + o;
  double* __restrict__ xw = a.X[a.ix ^ 1] + o;
  float* __restrict__ ux32 = a.UX32 + o;
  float* __restrict__ xn32 = a.UX32 + ((int64_t)gridDim.x + j) * a.ldx;
  const double* __restrict__ ut = Ut + (int64_t)j * a.n;
  const float* __restrict__ ut32 = Ut32 + (int64_t)j * a.n;
  const bool relest = a.C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool f32 = a.f32;
  const int64_t n = a.n;
  const double beta = a.beta, sc = a.s;
  double s[6] = {0, 0, 0, 0, 0, 0};                       // l1, max|Aty|, max|x|, dx2, xp2, -
  if constexpr (VEC) {
    const int64_t h = a.N / 2;
#pragma unroll 4
    for (int64_t t = threadIdx.x; t < h; t += BT) {
      const int64_t k = 2 * t;
      double u0, u1;
      if (k < n) {
        const float2 uu = ldf2(ut32 + k);
        u0 = uu.x; u1 = uu.y;
      } else {
        const double2 yy = ld2(y + (k - n));
        u0 = sc * yy.x; u1 = sc * yy.y;
      }
      const double2 xo = ld2(x + k), z2 = ld2(zz + k);
      const double v0 = xo.x - beta * (z2.x - u0), v1 = xo.y - beta * (z2.y - u1);
      st2(xw + k, v0, v1);
      if (k < n) {
        stf2s(ux32 + k, a.UX32l + o + k, a.pre, u0, u1);
        stf2s(xn32 + k, a.UX32l + ((int64_t)gridDim.x + j) * a.ldx + k, a.pre, v0, v1);
      }
      s[0] += fabs(v0); s[0] += fabs(v1);
      s[1] = nmax(nmax(s[1], fabs(u0)), fabs(u1));
      s[2] = nmax(nmax(s[2], fabs(v0)), fabs(v1));
      if (relest) {
        const double d0 = v0 - xo.x, d1 = v1 - xo.y;
        s[3] += d0 * d0; s[3] += d1 * d1;
        s[4] += xo.x * xo.x; s[4] += xo.y * xo.y;
      }
    }
  } else
#pragma unroll 4
  for (int64_t k = threadIdx.x; k < a.N; k += BT) {
    double uk;
    if (k < n) uk = f32 ? (double)ut32[k] : ut[k];
    else uk = sc * y[k - n];                              // robust.py:96
    const double xo = x[k];
    const double xv = xo - beta * (zz[k] - uk);
    if (!f32) { u[k] = uk; xn[k] = xv; }                  // fp64 GEMM operand [U | x_new]
    xw[k] = xv;
    if (f32 && k < n) {
      ux32[k] = (float)uk;
      xn32[k] = (float)xv;
    }
    s[0] += fabs(xv);
    s[1] = nmax(s[1], fabs(uk));
    s[2] = nmax(s[2], fabs(xv));
    if (relest) { const double dd = xv - xo; s[3] += dd * dd; s[4] += xo * xo; }
  }
  cta_reduce<6>(s, 0x6u, sh);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) I.S[k] = s[k];
}

// certificate, residual, trace, convergence (alm.py:181-188, 249-268)
template <bool VEC>
__global__ void __launch_bounds__(BT, BD_MINB_ZC) bd_c(const BDArgs a, int refine_only) {
  const int j = blockIdx.x;
  const int B = gridDim.x;
  __shared__ double sh[BW * 3 + 3];
  __shared__ int fin;
  DI& I = a.inst[j];
  if (!I.active || (refine_only && !I.refine)) return;
  const int64_t oj = (int64_t)j * a.ld;
  const double* b = a.Bm + oj;
  const double* u = a.UX + (int64_t)j * a.ldx;
  // x_new: fp32 storage keeps it only in X (the UX copy is the fp64 GEMM operand)
  const double* xn = a.f32 ? a.X[a.ix ^ 1] + (int64_t)j * a.ldx : a.UX + ((int64_t)B + j) * a.ldx;
  const double* ynew = a.Y[a.iy ^ 1] + oj;
  const double cut = 1e-10 * pymax(I.S[2], 1.0);
  double q[3] = {0.0, 0.0, 0.0};
  {
    const float* __restrict__ pu = a.P2f + (int64_t)j * a.ld;
    const float* __restrict__ px = a.P2f + ((int64_t)B + j) * a.ld;
    const double* __restrict__ pu64 = a.P2 + (int64_t)j * a.ld;
    const double* __restrict__ px64 = a.P2 + ((int64_t)B + j) * a.ld;
    const double* __restrict__ rh = a.RHS + oj;
    const double* __restrict__ bb = b;
    const double* __restrict__ yn = ynew;
    const double* __restrict__ ue = u + a.n;
    const double* __restrict__ xe = xn + a.n;
    double* __restrict__ res = a.RES + oj;
    double* __restrict__ axo = a.AX + oj;
    const bool f32 = a.f32, ext = a.ext;
    const double sc = a.s;
    if constexpr (VEC) {
      const int64_t h = a.d / 2;
      const bool gc = a.gcert;
#pragma unroll 4
      for (int64_t t = threadIdx.x; t < h; t += BT) {
        const int64_t i = 2 * t;
        const float2 u2 = ldf2(pu + i), x2 = ldf2(px + i);
        double au0 = u2.x, au1 = u2.y, ax0 = x2.x, ax1 = x2.y;
        if (ext) {
          if (!gc) {
            const double2 yy = ld2(yn + i);
            au0 = au0 + sc * (sc * yy.x); au1 = au1 + sc * (sc * yy.y);
          }
          const double2 xx = ld2(xe + i);
          ax0 = ax0 + sc * xx.x; ax1 = ax1 + sc * xx.y;
        }
        const double2 r2 = ld2(rh + i), b2 = ld2(bb + i);
        const double e0 = r2.x - au0, e1 = r2.y - au1;
        st2(res + i, e0, e1);
        st2(axo + i, ax0, ax1);
        const double q0 = b2.x - ax0, q1 = b2.y - ax1;
        q[0] += e0 * e0; q[0] += e1 * e1;
        q[1] += q0 * q0; q[1] += q1 * q1;
      }
      const double* __restrict__ xs = xn;
      const int64_t hN = a.N / 2;
#pragma unroll 4
      for (int64_t t = threadIdx.x; t < hN; t += BT) {
        const double2 v = ld2(xs + 2 * t);
        if (fabs(v.x) > cut) q[2] += 1.0;
        if (fabs(v.y) > cut) q[2] += 1.0;
      }
    } else {
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < a.d; i += BT) {
      double aau = f32 ? (double)pu[i] : pu64[i];
      double ax = f32 ? (double)px[i] : px64[i];
      if (ext) {
        if (!a.gcert) aau = aau + sc * (f32 ? sc * yn[i] : ue[i]);
        ax = ax + sc * xe[i];
      }
      const double resid = rh[i] - aau;
      res[i] = resid;
      axo[i] = ax;
      const double r = bb[i] - ax;
      q[0] += resid * resid;
      q[1] += r * r;
    }
    const double* __restrict__ xs = xn;
#pragma unroll 4
    for (int64_t k = threadIdx.x; k < a.N; k += BT) if (fabs(xs[k]) > cut) q[2] += 1.0;
    }
  }
  cta_reduce<3>(q, 0u, sh);
  if (threadIdx.x == 0) {
    int done = 0;
    I.resid2 = q[0]; I.rr = q[1]; I.cnt = (int)q[2];
    if (!a.cg && sqrt(q[0]) > a.ytol * pymax(1.0, sqrt(I.rhs2))) {
      if (I.refine) { I.status = ELL1_ILL_CONDITIONED; done = 3; }
      else { I.refine = 1; atomicAdd(a.counters, 1); done = -1; }
    }
    if (done == 0) {
      I.refine = 0;
      const double rn = sqrt(I.rr);
      const double l1 = I.S[0];
      if (a.trace) {
        double* tr = a.trace + ((int64_t)I.orig * (a.C.max_iter + 1) + I.it) * 4;
        tr[0] = (double)I.it; tr[1] = l1; tr[2] = rn; tr[3] = (double)I.cnt;
      }
      const double rel = rn / I.bn;
      const double gap = l1 - I.by / pymax(1.0, I.S[1]);
      if (rel <= a.C.tol && gap <= a.C.tol * pymax(1.0, l1)) done = 1;
      else if (a.C.stop_kind != ELL1_STOP_NONE) {
        I.hist = I.hist < 2 ? I.hist + 1 : 2;
        if (stop_fires(a.C.stop_kind, a.C.stop_thr, I.hist, l1, I.l1_prev, I.S[3], I.S[4], 0.0,
                       a.C.gt_norm, rel))
          done = 1;
        I.l1_prev = l1;
      }
      if (!done && I.it >= a.C.max_iter) done = 2;
    }
    if (done > 0) {
      I.conv = done == 1;
      I.active = 0;
      a.it_out[I.orig] = I.it; a.conv_out[I.orig] = I.conv;
      a.status_out[I.orig] = done == 3 ? ELL1_ILL_CONDITIONED : ELL1_OK;
      atomicSub(a.counters + 1, 1);
    }
    fin = done > 0;
  }
  __syncthreads();
  if (fin) {
    double* xo = a.x_out + (int64_t)I.orig * a.N;
    for (int64_t k = threadIdx.x; k < a.N; k += BT) xo[k] = xn[k];
  }
}

// refinement y += Ginv resid (alm.py:184), flagged instances only
__global__ void __launch_bounds__(BT) bd_refine(const BDArgs a, const double* delta) {
  const int j = blockIdx.x;
  __shared__ double sh[BW + 1];
  DI& I = a.inst[j];
  if (!I.active || !I.refine) return;
  const int64_t oj = (int64_t)j * a.ld;
  double* y = a.Y[a.iy ^ 1] + oj;
  const double* b = a.Bm + oj;
  double q[1] = {0.0};
  for (int64_t i = threadIdx.x; i < a.d; i += BT) {
    const double yi = y[i] + delta[oj + i];
    y[i] = yi;
    if (a.f32) {
      const float f = (float)yi;
      if (a.pre) {
        const float h = tf32_rna(f);
        a.Y32[oj + i] = h;
        a.Y32l[oj + i] = tf32_rna(f - h);
      } else {
        a.Y32[oj + i] = f;
      }
    }
    q[0] += b[i] * yi;
  }
  cta_reduce<1>(q, 0u, sh);
  if (threadIdx.x == 0) I.by = q[0];
}

// row-major 3xTF32 split of [M | Ginv] (ld x N, pitch pr): the y-step's two
// products M v_A + Ginv (s v_ext) as one K = n + d GEMM
__global__ void bd_mext_split(const float* __restrict__ M, const double* __restrict__ Ginv, int64_t ld, int64_t n,
                              int64_t d, int64_t pr, float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ float t[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, i = i0 + threadIdx.x;
    float x = 0.f;
    if (i < ld) x = k < n ? M[k * ld + i] : (k < n + d ? (float)Ginv[(k - n) * ld + i] : 0.f);
    t[r][threadIdx.x] = x;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, k = k0 + threadIdx.x;
    if (i < ld && k < pr) {
      const float x = t[threadIdx.x][r];
      const float h = tf32_rna(x);
      hi[i * pr + k] = h;
      lo[i * pr + k] = tf32_rna(x - h);
    }
  }
}

// delta[:, j] = Ginv resid[:, j] for the instances flagged for refinement
// (graph driver: cuBLAS may record nodes a conditional body cannot hold).
// grid (row blocks of 256, instances); Ginv column-major ld x d (symmetric)
__global__ void __launch_bounds__(256) bd_refine_gemv(const BDArgs a, const double* __restrict__ Ginv,
                                                      double* __restrict__ delta) {
  const int j = blockIdx.y;
  const DI& I = a.inst[j];
  if (!I.active || !I.refine) return;
  __shared__ double r[1024];
  const double* __restrict__ res = a.RES + (int64_t)j * a.ld;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double acc = 0.0;
  for (int64_t k0 = 0; k0 < a.d; k0 += 1024) {
    const int64_t kn = a.d - k0 < 1024 ? a.d - k0 : 1024;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < kn; t += 256) r[t] = res[k0 + t];
    __syncthreads();
    if (i < a.ld) {
#pragma unroll 8
      for (int64_t k = 0; k < kn; ++k) acc = fma(Ginv[(k0 + k) * a.ld + i], r[k], acc);
    }
  }
  if (i < a.ld) delta[(int64_t)j * a.ld + i] = acc;
}

// graph driver: IF condition = refinement flagged by this certificate round
__global__ void bd_if(const int* ctr, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, ctr[0] > 0 ? 1u : 0u);
}

// graph driver: keep iterating while no compaction is due (same rule as the
// host loop) and the pass budget of one launch lasts; ctr[4] counts passes
__global__ void bd_loop(int* ctr, cudaGraphConditionalHandle h, int Bcur) {
  if (threadIdx.x == 0) {
    const int nact = ctr[1];
    const int passes = ++ctr[4];
    const bool compact = nact < Bcur * 3 / 4 || (nact < Bcur && nact <= 64);
    cudaGraphSetConditional(h, (nact > 0 && !compact && passes < 4096) ? 1u : 0u);
  }
}

__global__ void bd_scan(DI* inst, int B, int* perm, int* newB) {
  __shared__ int base;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < B; c0 += blockDim.x) {
    const int j = c0 + threadIdx.x;
    const int act = (j < B) ? inst[j].active : 0;
    const unsigned m = __ballot_sync(0xffffffffu, act);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) wsum[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = base;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { const int t = wsum[k]; wsum[k] = acc; acc += t; }
      base = acc;
    }
    __syncthreads();
    if (act) perm[wsum[w] + __popc(m & ((1u << l) - 1))] = j;
    __syncthreads();
  }
  if (threadIdx.x == 0) *newB = base;
}

template <class T>
__global__ void bd_gather(const T* src, T* dst, int64_t rows, int64_t ld, const int* perm, int B) {
  const int k = blockIdx.y;
  if (k >= B) return;
  const int64_t s = (int64_t)perm[k] * ld, d = (int64_t)k * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    dst[d + i] = src[s + i];
}

__global__ void bd_f2d(const double* src, float* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

}  // namespace ell1

using namespace ell1;

static int64_t r4(int64_t x) { return (x + 3) / 4 * 4; }

extern "C" size_t ell1_batch_dalm_workspace(const ell1_dict_t* D, int32_t B) {
  if (!dict_ok(D) || B < 1) return 0;
  const int64_t N = ncols_of(D), ldx = r4(N), ld = D->ld;
  size_t s = 0;
  s += 5 * align_up(ldx * B * 8, 256) + align_up(ldx * 2 * B * 8, 256);   // X[2], Z, V, scratch-x, UX
  s += 9 * align_up(ld * B * 8, 256) + align_up(ld * 2 * B * 8, 256);      // Y[2], AX, RHS, RES, C0, Bm, P1, GEXT, P2
  s += align_up(ldx * B * 4, 256) * 3 + align_up(ldx * 2 * B * 4, 256) + align_up(ld * B * 4, 256) * 3 +
       align_up(ld * 2 * B * 4, 256);
  s += 2 * align_up((int64_t)sizeof(DI) * B, 256) + align_up(B * 4, 256) + align_up(ldx * B * 8, 256);
  if (D->dtype == ELL1_F32)                                  // producer-split operand lo halves
    s += align_up(ldx * B * 4, 256) * 2 + align_up(ldx * 2 * B * 4, 256) + align_up(ld * B * 4, 256);
  if (D->dtype == ELL1_F32)                                  // splits of A and M + operand scratch
    s += (size_t)(f32split_floats(D, (ldx > ld ? ldx : ld) * 2 * B) + f32split_dict_floats(D) +
                  2 * align_up(ld * ld, 64) + 2 * align_up(ld * align_up(ld, 4), 64) + align_up(ld * ld, 64) +
                  2 * align_up(ld * ldx, 64)) * 4 + 2048;
  return s + 8192;
}

extern "C" int ell1_batch_dalm(const ell1_dict_t* D, const double* Bmat, int32_t B, const ell1_ctrl_t* C,
                               const ell1_dalm_opts_t* O, const ell1_batch_out_t* out, void* ws,
                               size_t wsb, void* stream) {
  if (!dict_ok(D) || !Bmat || B < 1 || !C || !O || !O->M || !O->Ginv || !(O->beta > 0) || !out ||
      !out->x || !out->iterations || !out->converged || !out->status)
    return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t N = ncols_of(D), ldx = r4(N), ld = D->ld, d = D->d;
  BDArgs a;
  a.d = d; a.n = D->n; a.N = N; a.ld = ld; a.ldx = ldx;
  a.ext = D->ext; a.f32 = D->dtype == ELL1_F32; a.cg = O->y_cg_step; a.fuse_ext = 0;
  a.vec = a.f32 && D->n % 2 == 0 && D->d % 2 == 0 && D->ld % 2 == 0;
  a.gcert = O->G != nullptr;
  a.s = D->ext_scale; a.beta = O->beta; a.ytol = O->y_tol;
  a.C = *C;
  if (a.cg) return ELL1_ERR_ARG;   // batched CG y-step: not provided (use the single-instance solver)
  Carve cv(ws, wsb);
  a.X[0] = cv.take<double>(ldx * B); a.X[1] = cv.take<double>(ldx * B);
  a.Z = cv.take<double>(ldx * B); a.V = cv.take<double>(ldx * B);
  double* xscr = cv.take<double>(ldx * B);
  a.UX = cv.take<double>(ldx * 2 * B);
  a.Y[0] = cv.take<double>(ld * B); a.Y[1] = cv.take<double>(ld * B);
  a.AX = cv.take<double>(ld * B); a.RHS = cv.take<double>(ld * B); a.RES = cv.take<double>(ld * B);
  double* C0 = cv.take<double>(ld * B);
  double* Bm = cv.take<double>(ld * B);
  a.P1 = cv.take<double>(ld * B); a.GEXT = cv.take<double>(ld * B);
  a.P2 = cv.take<double>(ld * 2 * B);
  a.V32 = cv.take<float>(ldx * B); a.Z32 = cv.take<float>(ldx * B);
  float* T32 = cv.take<float>(ldx * B);
  a.UX32 = cv.take<float>(ldx * 2 * B);
  a.Y32 = cv.take<float>(ld * B); a.P1f = cv.take<float>(ld * B); a.P3f = cv.take<float>(ld * B);
  a.pre = a.vec;
  if (const char* e = getenv("ELL1_BD_PRE")) a.pre = a.pre && e[0] != '0';   // diagnostics (A/B)
  a.V32l = a.Z32l = a.UX32l = a.Y32l = nullptr;
  if (a.pre) {
    a.V32l = cv.take<float>(ldx * B); a.Z32l = cv.take<float>(ldx * B);
    a.UX32l = cv.take<float>(ldx * 2 * B); a.Y32l = cv.take<float>(ld * B);
  }
  a.P2f = cv.take<float>(ld * 2 * B);
  a.inst = cv.take<DI>(B);
  DI* inst2 = cv.take<DI>(B);
  int* perm = cv.take<int>(B);
  double* scratch = cv.take<double>(ldx * B);
  int* ctr = cv.take<int>(8);
  if (!cv.ok) return ELL1_ERR_ARG;
  (void)xscr;
  a.UT32 = T32;
  F32Split spA, spM, spX, spG;
  const F32Split* pA = nullptr;
  const F32Split* pM = nullptr;
  if (a.f32 && a.gcert) {
    // G (d columns x ld, fp64) -> fp32 -> 3xTF32 split, the certificate's G y operand
    float* Gf = cv.take<float>(ld * ld);
    if (!cv.ok) return ELL1_ERR_ARG;
    bd_f2d<<<(unsigned)((d * ld + 255) / 256 < 148 * 8 ? (d * ld + 255) / 256 : 148 * 8), 256, 0, s>>>(O->G, Gf,
                                                                                                   d * ld);
    ell1_dict_t GD = *D;
    GD.A = Gf; GD.n = d; GD.ext = 0;
    if (!f32split_dict(spG, cv, &GD, Gf, s)) return ELL1_ERR_ARG;
  }
  if (a.f32) {
    if (!f32split_setup(spA, cv, D, (ldx > ld ? ldx : ld) * 2 * B, s)) return ELL1_ERR_ARG;
    spM = spA;                                               // shares the operand scratch
    if (!f32split_dict(spM, cv, D, (const float*)O->M, s)) return ELL1_ERR_ARG;
    if (a.ext) {
      float* xh = cv.take<float>(ld * ldx);
      float* xl = cv.take<float>(ld * ldx);
      if (!cv.ok) return ELL1_ERR_ARG;
      dim3 g((unsigned)((ldx + 31) / 32), (unsigned)((ld + 31) / 32));
      bd_mext_split<<<g, dim3(32, 8), 0, s>>>((const float*)O->M, O->Ginv, ld, D->n, d, ldx, xh, xl);
      spX = spM;
      spX.Arhi = xh; spX.Arlo = xl; spX.pr = ldx;
      a.fuse_ext = 1;
    }
    pA = &spA; pM = &spM;
  }
  a.Bm = Bm; a.C0 = C0;
  a.counters = ctr;
  a.x_out = out->x; a.it_out = out->iterations; a.conv_out = out->converged; a.status_out = out->status;
  a.trace = out->trace;
  a.ix = 0; a.iy = 0;
  if (cudaMemcpyAsync(Bm, Bmat, ld * B * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaMemsetAsync(ctr, 0, 32, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaMemsetAsync(a.UX32, 0, ldx * 2 * B * 4, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (a.pre && cudaMemsetAsync(a.UX32l, 0, ldx * 2 * B * 4, s) != cudaSuccess) return ELL1_ERR_CUDA;
  // C0 = Ginv B (Ginv column-major ld x d, float64), the fp32 y step's constant term
  if (a.f32 && !dgemm(0, 0, ld, B, d, O->Ginv, ld, Bm, ld, C0, ld, s)) return ELL1_ERR_CUDA;
  bd_init<<<B, BT, 0, s>>>(a);
  ell1_dict_t MD = *D;
  MD.A = O->M;                                              // M has A's layout / dtype
  int Bcur = B;
  // hc = {refine flags, active instances}: read once here, then together with
  // every certificate round's refine count (one device->host sync per iteration)
  int* hc = host_mailbox();
  hc[0] = hc[1] = 0;
  if (cudaMemcpyAsync(hc, ctr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;

  cudaStream_t ks = s;                                   // launch stream (a capture stream while recording)
  // U = A^T y_new (n x B), x_new, A [U | x_new], certificate (refine_only: flagged instances)
  auto tail_part = [&](const BDArgs& aa, int Bc, int refine_only) -> bool {
    void* Ut = aa.f32 ? (void*)T32 : (void*)scratch;
    if (!gemm_AtR(ks, D, aa.f32 ? (const void*)aa.Y32 : (const void*)aa.Y[aa.iy ^ 1], ld, Ut, D->n, Bc, pA,
                  aa.Y32l))
      return false;
    // [U | x_new] for the Bc instances: the x_new block starts at column Bc
    if (aa.vec) bd_x<true><<<Bc, BT, 0, ks>>>(aa, (const double*)Ut, (const float*)Ut, refine_only);
    else bd_x<false><<<Bc, BT, 0, ks>>>(aa, (const double*)Ut, (const float*)Ut, refine_only);
    if (aa.gcert) {
      // certificate A A^T y as G y (d^2 per instance instead of d n) and A x_new
      if (aa.f32) {
        if (!sgemm_split(ks, 0, (int)ld, Bc, (int)d, &spG, aa.Y32, ld, aa.P2f, ld, aa.Y32l)) return false;
        if (!gemm_AX(ks, D, aa.UX32 + (int64_t)Bc * ldx, ldx, aa.P2f + (int64_t)Bc * ld, ld, Bc, pA,
                     aa.pre ? aa.UX32l + (int64_t)Bc * ldx : nullptr))
          return false;
      } else {
        if (!dgemm(0, 0, ld, Bc, d, O->G, ld, aa.Y[aa.iy ^ 1], ld, aa.P2, ld, ks)) return false;
        if (!gemm_AX(ks, D, aa.UX + (int64_t)Bc * ldx, ldx, aa.P2 + (int64_t)Bc * ld, ld, Bc)) return false;
      }
    } else if (aa.f32) {
      if (!gemm_AX(ks, D, aa.UX32, ldx, aa.P2f, ld, 2 * Bc, pA, aa.UX32l)) return false;
    } else {
      if (!gemm_AX(ks, D, aa.UX, ldx, aa.P2, ld, 2 * Bc)) return false;
    }
    if (cudaMemsetAsync(ctr, 0, 4, ks) != cudaSuccess) return false;
    if (aa.vec) bd_c<true><<<Bc, BT, 0, ks>>>(aa, refine_only);
    else bd_c<false><<<Bc, BT, 0, ks>>>(aa, refine_only);
    return cudaGetLastError() == cudaSuccess;
  };
  // one iteration up to the certificate (bd_c raises ctr[0] refine flags)
  auto main_part = [&](const BDArgs& aa, int Bc) -> bool {
    if (aa.vec) bd_z<true><<<Bc, BT, 0, ks>>>(aa);
    else bd_z<false><<<Bc, BT, 0, ks>>>(aa);
    if (!aa.f32) {
      // y = G^-1 rhs (dual_y_solve's cho_solve, alm.py:179-180) on the DMMA path
      if (!gemm_AX(ks, D, aa.Z, ldx, aa.P2, ld, Bc)) return false;
      bd_rhs<<<Bc, BT, 0, ks>>>(aa);
      if (!dgemm(0, 0, ld, Bc, d, O->Ginv, ld, aa.RHS, ld, aa.P1, ld, ks)) return false;
      bd_yg<<<Bc, BT, 0, ks>>>(aa);
      return tail_part(aa, Bc, 0);
    }
    const void* Vop = aa.f32 ? (const void*)aa.V32 : (const void*)aa.V;
    const void* Zop = aa.f32 ? (const void*)aa.Z32 : (const void*)aa.Z;
    if (aa.fuse_ext) {
      // P1 = [M | Ginv] V over K = n + d (V's identity block already carries s)
      if (!sgemm_split(ks, 0, (int)ld, Bc, (int)N, &spX, aa.V32, ldx, aa.P1f, ld, aa.V32l))
        return false;
    } else if (!gemm_AX(ks, &MD, Vop, ldx, aa.f32 ? (void*)aa.P1f : (void*)aa.P1, ld, Bc, pM, aa.V32l)) {
      return false;
    }
    if (!gemm_AX(ks, D, Zop, ldx, aa.f32 ? (void*)aa.P2f : (void*)aa.P2, ld, Bc, pA, aa.Z32l)) return false;
    if (aa.ext && !aa.fuse_ext) {
      // identity block of M: s Ginv v_ext (s folded into v_ext by bd_z)
      if (!dgemm(0, 0, ld, Bc, d, O->Ginv, ld, aa.V + D->n, ldx, aa.GEXT, ld, ks)) return false;
    }
    if (aa.vec) bd_y<true><<<Bc, BT, 0, ks>>>(aa);
    else bd_y<false><<<Bc, BT, 0, ks>>>(aa);
    return tail_part(aa, Bc, 0);
  };
  // y += Ginv resid for the flagged instances (alm.py:184), then their certificate again
  auto refine_part = [&](const BDArgs& aa, int Bc, bool own_gemv) -> bool {
    if (own_gemv) {
      bd_refine_gemv<<<dim3((unsigned)((ld + 255) / 256), (unsigned)Bc), 256, 0, ks>>>(aa, O->Ginv, aa.GEXT);
    } else if (!dgemm(0, 0, ld, Bc, d, O->Ginv, ld, aa.RES, ld, aa.GEXT, ld, ks)) {
      return false;
    }
    bd_refine<<<Bc, BT, 0, ks>>>(aa, aa.GEXT);
    return tail_part(aa, Bc, 1);
  };

  // CUDA-graph driver (fp32 storage on the tensor-core GEMM path; the fp64
  // path's cuBLAS DGEMMs record nodes a conditional body cannot hold): two
  // iterations (both buffer parities) per WHILE-body pass, each followed by
  // an IF node running the refinement when bd_c raised a flag; the WHILE
  // condition (bd_loop) drops when compaction is due or everything finished.
  bool use_graph = true;
  if (const char* e = getenv("ELL1_BATCH_GRAPH")) use_graph = use_graph && e[0] != '0';
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int gB = -1, gpar = -1, gfail = 0;
  bool use_plain = true;
  if (const char* e = getenv("ELL1_BATCH_GRAPH")) use_plain = e[0] != '0';
  cudaGraphExec_t pexec[2] = {nullptr, nullptr};
  struct GraphGuard {                                  // every exit path releases the graphs
    cudaGraph_t& g;
    cudaGraphExec_t& e;
    cudaGraphExec_t* pe;
    ~GraphGuard() {
      if (e) cudaGraphExecDestroy(e);
      if (g) cudaGraphDestroy(g);
      for (int q = 0; q < 2; ++q)
        if (pe[q]) cudaGraphExecDestroy(pe[q]);
    }
  } graph_guard{graph, gexec, pexec};
  int pB = -1;
  auto build_graph = [&]() -> bool {
    gfail = 0;
#define GSTEP(expr)          \
  do {                       \
    ++gfail;                 \
    if (!(expr)) return false; \
  } while (0)
    GSTEP(cudaGraphCreate(&graph, 0) == cudaSuccess);
    cudaGraphConditionalHandle hloop, hif[2];
    GSTEP(cudaGraphConditionalHandleCreate(&hloop, graph, 1, cudaGraphCondAssignDefault) == cudaSuccess);
    for (int q = 0; q < 2; ++q)
      GSTEP(cudaGraphConditionalHandleCreate(&hif[q], graph, 0, cudaGraphCondAssignDefault) == cudaSuccess);
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hloop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    GSTEP(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp) == cudaSuccess);
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraphNode_t last = nullptr;
    BDArgs aa = a;
    // record on a private stream (the caller's may be the legacy default
    // stream, which cannot capture); the graph is launched on the caller's
    cudaStream_t cs = nullptr;
    GSTEP(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess);
    struct Restore {
      cudaStream_t& ks; cudaStream_t s; cudaStream_t cs;
      ~Restore() { ks = s; cudaStreamDestroy(cs); }
    } restore{ks, s, cs};
    ks = cs;
    for (int q = 0; q < 2; ++q) {
      aa.ix = aa.iy = a.ix ^ q;
      GSTEP(cudaStreamBeginCaptureToGraph(cs, body, last ? &last : nullptr, nullptr, last ? 1 : 0,
                                          cudaStreamCaptureModeRelaxed) == cudaSuccess);
      bool ok = main_part(aa, Bcur);
      if (ok) bd_if<<<1, 32, 0, cs>>>(ctr, hif[q]);
      cudaStreamCaptureStatus cst;
      ok = ok && cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps) == cudaSuccess && ndeps == 1;
      cudaGraphNode_t tailn = ok ? deps[0] : nullptr;
      cudaGraph_t tmp;
      GSTEP(cudaStreamEndCapture(cs, &tmp) == cudaSuccess);
      GSTEP(ok);
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hif[q];
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      cudaGraphNode_t inode;
      GSTEP(cudaGraphAddNode(&inode, body, &tailn, 1, &ip) == cudaSuccess);
      GSTEP(cudaStreamBeginCaptureToGraph(cs, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed) == cudaSuccess);
      ok = refine_part(aa, Bcur, true);
      GSTEP(cudaStreamEndCapture(cs, &tmp) == cudaSuccess);
      GSTEP(ok);
      last = inode;
    }
    GSTEP(cudaStreamBeginCaptureToGraph(cs, body, &last, nullptr, 1, cudaStreamCaptureModeRelaxed) == cudaSuccess);
    bd_loop<<<1, 32, 0, cs>>>(ctr, hloop, Bcur);
    cudaGraph_t tmp;
    GSTEP(cudaStreamEndCapture(cs, &tmp) == cudaSuccess);
    ++gfail;
    return cudaGraphInstantiate(&gexec, graph, 0) == cudaSuccess;
#undef GSTEP
  };

  while (true) {
    const int nact = hc[1];
    if (nact <= 0) break;
    if (nact < Bcur * 3 / 4 || (nact < Bcur && nact <= 64)) {
      bd_scan<<<1, 1024, 0, s>>>(a.inst, Bcur, perm, ctr + 2);
      bool cok = true;
      auto pm = [&](double* M, int64_t rows, int64_t ldm) {
        dim3 g((unsigned)((rows + 255) / 256 < 64 ? (rows + 255) / 256 : 64), (unsigned)nact);
        bd_gather<double><<<g, 256, 0, s>>>(M, scratch, rows, ldm, perm, nact);
        cok = cok && cudaMemcpyAsync(M, scratch, ldm * nact * 8, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      };
      pm(a.X[a.ix], N, ldx);
      if (a.f32) {                                          // A^T y of the current y
        dim3 g((unsigned)((D->n + 255) / 256 < 64 ? (D->n + 255) / 256 : 64), (unsigned)nact);
        bd_gather<float><<<g, 256, 0, s>>>(T32, (float*)scratch, D->n, D->n, perm, nact);
        cok = cok && cudaMemcpyAsync(T32, scratch, D->n * nact * 4, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      } else {
        pm(a.UX, N, ldx);
      }
      pm(a.Y[a.iy], ld, ld);
      pm(a.AX, ld, ld);
      if (a.f32) pm(C0, ld, ld);
      pm(Bm, ld, ld);
      {
        const int64_t words = (int64_t)sizeof(DI) / 4;
        bd_gather<int><<<dim3(1, (unsigned)nact), 64, 0, s>>>((const int*)a.inst, (int*)inst2, words, words, perm, nact);
        cok = cok && cudaMemcpyAsync(a.inst, inst2, sizeof(DI) * nact, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      }
      if (!cok || cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
      Bcur = nact;
    }
    // ---- DALM iterations over Bcur instances
    if (use_graph && Bcur >= 32) {
      // device-driven: whole iterations (and the rare certificate refinement)
      // inside one CUDA graph whose WHILE node runs until an instance
      // finishes often enough to warrant compaction
      if (!gexec || gB != Bcur || gpar != a.ix) {
        if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
        if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
        if (!build_graph()) {
          if (getenv("ELL1_DEBUG"))
            fprintf(stderr, "ell1_batch_dalm: graph build (B=%d) failed at step %d (%s)\n", Bcur, gfail,
                    cudaGetErrorString(cudaGetLastError()));
          use_graph = false;                                 // fall back to host-driven iterations
          if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
          cudaGetLastError();
          continue;
        }
        gB = Bcur;
        gpar = a.ix;
      }
      if (cudaMemsetAsync(ctr + 4, 0, 4, s) != cudaSuccess) return ELL1_ERR_CUDA;
      if (cudaGraphLaunch(gexec, s) != cudaSuccess) return ELL1_ERR_CUDA;
      if (cudaMemcpyAsync(hc, ctr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
      if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
      continue;                                              // parity unchanged (even iteration count)
    }
    // host-driven iteration; its launches are replayed from a per-(B, parity)
    // graph when one could be recorded (one API call instead of ~10 library calls)
    if (use_plain && (pB != Bcur)) {
      for (int q = 0; q < 2; ++q)
        if (pexec[q]) { cudaGraphExecDestroy(pexec[q]); pexec[q] = nullptr; }
      pB = Bcur;
    }
    if (use_plain && !pexec[a.ix]) {
      cudaStream_t cs = nullptr;
      cudaGraph_t pg = nullptr;
      bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
      if (ok) {
        ks = cs;
        ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        if (ok) {
          ok = main_part(a, Bcur);
          ok = cudaStreamEndCapture(cs, &pg) == cudaSuccess && ok;
        }
        ks = s;
        cudaStreamDestroy(cs);
      }
      ok = ok && cudaGraphInstantiate(&pexec[a.ix], pg, 0) == cudaSuccess;
      if (pg) cudaGraphDestroy(pg);
      if (!ok) {
        pexec[a.ix] = nullptr;
        use_plain = false;
        cudaGetLastError();
      }
    }
    if (use_plain && pexec[a.ix]) {
      if (cudaGraphLaunch(pexec[a.ix], s) != cudaSuccess) return ELL1_ERR_CUDA;
    } else if (!main_part(a, Bcur)) {
      return ELL1_ERR_CUDA;
    }
    if (cudaMemcpyAsync(hc, ctr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
    if (hc[0] != 0) {
      // one refinement round; instances failing it again end ill-conditioned
      // inside bd_c, so no further refine flags can be raised
      if (!refine_part(a, Bcur, false)) return ELL1_ERR_CUDA;
      if (cudaMemcpyAsync(hc, ctr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
      if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
    }
    a.ix ^= 1;
    a.iy ^= 1;
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}
