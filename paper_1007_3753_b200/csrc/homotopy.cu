// homotopy.cu — LASSO solution path (homotopy.solve_path, homotopy.py:128-244)
// as one persistent cooperative launch.
//
// Per breakpoint: the direction d_I = (A_I^T A_I)^{-1} sgn(c_I) = W W^T sgn
// from the maintained upper Cholesky factor R AND its inverse W = R^{-1}
// (CTA 0: two parallel triangular matvecs instead of two serial
// substitutions; appends extend W by one column, deletes rotate W's columns
// with the same Givens sequence that re-triangularises R, refactorisations
// rebuild W column-parallel over the whole grid),
// v = A_I d_I (support-sparse panel GEMV: only support columns are read),
// w = A^T v (panel GEMV^T), the drift check ||w_I - sgn|| (w_I == A_I^T v),
// the step lengths gamma+/gamma- as grid-wide (value, lowest index) argmins,
// the add (chol_append: triangular solve) or remove (chol_delete: block shift
// + LINPACK rank-1 update) event on CTA 0, then r = b - A_I x_I, c = A^T r and
// the lambda drift repair.  Degenerate supports fall back to a dense
// refactorisation / ridge (homotopy.py:53-64, 118-125) on CTA 0.
#include "solvers_common.cuh"
#include "factor.cuh"

namespace ell1 {

struct HomArgs {
  DictRaw D;
  const double* b;
  double target;
  int max_iter;
  int mmax;                 // factor capacity
  GridBufs g;
  double* R;                // mmax x mmax row-major upper factor
  double* W;                // mmax x mmax row-major upper inverse W = R^{-1}
  double* Wt;               // its transpose (row-major lower), so W^T v is a row-wise matvec too
  double* G;                // mmax x mmax scratch (dense refactor, shifts)
  int* sup;                 // support list (reference order)
  int* posof;               // column -> support position or -1 (N)
  double* sgn;              // mmax
  double* dI;               // mmax
  double* gcol;             // mmax
  double* dfull;            // N, direction (zero off support)
  double* colv;             // ld: the entering column / scratch d-vector
  double* Vd;               // replicated v = A_I d_I (ld)
  double* Rd;               // replicated r = b - A_I x_I (ld)
  ell1_state_t* st;
  double* trace;
  double* x_out; double* c_out;
  double* lam_path;         // optional: lambda after each breakpoint (path CSV)
  int* sup_out;             // optional: support list (observer)
  double* R_out;            // optional: factor, m x m row-major (observer)
  int max_steps;
  int wmax;
  unsigned long long* prof;
};

enum { H_LAM = 0, H_LAM0, H_FLOOR, H_PASSES };
constexpr int HOM_OV = 5;       // x, c, w, mask, sgn-of-owned scratch

struct HomV {
  double lam, lam0, floor, passes, gp, gm, drift, sgnn, l1, rr, lam_emp, top, d2;
  int it, m, ip, im, conv, status, quit, phase, steps, remove, ridge, pos, fail, finish, note;
};

#define T0 if (threadIdx.x == 0)

// Triangular matvec out = M v over rows of a row-major m x m triangle (ldr):
// LOWER: row j uses columns [0, j]; else row i uses [i, m).  A warp takes 4
// rows at a time and issues every load of a 128-column segment of all 4 rows
// before the FMAs (one L2 round trip per 128-column segment, not per row).
template <bool LOWER>
static __device__ void tri_mv(const double* M, int ldr, int m, const double* v, double* out) {
  constexpr int RW = 4, CH = 4;
  for (int r0 = wpx() * RW; r0 < m; r0 += NWARP * RW) {
    double acc[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) acc[k] = 0.0;
    const int lo = LOWER ? 0 : r0;                   // union of the 4 rows' column ranges
    const int hi = LOWER ? (r0 + RW - 1 < m - 1 ? r0 + RW - 1 : m - 1) + 1 : m;
    for (int c0 = lo; c0 < hi; c0 += 32 * CH) {
      double a[RW][CH];
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const int r = r0 + k;
        const double* row = M + (size_t)r * ldr;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int c = c0 + q * 32 + lnx();
          const bool in = r < m && c < hi && (LOWER ? c <= r : c >= r);
          a[k][q] = in ? row[c] : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int c = c0 + q * 32 + lnx();
        const double x = c < hi ? v[c] : 0.0;
#pragma unroll
        for (int k = 0; k < RW; ++k) acc[k] = fma(a[k][q], x, acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const double t = warp_sum(acc[k]);
      if (lnx() == 0 && r0 + k < m) out[r0 + k] = t;
    }
  }
  __syncthreads();
}

// u = W^T s through the stored transpose (lower), d = W u
static __device__ __forceinline__ void wt_mv(const double* Wt, int ldr, int m, const double* s, double* u) {
  tri_mv<true>(Wt, ldr, m, s, u);
}
static __device__ __forceinline__ void w_mv(const double* W, int ldr, int m, const double* u, double* d) {
  tri_mv<false>(W, ldr, m, u, d);
}

// chol_delete's LINPACK rank-1 update of the trailing block (factor.cuh
// chol_update_shift) fused with the same Givens sequence on the inverse: step
// p rotates W's column so + p with the extra column X (the deleted row's
// column of W), W <- W G_p^T.  Whole CTA.
static __device__ void chol_update_shift_w(double* R, double* W, double* Wt, int ldr, int so, int dof, int mt,
                                           double* w, double* X, double* sc) {
  for (int p = 0; p < mt; ++p) {
    if (tix() == 0) {
      const double rkk = R[(size_t)(so + p) * ldr + so + p];
      const double r = hypot(rkk, w[p]);
      sc[0] = r / rkk;
      sc[1] = w[p] / rkk;
      sc[2] = r;
      sc[3] = rkk / r;
      sc[4] = w[p] / r;
    }
    __syncthreads();
    const double c = sc[0], s = sc[1];
    for (int j = p + tix(); j < mt; j += NTHR) {
      double row;
      if (j == p) row = sc[2];
      else {
        row = (R[(size_t)(so + p) * ldr + so + j] + s * w[j]) / c;
        w[j] = c * w[j] - s * row;
      }
      R[(size_t)(dof + p) * ldr + dof + j] = row;
    }
    const double cg = sc[3], sg = sc[4];
    const int col = so + p;
    for (int i = tix(); i <= col; i += NTHR) {
      const double wa = Wt[(size_t)col * ldr + i], xb = X[i];
      const double v = cg * wa + sg * xb;
      W[(size_t)i * ldr + col] = v;
      Wt[(size_t)col * ldr + i] = v;
      X[i] = -sg * wa + cg * xb;
    }
    __syncthreads();
  }
}

template <class TA>
__device__ __forceinline__ void homotopy_body(const HomArgs& a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Ctx E;
  __shared__ HomV V;
  __shared__ double tile[32 * 32];
  __shared__ double sc[8];
  const DictV<TA> D = dict_view<TA>(a.D);
  double* ov = smem;
  T0 {
    ctx_init(E, D.d, D.n, D.ext, a.g.nb);
    ctx_bind(E, a.g, smem);
    E.prof = a.prof;
    E.sh = ov + HOM_OV * a.wmax;
    const ell1_state_t* st = a.st;
    V.phase = st->phase;
    V.status = ELL1_OK; V.conv = 0; V.quit = 0; V.steps = 0; V.note = 0;
    V.it = 0; V.passes = 0; V.m = 0;
    if (V.phase != 0) {
      V.it = st->iterations; V.m = st->rot[0]; V.note = st->rot[1];
      V.lam = st->scal[H_LAM]; V.lam0 = st->scal[H_LAM0]; V.floor = st->scal[H_FLOOR];
      V.passes = st->scal[H_PASSES];
    }
  }
  __syncthreads();
  const Panel<TA> PN = setup_panel<TA>(E, D, nullptr, 0);
  const int Wm = a.wmax;
  const double* b = a.b;
  const double s_ext = D.s;
  const int ldr = a.mmax;
  double* X = ov;
  double* Cc = ov + Wm;
  double* Wv = ov + 2 * Wm;
  double* MK = ov + 3 * Wm;    // support mask (1.0 / 0.0)
  double* T = ov + 4 * Wm;     // scratch (d_I on owned support / x_I)
  const int64_t N = D.n + (D.ext ? D.d : 0);
  double* zs = E.sh + 512;     // CTA-0 solves: z vector (mmax doubles) past the reduction scratch
  double* us = zs + ldr;       // second CTA-0 vector (mmax doubles)

  // dot of the owned column k with a replicated d-vector (A column or s e_i)
  auto col_dot = [&](int k, const double* vec) -> double {
    // called by a full warp; returns the warp sum on every lane
    if (k >= E.w) return s_ext * ldcg(vec + E.r0 + (k - E.w));
    const TA* col = PN.gl + (int64_t)k * D.ld;
    double acc = 0.0;
    for (int64_t i = lnx(); i < D.ld; i += 32) acc = fma((double)col[i], ldcg(vec + i), acc);
    return warp_sum(acc);
  };

  // W = R^{-1} rebuilt column-parallel over the grid (after a dense
  // refactorisation): CTA b solves R[0:j+1, 0:j+1] w = e_j for j = b, b + nb, ...
  auto rebuild_w = [&](int m) {
    for (int j = E.b; j < m; j += E.nb) {
      for (int p = tix(); p <= j; p += NTHR) zs[p] = (p == j) ? 1.0 : 0.0;
      __syncthreads();
      trsv_R(a.R, ldr, j + 1, zs, tile);
      for (int p = tix(); p <= j; p += NTHR) {
        a.W[(size_t)p * ldr + j] = zs[p];
        a.Wt[(size_t)j * ldr + p] = zs[p];
      }
      __syncthreads();
    }
  };

  if (V.phase == 0) {
    // c = A^T b, lambda0 = ||c||_inf, first atom (homotopy.py:142-177)
    {
      const double* rs[1] = {b};
      double* os[1] = {Cc};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    double v[3] = {0.0, 0.0, 0.0};
    for_owned(E, [&](int k) {
      if (k >= E.w) Cc[k] = s_ext * b[E.r0 + (k - E.w)];
      X[k] = 0.0; MK[k] = 0.0;
      a.posof[gcol(E, D.n, k)] = -1;
      v[0] = nmax(v[0], fabs(Cc[k]));
    });
    for (int64_t i = E.r0 + tix(); i < E.r1; i += NTHR) v[1] += b[i] * b[i];
    if (!allreduce<2>(E, *reinterpret_cast<double(*)[2]>(v), 1u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    // argmax |c| (first index on ties, numpy argmax)
    double amax[2] = {INFINITY, INFINITY};
    {
      const double lam0 = v[0];
      for_owned(E, [&](int k) {
        if (fabs(Cc[k]) == lam0) amax[0] = fmin(amax[0], (double)gcol(E, D.n, k));
      });
      double am1[1] = {-amax[0]};
      if (!allreduce<1>(E, am1, 1u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      amax[0] = -am1[0];
    }
    T0 {
      V.lam0 = v[0];
      const double bn = sqrt(v[1]);
      if (V.lam0 <= a.target || V.lam0 == 0.0) {          // homotopy.py:161-166
        const double lamr = pymax(V.lam0, a.target);
        if (E.b == 0) {
          a.trace[0] = 0.0; a.trace[1] = 0.5 * bn * bn; a.trace[2] = bn; a.trace[3] = 0.0;
          a.st->ntrace = 1;
        }
        V.lam = lamr;
        V.status = ELL1_ZERO_DATA; V.conv = 1; V.quit = 1;
      } else {
        V.lam = V.lam0;
        V.floor = pymax(a.target, 1e-12 * V.lam0);
        V.ip = (int)amax[0];
        V.m = 0;
      }
    }
    __syncthreads();
    if (V.quit) goto out;
    // first atom: R = [sqrt(a_j0 . a_j0)]
    {
      const int j0 = V.ip;
      // copy the column into colv (owner), then everyone dots
      for_owned(E, [&](int k) {
        if (gcol(E, D.n, k) == j0) MK[k] = 1.0;
      });
      const bool own = (j0 >= E.c0 && j0 < E.c1) || (D.ext && j0 >= D.n && j0 - D.n >= E.r0 && j0 - D.n < E.r1);
      if (own) {
        if (j0 < D.n) {
          const TA* col = D.A + (int64_t)j0 * D.ld;
          for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (double)col[i];
        } else {
          for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (i == j0 - D.n) ? s_ext : 0.0;
        }
      }
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    if (E.b == 0) {
      double q[1] = {0.0};
      for (int64_t i = tix(); i < D.ld; i += NTHR) { const double c = ldcg(a.colv + i); q[0] += c * c; }
      block_reduce<1>(E, q, 0u);
      T0 {
        if (!(q[0] > 0.0)) { V.status = ELL1_NOT_PD; }
        a.R[0] = sqrt(q[0]);
        a.W[0] = 1.0 / a.R[0];
        a.Wt[0] = a.W[0];
        a.sup[0] = V.ip;
        a.posof[V.ip] = 0;
        V.m = 1;
      }
    }
    T0 V.m = 1;
    __syncthreads();
    T0 V.phase = 1;
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
  } else {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      X[k] = a.x_out[j]; Cc[k] = a.c_out[j]; MK[k] = a.posof[j] >= 0 ? 1.0 : 0.0;
    });
    __syncthreads();
  }

  while (true) {
    mark(E, 7);
    mark(E, -1);
    T0 V.quit = V.it >= a.max_iter || (a.max_steps > 0 && V.steps >= a.max_steps);
    __syncthreads();
    if (V.quit) break;
    T0 { V.it++; V.steps++; V.ridge = 0; V.fail = 0; }
    // ---- sgn(c_I) in support order (owners write), then CTA 0 solves the direction
    for_owned(E, [&](int k) {
      if (MK[k] != 0.0) {
        const int p = a.posof[gcol(E, D.n, k)];
        a.sgn[p] = sgn(Cc[k]);
      }
    });
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    mark(E, 0);
    {
      bool retry = true;
      while (retry) {
        retry = false;
        if (E.b == 0) {
          const int m = V.m;
          for (int p = tix(); p < m; p += NTHR) zs[p] = ldcg(a.sgn + p);
          __syncthreads();
          wt_mv(a.Wt, ldr, m, zs, us);                       // u = W^T sgn = R^{-T} sgn
          w_mv(a.W, ldr, m, us, zs);                         // d = W u
          for (int p = tix(); p < m; p += NTHR) {
            a.dI[p] = zs[p];
            a.dfull[a.sup[p]] = zs[p];
          }
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        mark(E, 1);
        // v = A_I d_I (support-sparse panel GEMV)
        for_owned(E, [&](int k) { T[k] = (MK[k] != 0.0) ? ldcg(a.dfull + gcol(E, D.n, k)) : 0.0; });
        __syncthreads();
        {
          const double* xs[1] = {T};
          panel_gemv<TA, 1>(E, D, PN, xs);   // zero coefficients -> zero contribution
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        gather_slice<0, 1, 0>(E, nullptr, 0u, D.ld, {nullptr}, [&](int64_t i, const double* sums, const double*) {
          double v = sums[0];
          if (D.ext) v = v + s_ext * T[E.w + (int)(i - E.r0)];
          a.Vd[i] = v;
        });
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        mark(E, 2);
        // w = A^T v; drift ||w_I - sgn||, ||sgn||; step lengths (homotopy.py:78-105)
        {
          const double* rs[1] = {a.Vd};
          double* os[1] = {Wv};
          panel_gemv_t<TA, 1>(E, D, PN, rs, os);
        }
        __syncthreads();
        double s[8] = {0, 0, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
        {
          const double lam = V.lam;
          const double floor = 1e-10 * pymax(lam, 1e-30);
          double bp1 = INFINITY, bi1 = INFINITY, bp2 = INFINITY, bi2 = INFINITY, bm = INFINITY, bmi = INFINITY;
          for_owned(E, [&](int k) {
            if (k >= E.w) Wv[k] = s_ext * a.Vd[E.r0 + (k - E.w)];
            const double j = (double)gcol(E, D.n, k);
            const double ck = Cc[k], wk = Wv[k];
            if (MK[k] != 0.0) {
              const int p = a.posof[(int64_t)j];
              const double sg = ldcg(a.sgn + p);
              const double e = wk - sg;
              s[0] += e * e;
              s[1] += sg * sg;
              const double dk = ldcg(a.dfull + (int64_t)j);
              const double r = -X[k] / dk;
              if (isfinite(r) && r > 0.0 && (r < bm || (r == bm && j < bmi))) { bm = r; bmi = j; }
            } else {
              const double r1 = (lam - ck) / (1.0 - wk);
              const double r2 = (lam + ck) / (1.0 + wk);
              if (isfinite(r1) && r1 > floor && (r1 < bp1 || (r1 == bp1 && j < bi1))) { bp1 = r1; bi1 = j; }
              if (isfinite(r2) && r2 > floor && (r2 < bp2 || (r2 == bp2 && j < bi2))) { bp2 = r2; bi2 = j; }
            }
          });
          // (value, index) pairs reduced as max of negatives in two passes
          s[2] = -bp1; s[3] = -bp2; s[4] = -bm;
          s[5] = -bi1; s[6] = -bi2; s[7] = -bmi;
          double v3[3] = {s[2], s[3], s[4]};
          double sums2[2] = {s[0], s[1]};
          block_reduce<2>(E, sums2, 0u);
          block_reduce<3>(E, v3, 0x7u);
          // indices attaining the block minimum
          double i3[3] = {-INFINITY, -INFINITY, -INFINITY};
          if (bp1 == -v3[0]) i3[0] = -bi1;
          if (bp2 == -v3[1]) i3[1] = -bi2;
          if (bm == -v3[2]) i3[2] = -bmi;
          block_reduce<3>(E, i3, 0x7u);
          double pubv[8] = {sums2[0], sums2[1], v3[0], v3[1], v3[2], i3[0], i3[1], i3[2]};
          publish<8>(E, pubv);
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        {
          // gather: sums, min values; then the lowest index among CTAs attaining the min
          double G8[8];
          gather<8>(E, G8, 0xFCu);
          // CTAs whose block min != global min must not contribute their index: recheck
          // by publishing again (cheap, scalars only)
          double fix[3] = {-INFINITY, -INFINITY, -INFINITY};
          if (wpx() == 0) {
            // warp 0 only (thread 0 consumes it); every load of a round is in flight at once
            constexpr int QU = 4;
            double best[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int q0 = 0; q0 < E.nb; q0 += 32 * QU) {
              double val[QU][3], idx[QU][3];
#pragma unroll
              for (int u = 0; u < QU; ++u) {
                const int q = q0 + 32 * u + lnx();
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                  val[u][t] = q < E.nb ? ldcg(published(E, 8, q, 2 + t)) : NAN;
                  idx[u][t] = q < E.nb ? ldcg(published(E, 8, q, 5 + t)) : -INFINITY;
                }
              }
#pragma unroll
              for (int u = 0; u < QU; ++u)
#pragma unroll
                for (int t = 0; t < 3; ++t)
                  if (val[u][t] == G8[2 + t]) best[t] = nmax(best[t], idx[u][t]);
            }
#pragma unroll
            for (int t = 0; t < 3; ++t) fix[t] = warp_max(best[t]);
          }
          T0 {
            V.drift = sqrt(G8[0]);
            V.sgnn = sqrt(G8[1]);
            const double g1 = -G8[2], g2 = -G8[3];
            const double i1 = -fix[0], i2 = -fix[1];
            // gamma+: r1's min, replaced by r2's only when strictly smaller (homotopy.py:90-95)
            V.gp = g1; V.ip = isfinite(g1) ? (int)i1 : -1;
            if (g2 < V.gp) { V.gp = g2; V.ip = (int)i2; }
            V.gm = -G8[4];
            V.im = isfinite(V.gm) ? (int)(-fix[2]) : -1;
            V.passes += 2;
            const double tol = 1e-6 * pymax(1.0, V.sgnn);             // homotopy.py:50
            if (!(V.drift <= tol) && V.ridge != 2) V.fail = 1;   // 2: ridge factor, no check
          }
          __syncthreads();
        }
        if (V.fail) {
          // dense refactorisation of A_I^T A_I (homotopy.py:53-64): G built column by column
          const int m = V.m;
          for (int p = 0; p < m; ++p) {
            // column sup[p] into colv
            const int64_t jp = a.sup[p];
            const bool own = (jp >= E.c0 && jp < E.c1) || (D.ext && jp >= D.n && jp - D.n >= E.r0 && jp - D.n < E.r1);
            if (own) {
              if (jp < D.n) {
                const TA* col = D.A + jp * D.ld;
                for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (double)col[i];
              } else {
                for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (i == jp - D.n) ? s_ext : 0.0;
              }
            }
            if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
            for (int k = wpx(); k < E.W; k += NWARP) {
              if (MK[k] == 0.0) continue;
              const double g = col_dot(k, a.colv);
              if (lnx() == 0) a.G[(size_t)a.posof[gcol(E, D.n, k)] * ldr + p] = g;
            }
            if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          }
          if (E.b == 0) {
            const bool ok = V.ridge ? false : dense_chol(a.G, a.R, ldr, m, sc);
            if (!ok || V.ridge) {
              // ridge (homotopy.py:118-125): G + 1e-12 max(tr G, 1) I
              T0 {
                double tr = 0.0;
                for (int p = 0; p < m; ++p) tr += a.G[(size_t)p * ldr + p];
                sc[3] = 1e-12 * pymax(tr, 1.0);
              }
              __syncthreads();
              for (int p = tix(); p < m; p += NTHR) a.G[(size_t)p * ldr + p] += sc[3];
              __syncthreads();
              const bool ok2 = dense_chol(a.G, a.R, ldr, m, sc);
              T0 { if (!ok2) V.status = ELL1_NOT_PD; V.note = 1; sc[2] = 2.0; }
            } else {
              T0 sc[2] = 1.0;
            }
            __syncthreads();
            T0 a.st->rot[6] = (int)sc[2];
          }
          if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          T0 { V.ridge = ((volatile int*)a.st->rot)[6]; V.fail = 0; }
          rebuild_w(m);
          if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          if (V.status != ELL1_OK) goto out;
          T0 if (E.b == 0) a.st->rot[7] = a.st->rot[7] + 1;  // refactorisation count (diagnostics)
          retry = true;
        }
      }
    }
    mark(E, 3);
    // ---- event (homotopy.py:192-223)
    T0 {
      const double ge = fmin(V.gp, V.gm);
      const double cap = V.lam - a.target;
      if (cap <= ge) { V.finish = 1; V.remove = 0; sc[0] = cap; }
      else {
        V.finish = 0;
        V.remove = V.gm <= V.gp + 1e-12;
        sc[0] = V.remove ? V.gm : V.gp;
      }
      V.d2 = sc[0];
    }
    __syncthreads();
    {
      const double gamma = V.d2;
      for_owned(E, [&](int k) {
        if (MK[k] != 0.0) X[k] = X[k] + gamma * ldcg(a.dfull + gcol(E, D.n, k));
      });
      if (!V.finish && V.remove) {
        for_owned(E, [&](int k) {
          if (gcol(E, D.n, k) == V.im) { X[k] = 0.0; MK[k] = 0.0; }
        });
      }
    }
    __syncthreads();
    mark(E, 4);
    if (!V.finish) {
      if (V.remove) {
        // chol_delete(pos) on CTA 0 (numerics.py:140-158)
        if (E.b == 0) {
          const int m = V.m;
          const int pos = a.posof[V.im];
          const int mt = m - pos - 1;
          // X = W[:, pos] (rows <= pos): the column the rotations fold away
          for (int i = tix(); i < m; i += NTHR) us[i] = i <= pos ? a.Wt[(size_t)pos * ldr + i] : 0.0;
          // top rows of R: columns > pos shift left (two parallel passes through G)
          for (int t = tix(); t < pos * mt; t += NTHR) {
            const int i = t / mt, j = pos + 1 + (t - i * mt);
            a.G[(size_t)i * ldr + j - 1] = a.R[(size_t)i * ldr + j];
          }
          __syncthreads();
          for (int t = tix(); t < pos * mt; t += NTHR) {
            const int i = t / mt, j = pos + (t - i * mt);
            a.R[(size_t)i * ldr + j] = a.G[(size_t)i * ldr + j];
          }
          __syncthreads();
          if (mt > 0) {
            for (int j = tix(); j < mt; j += NTHR) zs[j] = a.R[(size_t)pos * ldr + pos + 1 + j];
            __syncthreads();
            chol_update_shift_w(a.R, a.W, a.Wt, ldr, pos + 1, pos, mt, zs, us, sc);
          }
          // W' = (W G^T) without row pos and column pos (entries with j' >= pos change)
          {
            const int m1 = m - 1, wc = m1 - pos;          // new columns pos .. m-2
            for (int t = tix(); t < m1 * wc; t += NTHR) {
              const int i = t / wc, j = pos + (t - i * wc);
              if (j >= i) a.G[(size_t)i * ldr + j] = a.W[(size_t)(i + (i >= pos ? 1 : 0)) * ldr + j + 1];
            }
            __syncthreads();
            for (int t = tix(); t < m1 * wc; t += NTHR) {
              const int i = t / wc, j = pos + (t - i * wc);
              if (j >= i) {
                const double v = a.G[(size_t)i * ldr + j];
                a.W[(size_t)i * ldr + j] = v;
                a.Wt[(size_t)j * ldr + i] = v;             // rows pos.. of Wt (row j, col i)
              }
            }
            __syncthreads();
          }
          // support list / positions
          T0 {
            for (int p = pos; p < m - 1; ++p) {
              const int j = a.sup[p + 1];
              a.sup[p] = j;
              a.posof[j] = p;
            }
            a.posof[V.im] = -1;
            a.dfull[V.im] = 0.0;
          }
        }
        T0 V.m = V.m - 1;
        mark(E, 5);
      } else {
        // chol_append (numerics.py:115-137): gcol = A_I^T a_ip, diag = a_ip . a_ip
        const int64_t ip = V.ip;
        const bool own = (ip >= E.c0 && ip < E.c1) || (D.ext && ip >= D.n && ip - D.n >= E.r0 && ip - D.n < E.r1);
        if (own) {
          if (ip < D.n) {
            const TA* col = D.A + ip * D.ld;
            for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (double)col[i];
          } else {
            for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (i == ip - D.n) ? s_ext : 0.0;
          }
          for_owned(E, [&](int k) { if (gcol(E, D.n, k) == ip) MK[k] = 1.0; });
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        for (int k = wpx(); k < E.W; k += NWARP) {
          if (MK[k] == 0.0 || gcol(E, D.n, k) == ip) continue;
          const double g = col_dot(k, a.colv);
          if (lnx() == 0) a.gcol[a.posof[gcol(E, D.n, k)]] = g;
        }
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        if (E.b == 0) {
          const int m = V.m;
          double q[1] = {0.0};
          for (int64_t i = tix(); i < D.ld; i += NTHR) { const double c = ldcg(a.colv + i); q[0] += c * c; }
          block_reduce<1>(E, q, 0u);
          for (int p = tix(); p < m; p += NTHR) us[p] = ldcg(a.gcol + p);
          __syncthreads();
          wt_mv(a.Wt, ldr, m, us, zs);                      // r = R^{-T} g = W^T g
          double uu[1] = {0.0};
          for (int p = tix(); p < m; p += NTHR) uu[0] += zs[p] * zs[p];
          block_reduce<1>(E, uu, 0u);
          const double d2 = q[0] - uu[0];
          if (d2 > 0.0 && m < ldr) {
            // inverse column: W[:m, m] = -(W r) / rho, W[m, m] = 1 / rho
            w_mv(a.W, ldr, m, zs, us);
            const double rho = sqrt(d2);
            for (int p = tix(); p < m; p += NTHR) {
              const double v = -us[p] / rho;
              a.W[(size_t)p * ldr + m] = v;
              a.Wt[(size_t)m * ldr + p] = v;
            }
            T0 { a.W[(size_t)m * ldr + m] = 1.0 / rho; a.Wt[(size_t)m * ldr + m] = 1.0 / rho; }
            for (int p = tix(); p < m; p += NTHR) a.R[(size_t)p * ldr + m] = zs[p];
            T0 {
              a.R[(size_t)m * ldr + m] = sqrt(d2);
              a.sup[m] = (int)ip;
              a.posof[ip] = m;
              sc[3] = 0.0;
            }
          } else {
            T0 {
              sc[3] = 1.0;                                    // NotPositiveDefinite -> ridge
              if (m >= ldr) V.status = ELL1_DEGENERATE;
              a.sup[m] = (int)ip;
              a.posof[ip] = m;
            }
          }
          __syncthreads();
          T0 V.ridge = sc[3] != 0.0 ? 3 : 0;
        }
        T0 V.m = V.m + 1;
        // broadcast the ridge decision (CTA 0 -> all) through state scratch
        if (E.b == 0 && threadIdx.x == 0) a.st->rot[5] = V.ridge == 3 ? 1 : 0;
        if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
        T0 V.ridge = ((volatile int*)a.st->rot)[5];
        __syncthreads();
        if (V.status != ELL1_OK) goto out;
        if (V.ridge) {
          // _ridge_factor over the grown support (homotopy.py:220-222)
          const int m = V.m;
          for (int p = 0; p < m; ++p) {
            const int64_t jp = a.sup[p];
            const bool own2 = (jp >= E.c0 && jp < E.c1) || (D.ext && jp >= D.n && jp - D.n >= E.r0 && jp - D.n < E.r1);
            if (own2) {
              if (jp < D.n) {
                const TA* col = D.A + jp * D.ld;
                for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (double)col[i];
              } else {
                for (int64_t i = tix(); i < D.ld; i += NTHR) a.colv[i] = (i == jp - D.n) ? s_ext : 0.0;
              }
            }
            if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
            for (int k = wpx(); k < E.W; k += NWARP) {
              if (MK[k] == 0.0) continue;
              const double g = col_dot(k, a.colv);
              if (lnx() == 0) a.G[(size_t)a.posof[gcol(E, D.n, k)] * ldr + p] = g;
            }
            if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          }
          if (E.b == 0) {
            T0 {
              double tr = 0.0;
              for (int p = 0; p < m; ++p) tr += a.G[(size_t)p * ldr + p];
              sc[3] = 1e-12 * pymax(tr, 1.0);
            }
            __syncthreads();
            for (int p = tix(); p < m; p += NTHR) a.G[(size_t)p * ldr + p] += sc[3];
            __syncthreads();
            const bool ok2 = dense_chol(a.G, a.R, ldr, m, sc);
            T0 { if (!ok2) V.status = ELL1_NOT_PD; V.note = 1; }
          }
          if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
          rebuild_w(m);
          T0 V.ridge = 0;
        }
        mark(E, 6);
      }
    }
    // ---- fresh residual and correlations (homotopy.py:224-234)
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double s2[2] = {0.0, 0.0};                            // l1, max|x|
      for_owned(E, [&](int k) { s2[0] += fabs(X[k]); s2[1] = nmax(s2[1], fabs(X[k])); T[k] = X[k]; });
      block_reduce<2>(E, s2, 0x2u);
      publish<2>(E, s2);
      const double* xs[1] = {T};
      panel_gemv<TA, 1>(E, D, PN, xs);
    }
    if (!grid_sync(E)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
    {
      double S2[2];
      double q[1] = {0.0};
      const double* aux[1] = {b};
      gather_slice<2, 1, 1>(E, S2, 0x2u, D.ld, aux, [&](int64_t i, const double* sums, const double* au) {
        double ax = sums[0];
        if (D.ext) ax = ax + s_ext * T[E.w + (int)(i - E.r0)];
        const double r = au[0] - ax;
        a.Rd[i] = r;
        q[0] += r * r;
      });
      T0 { V.l1 = S2[0]; V.top = S2[1]; }
      if (!allreduce<1>(E, q, 0u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 V.rr = q[0];
    }
    {
      const double* rs[1] = {a.Rd};
      double* os[1] = {Cc};
      panel_gemv_t<TA, 1>(E, D, PN, rs, os);
    }
    __syncthreads();
    {
      const double cut = 1e-10 * pymax(V.top, 1.0);
      double s2[2] = {0.0, 0.0};                            // max|c|, support count
      for_owned(E, [&](int k) {
        if (k >= E.w) Cc[k] = s_ext * a.Rd[E.r0 + (k - E.w)];
        s2[0] = nmax(s2[0], fabs(Cc[k]));
        if (fabs(X[k]) > cut) s2[1] += 1.0;
      });
      if (!allreduce<2>(E, s2, 0x1u)) { T0 V.status = ELL1_ERR_TIMEOUT; goto out; }
      T0 {
        V.passes += 2;
        double lam;
        if (V.finish) lam = a.target;
        else {
          const double lam_step = V.lam - V.d2;
          const double lam_emp = s2[0];
          if (fabs(lam_emp - lam_step) <= 1e-9 * pymax(lam_step, 1e-30) || V.m == 0) lam = lam_step;
          else lam = lam_emp;                                // homotopy.py:227-234
        }
        V.lam = lam;
        const double rn = sqrt(V.rr);
        if (E.b == 0) {
          double* tr = a.trace + (size_t)(V.it - 1) * 4;
          tr[0] = (double)V.it; tr[1] = 0.5 * rn * rn + lam * V.l1; tr[2] = rn; tr[3] = s2[1];
          if (a.lam_path) a.lam_path[V.it - 1] = lam;
        }
        if (V.finish || lam <= V.floor) V.conv = 1;
      }
      __syncthreads();
      if (V.conv) break;
    }
  }
  T0 if (!V.conv && V.status == ELL1_OK && V.it < a.max_iter && a.max_steps > 0) V.status = ELL1_RUNNING;
  __syncthreads();

out:
  __syncthreads();
  if (V.status != ELL1_ERR_TIMEOUT) {
    for_owned(E, [&](int k) {
      const int64_t j = gcol(E, D.n, k);
      a.x_out[j] = X[k];
      a.c_out[j] = Cc[k];
    });
    if (E.b == 0) {
      const int m = V.m;
      if (a.sup_out)
        for (int p = tix(); p < m; p += NTHR) a.sup_out[p] = a.sup[p];
      if (a.R_out)
        for (int64_t t = tix(); t < (int64_t)m * m; t += NTHR) {
          const int64_t i = t / m, j = t - i * m;
          a.R_out[t] = j >= i ? a.R[i * a.mmax + j] : 0.0;
        }
    }
  }
  if (E.b == 0 && threadIdx.x == 0) {
    ell1_state_t* st = a.st;
    st->status = V.status;
    st->phase = (V.status == ELL1_RUNNING) ? 1 : 2;
    st->iterations = V.it;
    st->converged = V.conv;
    if (V.status != ELL1_ZERO_DATA) st->ntrace = V.it;
    st->rot[0] = V.m; st->rot[1] = V.note;
    st->scal[H_LAM] = V.lam; st->scal[H_LAM0] = V.lam0; st->scal[H_FLOOR] = V.floor;
    st->scal[H_PASSES] = V.passes;
  }
}

template <class TA>
__global__ void __launch_bounds__(NTHR, 1) homotopy_kernel(const __grid_constant__ HomArgs a) {
  homotopy_body<TA>(a);
}

}  // namespace ell1

using namespace ell1;

static int hom_mmax(const ell1_dict_t* D) {
  const int64_t N = ncols_of(D);
  int64_t m = D->d + 256;
  if (m > N) m = N;
  return (int)m;
}

extern "C" size_t ell1_homotopy_workspace(const ell1_dict_t* D, int32_t blocks) {
  if (!dict_ok(D)) return 0;
  const int nb = pick_blocks(D->n, blocks);
  const int64_t N = ncols_of(D);
  const int64_t m = hom_mmax(D);
  return grid_bytes(nb, D->d, 1) + 4 * align_up(m * m * 8, 256) + 2 * align_up(m * 4, 256) +
         align_up(N * 4, 256) + 3 * align_up(m * 8, 256) + align_up(N * 8, 256) +
         3 * align_up(D->ld * 8, 256) + 4096;
}

extern "C" int ell1_homotopy_capacity(const ell1_dict_t* D) { return dict_ok(D) ? hom_mmax(D) : 0; }

static int homotopy_setup(const ell1_dict_t* D, const double* b, double target_lambda,
                             int32_t max_iter, const ell1_homotopy_out_t* O, const ell1_io_t* io, int nb, HomArgs& a, SmemPlan& sp) {
  if (!dict_ok(D) || !b || !O || !O->c || !io || !io->state || !io->trace || !io->x) return ELL1_ERR_ARG;
  double* c_out = O->c;
  if (!(target_lambda >= 0) || max_iter < 1) return ELL1_ERR_ARG;
  const int64_t N = ncols_of(D);
  a.D = to_raw(D);
  a.b = b;
  a.target = target_lambda;
  a.max_iter = max_iter;
  a.mmax = hom_mmax(D);
  const int64_t m = a.mmax;
  Carve cv(io->workspace, io->workspace_bytes);
  if (!carve_grid(cv, a.g, nb, D->d, 1)) return ELL1_ERR_ARG;
  a.R = cv.take<double>(m * m); a.W = cv.take<double>(m * m); a.Wt = cv.take<double>(m * m);
  a.G = cv.take<double>(m * m);
  a.sup = cv.take<int>(m); a.posof = cv.take<int>(N);
  a.sgn = cv.take<double>(m); a.dI = cv.take<double>(m); a.gcol = cv.take<double>(m);
  a.dfull = cv.take<double>(N);
  a.colv = cv.take<double>(D->ld); a.Vd = cv.take<double>(D->ld); a.Rd = cv.take<double>(D->ld);
  if (!cv.ok) return ELL1_ERR_ARG;
  a.st = io->state;
  a.trace = io->trace;
  a.x_out = io->x;
  a.c_out = c_out;
  a.lam_path = O->lam_path;
  a.sup_out = O->support;
  a.R_out = O->factor;
  a.max_steps = io->max_steps;
  a.prof = io->phase_ns;
  sp = plan_smem(a.D, nb, HOM_OV, 8, false);
  // CTA-0 solves keep z and u (2 x mmax doubles) in the scratch area past 512 reduction doubles
  if (sp.scratch < 512 + 2 * m) { sp.bytes += (size_t)(512 + 2 * m - sp.scratch) * 8; sp.scratch = 512 + 2 * m; }
  a.g.shcap = sp.scratch;
  a.g.panel_bytes = 0;
  a.wmax = sp.wmax;
  return ELL1_OK;
}

extern "C" int ell1_homotopy(const ell1_dict_t* D, const double* b, double target_lambda,
                             int32_t max_iter, const ell1_homotopy_out_t* O, const ell1_io_t* io,
                             void* stream) {
  if (!dict_ok(D) || !io) return ELL1_ERR_ARG;
  const int nb = pick_blocks(D->n, io->blocks);
  HomArgs a;
  SmemPlan sp;
  const int rc0 = homotopy_setup(D, b, target_lambda, max_iter, O, io, nb, a, sp);
  if (rc0 != ELL1_OK) return rc0;
  const int64_t N = ncols_of(D);
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(a.dfull, 0, N * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  for (double* p : {a.colv, a.Vd, a.Rd})
    if (cudaMemsetAsync(p, 0, D->ld * 8, s) != cudaSuccess) return ELL1_ERR_CUDA;
  return (D->dtype == ELL1_F64) ? coop_launch(homotopy_kernel<double>, nb, sp.bytes, s, a, a.g.bar)
                                : coop_launch(homotopy_kernel<float>, nb, sp.bytes, s, a, a.g.bar);

}

namespace ell1 {
template <class TA>
struct HomRun {
  static __device__ void run(const HomArgs& a) { homotopy_body<TA>(a); }
  static __device__ void reset(const HomArgs& a, int lane) {
    reset_bar(a.g.bar, lane);
    const int64_t N = a.D.n + (a.D.ext ? a.D.d : 0);
    for (int64_t i = lane; i < N; i += 32) a.dfull[i] = 0.0;
    for (int64_t i = lane; i < a.D.ld; i += 32) { a.colv[i] = 0.0; a.Vd[i] = 0.0; a.Rd[i] = 0.0; }
  }
};
static_assert(sizeof(HomArgs) <= ELL1_GROUP_ARG_BYTES, "HomArgs too large for the group scratch");
}  // namespace ell1

// the path streams the dictionary (no resident panel); the breakpoint
// bookkeeping is CTA 0's, so one CTA per solve
int32_t ell1_homotopy_group_team_impl(const ell1_dict_t* D) { return dict_ok(D) ? 1 : 0; }

extern "C" int ell1_homotopy_group(const ell1_group_t* G, const double* target_lambda, int32_t max_iter,
                                   const ell1_homotopy_out_t* O, void* stream) {
  if (!G || (G->count > 0 && (!target_lambda || !O))) return ELL1_ERR_ARG;
  ell1_group_t H = *G;
  if (H.team <= 0) H.team = 1;
  return run_group<HomArgs, HomRun>(&H, HOM_OV, 8, 0, [&](int i, int nb, HomArgs& a, SmemPlan& sp) {
    return homotopy_setup(&G->dicts[i], G->b[i], target_lambda[i], max_iter, &O[i], &G->io[i], nb, a, sp);
  }, stream);
}
