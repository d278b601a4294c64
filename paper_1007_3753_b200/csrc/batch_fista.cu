// batch_fista.cu — FISTA over a batch of instances sharing one dictionary
// (element j equals shrinkage.fista_solve on (A, b_j), shrinkage.py:231-298).
//
// One host round = one backtracking trial of every active instance:
//   bf_step   accepted last round: KKT, support, trace, stopping rules,
//             continuation of that iteration, then the next momentum point;
//             retrying: undo the global ring rotation for this instance
//             (copies) and rebuild the momentum point from the rings; then
//             soft-threshold + backtracking reductions
//   GEMM      A X_next
//   bf_resid  r_next, F, Q: accept, or grow L and mark the instance for a retry
//   GEMM      A^T R_next  (speculative for instances that will retry)
// Instances run their own backtracking independently, so the host never
// waits for a retry decision: it reads one device counter every few rounds
// (termination / compaction of finished instances).
#include "batched.cuh"

namespace ell1 {

struct BI {                 // per-instance control state
  double L, tp, tc, lam, lam_bar, Fprev, fy, fy_next, m, tn, mn, rr, Fn, c0, bn;
  double S[7];
  int it, hist, bt, active, accepted, status, conv, orig, retry;
};

struct BFArgs {
  int64_t d, n, N, ld, ldx;
  int ext;
  double s;
  int f32;
  const double* Bm;           // ld x B (b columns)
  double* X[3];               // ldx x B
  double* G[3];               // ldx x B: g(x_k), g(x_{k-1}) and the slot the speculative A^T r_next fills
  double* R[3];               // ld x B
  double* AX;                 // raw GEMM1 output (fp64 mode) ld x B
  float* X32; float* R32; float* AX32; float* G32;   // fp32 GEMM operands
  float* X32l; float* R32l;   // the step / residual kernels write the GEMM operands pre-split (3xTF32 hi in
                              // X32 / R32, lo here: the same bits as the GEMM's in-kernel split)
  int stage;                  // bf_step stages its four input rows in shared memory by bulk copies
  float* G32r[3];             // fp32 storage without the [A, sI] block: the gradient ring IS the GEMM
                              // output (fp32 values, n x B, pitch n): no fp64 copy is written or read
  int g32ring;
  BI* inst;
  ell1_ctrl_t C;
  ell1_fista_opts_t O;
  int* counters;              // [0] retry, [1] active
  double* x_out;              // N x B0 (original order)
  int* it_out; int* conv_out; int* status_out;
  double* trace;              // optional [B0][max_iter][4]
  int ix, ixp, ixn, igx, igxp, ign, irx, irxp, irn;
};

__global__ void __launch_bounds__(BT) bf_init(const BFArgs a, const double* CT, const float* CT32, int B) {
  const int j = blockIdx.x;
  __shared__ double sh[BW * 4 + 4];
  BI& I = a.inst[j];
  const double* b = a.Bm + (int64_t)j * a.ld;
  double v[2] = {0.0, 0.0};
  for (int64_t k = threadIdx.x; k < a.N; k += BT) {
    double c;
    if (k < a.n) c = a.f32 ? (double)CT32[(int64_t)j * a.n + k] : CT[(int64_t)j * a.n + k];
    else c = a.s * b[k - a.n];
    v[0] = nmax(v[0], fabs(c));
    for (int r = 0; r < 3; ++r) a.X[r][(int64_t)j * a.ldx + k] = 0.0;
    if (a.g32ring) for (int r = 0; r < 3; ++r) a.G32r[r][(int64_t)j * a.n + k] = (float)-c;
    else for (int r = 0; r < 3; ++r) a.G[r][(int64_t)j * a.ldx + k] = -c;
  }
  for (int64_t i = threadIdx.x; i < a.ld; i += BT) {
    const double bi = i < a.d ? b[i] : 0.0;
    a.R[0][(int64_t)j * a.ld + i] = -bi;
    a.R[1][(int64_t)j * a.ld + i] = -bi;
    a.R[2][(int64_t)j * a.ld + i] = 0.0;
    v[1] += bi * bi;
  }
  cta_reduce<2>(v, 1u, sh);
  if (threadIdx.x == 0) {
    I.orig = j;
    I.c0 = v[0];
    I.bn = sqrt(v[1]);
    I.it = 0; I.hist = 0; I.bt = 0; I.accepted = 0; I.conv = 0; I.status = ELL1_OK; I.active = 1; I.retry = 0;
    I.Fprev = 0.0;
    if (I.c0 == 0.0) {                                    // shrinkage.py:245-247
      I.status = ELL1_ZERO_DATA; I.conv = 1; I.active = 0;
      if (a.trace) { double* tr = a.trace + (int64_t)j * a.C.max_iter * 4; tr[0] = 0; tr[1] = 0; tr[2] = I.bn; tr[3] = 0; }
    } else {
      I.lam_bar = (a.C.lam < 0.0) ? 1e-2 * I.c0 : a.C.lam;
      if (!(I.lam_bar > 0.0)) { I.status = ELL1_LAMBDA_NONPOS; I.active = 0; }
      I.L = a.O.exact_L ? a.O.L_exact : a.O.L0;
      I.lam = a.O.continuation ? pymax(0.9 * I.c0, I.lam_bar) : I.lam_bar;
      I.tp = I.tc = 1.0;
      I.fy = 0.5 * v[1];
    }
    if (!I.active) {
      a.it_out[j] = 0; a.conv_out[j] = I.conv; a.status_out[j] = I.status;
      for (int64_t k = 0; k < a.N; ++k) a.x_out[(int64_t)j * a.N + k] = 0.0;
    } else {
      atomicAdd(a.counters + 1, 1);
    }
  }
}

// One kernel per round before the GEMMs, run AFTER the host rotated the
// rings (x_prev <- x <- x_next, r likewise, g_x <-> g slot):
//   accepted last round -> finalise that iteration (KKT with the g_next the
//     previous A^T R GEMM produced, trace, stopping, continuation), then start
//     the next one (momentum point, prox trial)
//   rejected last round -> undo the rotation for this instance (copies), then
//     a new prox trial from the stored momentum point with the grown L
//   first round         -> first prox trial
// One prox trial element (shrinkage.py:204-207 + the backtracking / stopping
// partial sums), shared by the fused and the plain passes.
// fp32 GEMM operand element as its 3xTF32 split
__device__ __forceinline__ void st_split(float* hi, float* lo, int64_t i, float x) {
  const float h = tf32_rna(x);
  hi[i] = h;
  lo[i] = tf32_rna(x - h);
}

struct ProxAcc {
  double s[7];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < 7; ++k) s[k] = 0.0;
  }
  __device__ __forceinline__ void add(double u, double yk, double gk, double xk, bool relest, bool gtr, double gt) {
    const double dl = u - yk;
    s[0] += fabs(u);
    s[1] += gk * dl;
    s[2] += dl * dl;
    s[3] = nmax(s[3], fabs(u));
    if (relest) { const double dd = u - xk; s[4] += dd * dd; s[5] += xk * xk; }
    if (gtr) { const double e = u - gt; s[6] += e * e; }
  }
};

// UNROLL independent elements per thread and trip: all loads of a trip are
// issued before any use, so each CTA keeps UNROLL x BT loads in flight.
// bf_step is latency-bound, not bandwidth-bound: at 128 registers only two
// 256-thread CTAs fit an SM and each spends most of its life in its serial
// prologue / reduction / epilogue.  Capping it at 64 registers (four CTAs per
// SM, two elements per trip) is 1.6x faster at B = 8192 despite a few spills
// (sweep over 3-6 CTAs x 1/2/4 elements: tools/bf_variants.sh)
#ifndef BF_UNROLL
#define BF_UNROLL 2
#endif
#ifndef BF_MINB
#define BF_MINB 4
#endif
constexpr int UNROLL = BF_UNROLL;

__global__ void __launch_bounds__(BT, BF_MINB) bf_step(const BFArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW * 12 + 12];
  __shared__ double sc[6];
  __shared__ int mode;                  // 0 first trial of a new iteration, 1 retry, 2 stop
  BI& I = a.inst[j];
  if (!I.active) return;
  const int64_t o = (int64_t)j * a.ldx;
  const int64_t orr = (int64_t)j * a.ld;
  const int64_t N = a.N;
  const bool relest = a.C.stop_kind == ELL1_STOP_REL_ESTIMATE;
  const bool gtr = a.C.stop_kind == ELL1_STOP_GROUND_TRUTH;
  const double* gtj = gtr ? a.C.ground_truth + (int64_t)I.orig * N : nullptr;
  if (I.accepted && !I.retry) {
    // ---- accepted last round: finish that iteration (shrinkage.py:283-297) and,
    // in the same pass, the next iteration's first prox trial with the momentum
    // parameters it would use (they do not depend on the KKT outcome; discarded
    // when the instance stops)
    // Staged inputs (no [A, sI] block, rows 16-byte sized): one thread starts bulk
    // copies of the instance's four input rows (x_k, x_{k-1}, g(x_k), g(x_{k-1}))
    // into shared memory before anything else, so all of the CTA's bytes are in
    // flight at once at no register cost; the loop below then reads shared memory.
    extern __shared__ __align__(16) unsigned char bf_dyn[];
    __shared__ uint64_t stage_bar;
    const bool staged = a.stage;
    double* sxc = reinterpret_cast<double*>(bf_dyn);
    double* sxp = sxc + N;
    if (staged && threadIdx.x == 0) {
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t xb = (uint32_t)(N * 8), gb = a.f32 ? (uint32_t)(N * 4) : xb;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * xb + 2 * gb) : "memory");
      const void* srcs[4] = {a.X[a.ix] + o, a.X[a.ixp] + o,
                             a.f32 ? (const void*)(a.G32r[a.igx] + (int64_t)j * a.n) : (const void*)(a.G[a.igx] + o),
                             a.f32 ? (const void*)(a.G32r[a.igxp] + (int64_t)j * a.n) : (const void*)(a.G[a.igxp] + o)};
      const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(bf_dyn);
      const uint32_t dsts[4] = {dst0, dst0 + xb, dst0 + 2 * xb, dst0 + 2 * xb + gb};
      const uint32_t szs[4] = {xb, xb, gb, gb};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dsts[q]),
                     "l"(srcs[q]), "r"(szs[q]), "r"(bar)
                     : "memory");
    }
    if (threadIdx.x == 0) {
      const double tp = I.tc, tc = I.tn;
      const double tn = fista_t_next(tc);
      const double lam_n = pymax(a.O.beta * I.lam, I.lam_bar);       // shrinkage.py:297
      sc[0] = (tp - 1.0) / tc;                                       // m of the next iteration
      sc[1] = tn;
      sc[2] = lam_n / I.L;
      sc[3] = 1e-10 * pymax(I.S[3], 1.0);                           // support cut, model.py:232
      sc[4] = lam_n;
    }
    __syncthreads();
    const double m = sc[0], L = I.L, thr = sc[2], cut = sc[3], lam = I.lam;
    const double* __restrict__ xc = staged ? sxc : a.X[a.ix] + o;
    const double* __restrict__ xp = staged ? sxp : a.X[a.ixp] + o;
    double* __restrict__ xn = a.X[a.ixn] + o;
    double* __restrict__ gc = a.G[a.igx] + o;
    const double* __restrict__ gcr = staged ? sxp + N : gc;                    // g(x_k) as read (fp64 storage)
    const double* __restrict__ gxp = staged ? sxp + 2 * N : a.G[a.igxp] + o;
    const double* __restrict__ rc = a.R[a.irx] + orr;
    const bool ring32 = a.g32ring;
    const float* __restrict__ sg32 = reinterpret_cast<const float*>(sxp + N);
    const float* __restrict__ g32 =
        a.f32 ? (staged ? sg32 : (ring32 ? a.G32r[a.igx] : a.G32) + (int64_t)j * a.n) : nullptr;
    const float* __restrict__ gq32 = ring32 ? (staged ? sg32 + N : a.G32r[a.igxp] + (int64_t)j * a.n) : nullptr;
    if (staged) {
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&stage_bar);
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "BFWAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n\t"
          "@!p bra BFWAIT_%=;\n\t}" ::"r"(bar)
          : "memory");
    }
    double k5[5] = {0, 0, 0, 0, 0};
    ProxAcc P;
    P.zero();
    for (int64_t base = threadIdx.x; base < N; base += UNROLL * BT) {
      double g[UNROLL], xk[UNROLL], xq[UNROLL], gq[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t k = base + u * BT;
        if (k < N) {
          if (k < a.n) g[u] = g32 ? (double)g32[k] : gcr[k];
          else g[u] = a.s * rc[k - a.n];
          xk[u] = xc[k];
          xq[u] = xp[k];
          gq[u] = ring32 ? (double)gq32[k] : gxp[k];
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t k = base + u * BT;
        if (k >= N) continue;
        if (!ring32 && (g32 || k >= a.n)) gc[k] = g[u];
        const double c = -g[u];
        if (xk[u] != 0.0) { k5[0] = nmax(k5[0], fabs(c - lam * sgn(xk[u]))); k5[2] = 1.0; }
        else { k5[1] = nmax(k5[1], fabs(c)); k5[3] = 1.0; }
        if (fabs(xk[u]) > cut) k5[4] += 1.0;
        const double yk = xk[u] + m * (xk[u] - xq[u]);                 // shrinkage.py:270
        const double gk = (1.0 + m) * g[u] - m * gq[u];               // A^T(A y - b)
        const double un = soft1(yk - gk / L, thr);                      // shrinkage.py:204
        xn[k] = un;
        if (a.f32 && k < a.n) st_split(a.X32, a.X32l, (int64_t)j * a.ldx + k, (float)un);
        P.add(un, yk, gk, xk[u], relest, gtr, gtr ? gtj[k] : 0.0);
      }
    }
    double v[12];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = k5[k];
#pragma unroll
    for (int k = 0; k < 7; ++k) v[5 + k] = P.s[k];
    cta_reduce<12>(v, 0xFu | (1u << 8), sh);                // max: k5[0..3], prox max|u| (slot 8)
    if (threadIdx.x == 0) {
      double kkt = v[2] > 0.0 ? v[0] : 0.0;
      if (v[3] > 0.0) kkt = pymax(pymax(kkt, v[1] - lam), 0.0);
      if (a.trace) {
        double* tr = a.trace + ((int64_t)I.orig * a.C.max_iter + (I.it - 1)) * 4;
        tr[0] = (double)I.it; tr[1] = I.Fn; tr[2] = sqrt(I.rr); tr[3] = v[4];
      }
      I.hist = I.hist < 2 ? I.hist + 1 : 2;
      int done = 0;
      if (lam == I.lam_bar && kkt <= a.C.tol * I.lam_bar) done = 1;   // shrinkage.py:291-293
      else if (stop_fires(a.C.stop_kind, a.C.stop_thr, I.hist, I.Fn, I.Fprev, I.S[4], I.S[5], I.S[6],
                          a.C.gt_norm, kkt))
        done = 1;
      I.Fprev = I.Fn;
      I.tp = I.tc; I.tc = I.tn;
      if (done) I.conv = 1;
      else if (I.it >= a.C.max_iter) done = 2;
      if (done) {
        I.active = 0;
        a.it_out[I.orig] = I.it; a.conv_out[I.orig] = I.conv; a.status_out[I.orig] = ELL1_OK;
        atomicSub(a.counters + 1, 1);
      } else {
        // commit the next iteration the pass already started
        I.lam = sc[4];
        I.fy = I.fy_next;
        I.it++;
        I.bt = 0;
        I.m = sc[0];
        I.tn = sc[1];
        I.mn = (I.tc - 1.0) / I.tn;
        I.accepted = 0;
        for (int k = 0; k < 7; ++k) I.S[k] = v[5 + k];
      }
      mode = done ? 2 : 0;
    }
    __syncthreads();
    if (mode == 2) {
      double* xo = a.x_out + (int64_t)I.orig * N;
      for (int64_t k = threadIdx.x; k < N; k += BT) xo[k] = xc[k];
    }
    return;
  }
  if (I.retry) {
    for (int64_t k = threadIdx.x; k < N; k += BT) {
      a.X[a.ix][o + k] = a.X[a.ixp][o + k];
      a.X[a.ixp][o + k] = a.X[a.ixn][o + k];
      // both gradients survive a failed trial (its speculative A^T r went into the
      // ring's third slot): the retry recomputes y and A^T(A y - b) from them
      if (a.g32ring) {
        const int64_t og = (int64_t)j * a.n + k;
        a.G32r[a.igx][og] = a.G32r[a.igxp][og];
        a.G32r[a.igxp][og] = a.G32r[a.ign][og];
      } else {
        a.G[a.igx][o + k] = a.G[a.igxp][o + k];
        a.G[a.igxp][o + k] = a.G[a.ign][o + k];
      }
    }
    for (int64_t i = threadIdx.x; i < a.ld; i += BT) {
      a.R[a.irx][orr + i] = a.R[a.irxp][orr + i];
      a.R[a.irxp][orr + i] = a.R[a.irn][orr + i];
    }
    if (threadIdx.x == 0) mode = 1;
  } else if (threadIdx.x == 0) {
    mode = 0;                                              // very first trial
  }
  if (threadIdx.x == 0) {
    if (mode == 0) {                                       // a new iteration
      I.it++;
      I.bt = 0;
      I.m = (I.tp - 1.0) / I.tc;
      I.tn = fista_t_next(I.tc);
      I.mn = (I.tc - 1.0) / I.tn;
    }
    I.accepted = 0;
    sc[0] = I.m; sc[1] = I.L; sc[2] = I.lam / I.L;
  }
  __syncthreads();
  const double m = sc[0], L = sc[1], thr = sc[2];
  const double* __restrict__ x = a.X[a.ix] + o;
  const double* __restrict__ xp = a.X[a.ixp] + o;
  double* __restrict__ xn = a.X[a.ixn] + o;
  const double* __restrict__ gx = a.G[a.igx] + o;
  const double* __restrict__ gxp = a.G[a.igxp] + o;
  const float* __restrict__ gx32 = a.g32ring ? a.G32r[a.igx] + (int64_t)j * a.n : nullptr;
  const float* __restrict__ gxp32 = a.g32ring ? a.G32r[a.igxp] + (int64_t)j * a.n : nullptr;
  ProxAcc P;
  P.zero();
  // a retry (larger L) rebuilds the momentum point and its gradient from the same
  // x_k, x_{k-1}, g(x_k), g(x_{k-1}) the first trial used: the same bits, and no
  // y / g_y arrays to write on every accepted iteration
  for (int64_t k = threadIdx.x; k < N; k += BT) {
    const double xk = x[k];
    const double yk = xk + m * (xk - xp[k]);                // shrinkage.py:270
    const double gxk = gx32 ? (double)gx32[k] : gx[k], gpk = gx32 ? (double)gxp32[k] : gxp[k];
    const double gk = (1.0 + m) * gxk - m * gpk;            // A^T(A y - b)
    const double u = soft1(yk - gk / L, thr);                // shrinkage.py:204
    xn[k] = u;
    if (a.f32 && k < a.n) st_split(a.X32, a.X32l, (int64_t)j * a.ldx + k, (float)u);
    P.add(u, yk, gk, xk, relest, gtr, gtr ? gtj[k] : 0.0);
  }
  cta_reduce<7>(P.s, 1u << 3, sh);
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) I.S[k] = P.s[k];
}

__global__ void __launch_bounds__(BT) bf_resid(const BFArgs a) {
  const int j = blockIdx.x;
  __shared__ double sh[BW * 2 + 2];
  BI& I = a.inst[j];
  if (!I.active) return;
  const double mn = I.mn;
  const double* b = a.Bm + (int64_t)j * a.ld;
  const double* xn = a.X[a.ixn] + (int64_t)j * a.ldx;
  const double* rx = a.R[a.irx] + (int64_t)j * a.ld;
  double* rn = a.R[a.irn] + (int64_t)j * a.ld;
  double q[2] = {0.0, 0.0};
  for (int64_t i = threadIdx.x; i < a.d; i += BT) {
    double ax = a.f32 ? (double)a.AX32[(int64_t)j * a.ld + i] : a.AX[(int64_t)j * a.ld + i];
    if (a.ext) ax = ax + a.s * xn[a.n + i];                 // robust.py:93
    const double r = ax - b[i];                             // shrinkage.py:205
    rn[i] = r;
    if (a.f32) st_split(a.R32, a.R32l, (int64_t)j * a.ld + i, (float)r);
    q[0] += r * r;
    const double ry = (1.0 + mn) * r - mn * rx[i];
    q[1] += ry * ry;
  }
  cta_reduce<2>(q, 0u, sh);
  if (threadIdx.x == 0) {
    I.rr = q[0];
    I.Fn = 0.5 * q[0] + I.lam * I.S[0];
    bool acc;
    if (a.O.exact_L) acc = true;
    else {
      const double Qm = I.fy + I.S[1] + 0.5 * I.L * I.S[2] + I.lam * I.S[0];
      // shrinkage.py:210; float32 GEMMs accumulate in fp32, so the tie slack is
      // scaled to that precision (documented fp32 deviation, SURVEY §7 hard part 4)
      const double slack = a.f32 ? 1e-6 : 1e-12;
      acc = I.Fn <= Qm + slack * pymax(1.0, fabs(Qm));
    }
    if (acc) {
      I.accepted = 1;
      I.retry = 0;
      I.fy_next = 0.5 * q[1];
    } else {
      I.L *= a.O.eta;
      I.bt++;
      I.retry = 1;
      if (I.bt > 100) {                                     // shrinkage.py:203,213
        I.status = ELL1_BREAKDOWN; I.active = 0;
        a.it_out[I.orig] = I.it; a.conv_out[I.orig] = 0; a.status_out[I.orig] = I.status;
        atomicSub(a.counters + 1, 1);
      }
    }
  }
}

__global__ void conv_f64_f32(const double* src, float* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

// ---- compaction: keep active instances, in order, at the front
__global__ void bf_scan(BI* inst, int B, int* perm, int* newB) {
  // single CTA prefix sum over the active flags
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < B; c0 += blockDim.x) {
    const int j = c0 + threadIdx.x;
    const int act = (j < B) ? inst[j].active : 0;
    const unsigned m = __ballot_sync(0xffffffffu, act);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __shared__ int wsum[32];
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
__global__ void gather_cols(const T* src, T* dst, int64_t rows, int64_t ld, const int* perm, int B) {
  const int k = blockIdx.y;
  if (k >= B) return;
  const int64_t s = (int64_t)perm[k] * ld, d = (int64_t)k * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    dst[d + i] = src[s + i];
}

}  // namespace ell1

using namespace ell1;

static int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }

extern "C" size_t ell1_batch_fista_workspace(const ell1_dict_t* D, int32_t B) {
  if (!dict_ok(D) || B < 1) return 0;
  const int64_t N = ncols_of(D), ldx = round4(N), ld = D->ld;
  size_t s = 0;
  s += 6 * align_up(ldx * B * 8, 256) + 4 * align_up(ld * B * 8, 256);     // X, G, R, AX / Bm
  s += align_up(ld * B * 8, 256);                                           // Bm
  s += align_up((int64_t)sizeof(BI) * B, 256) * 2;
  s += align_up(ldx * B * 4, 256) * 5 + align_up(ld * B * 4, 256) * 3;       // fp32 operands (hi / lo), fp32 gradient ring
  s += align_up((ldx > ld ? ldx : ld) * B * 8, 256);                        // compaction scratch
  s += align_up(B * 4, 256) + 4096;
  if (D->dtype == ELL1_F32) s += (size_t)f32split_floats(D, (ldx > ld ? ldx : ld) * B) * 4 + 1024;
  return s;
}

extern "C" int ell1_batch_fista(const ell1_dict_t* D, const double* Bmat, int32_t B,
                                const ell1_ctrl_t* C, const ell1_fista_opts_t* O,
                                const ell1_batch_out_t* out, void* ws, size_t wsb, void* stream) {
  if (!dict_ok(D) || !Bmat || B < 1 || !C || !O || !out || !out->x || !out->iterations ||
      !out->converged || !out->status)
    return ELL1_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t N = ncols_of(D), ldx = round4(N), ld = D->ld;
  BFArgs a;
  a.d = D->d; a.n = D->n; a.N = N; a.ld = ld; a.ldx = ldx;
  a.ext = D->ext; a.s = D->ext_scale; a.f32 = D->dtype == ELL1_F32;
  a.C = *C; a.O = *O;
  Carve cv(ws, wsb);
  for (int k = 0; k < 3; ++k) a.X[k] = cv.take<double>(ldx * B);
  for (int k = 0; k < 3; ++k) a.G[k] = cv.take<double>(ldx * B);
  for (int k = 0; k < 3; ++k) a.R[k] = cv.take<double>(ld * B);
  a.AX = cv.take<double>(ld * B);
  double* Bm = cv.take<double>(ld * B);
  a.inst = cv.take<BI>(B);
  BI* inst2 = cv.take<BI>(B);
  a.X32 = cv.take<float>(ldx * B); a.G32 = cv.take<float>(ldx * B);
  a.g32ring = a.f32 && !a.ext;
  a.G32r[0] = a.G32;
  for (int k = 1; k < 3; ++k) a.G32r[k] = a.g32ring ? cv.take<float>(ldx * B) : a.G32;
  a.R32 = cv.take<float>(ld * B); a.AX32 = cv.take<float>(ld * B);
  a.X32l = cv.take<float>(ldx * B); a.R32l = cv.take<float>(ld * B);
  double* scratch = cv.take<double>((ldx > ld ? ldx : ld) * B);
  int* perm = cv.take<int>(B);
  int* ctr = cv.take<int>(8);
  if (!cv.ok) return ELL1_ERR_ARG;
  F32Split sp;
  const F32Split* spp = nullptr;
  if (a.f32) {
    if (!f32split_setup(sp, cv, D, (ldx > ld ? ldx : ld) * B, s)) return ELL1_ERR_ARG;
    spp = &sp;
  }
  a.Bm = Bm;
  a.counters = ctr;
  a.x_out = out->x; a.it_out = out->iterations; a.conv_out = out->converged; a.status_out = out->status;
  a.trace = out->trace;
  if (cudaMemcpyAsync(Bm, Bmat, ld * B * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (cudaMemsetAsync(ctr, 0, 32, s) != cudaSuccess) return ELL1_ERR_CUDA;
  if (a.f32) {
    if (cudaMemsetAsync(a.X32, 0, ldx * B * 4, s) != cudaSuccess) return ELL1_ERR_CUDA;
    if (cudaMemsetAsync(a.X32l, 0, ldx * B * 4, s) != cudaSuccess) return ELL1_ERR_CUDA;
  }
  a.ix = 0; a.ixp = 1; a.ixn = 2; a.igx = 0; a.igxp = 1; a.ign = 2; a.irx = 0; a.irxp = 1; a.irn = 2;
  // c = A^T b for every instance (GEMM), then per-instance setup
  {
    const void* Bop = Bm;
    if (a.f32) {
      float* B32 = a.R32;                                   // fp32 operand copy of b
      conv_f64_f32<<<(unsigned)((ld * B + 255) / 256), 256, 0, s>>>(Bm, B32, ld * B);
      Bop = B32;
    }
    void* CT = a.f32 ? (void*)a.G32 : (void*)scratch;      // n x B
    if (!gemm_AtR(s, D, Bop, ld, CT, D->n, B, spp)) return ELL1_ERR_CUDA;
    bf_init<<<B, BT, 0, s>>>(a, (const double*)CT, (const float*)CT, B);
  }
  // bf_step input staging: fp32 storage (24 bytes per element: 48 KB at n = 2048, four CTAs per SM still
  // fit), rows of 16-byte multiples, no [A, sI] block.  fp64 storage would need 32 bytes per element
  // (three CTAs per SM at n = 2048): measured slower at B = 1024 (92 -> 133 ms per solve in bf_step) and
  // level at B = 8192, so it keeps the direct loads (the kernel supports both).
  const size_t stage_bytes = (size_t)N * (a.f32 ? 24 : 32);
  a.stage = a.f32 && a.g32ring && !a.ext && N % 4 == 0 && stage_bytes <= 56 * 1024;
  if (const char* e = getenv("ELL1_BF_STAGE")) a.stage = a.stage && e[0] != '0';    // diagnostics
  if (a.stage && stage_bytes > 40 * 1024 &&
      cudaFuncSetAttribute(bf_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_bytes) != cudaSuccess)
    return ELL1_ERR_CUDA;
  int Bcur = B;
  int* h_ctr = host_mailbox();
  h_ctr[0] = h_ctr[1] = 0;
  // rounds between reads of the active count: a multiple of 3 (the period of
  // the x / r / g ring rotations), so R rounds leave the ring indices as they
  // were and one recorded graph per batch size replays them
  constexpr int R = 12;
  cudaStream_t ks = s;
  auto one_round = [&](BFArgs& aa) -> bool {
    // ---- finish last round's accepted iterations, then one backtracking trial each
    bf_step<<<Bcur, BT, aa.stage ? stage_bytes : 0, ks>>>(aa);
    if (!gemm_AX(ks, D, aa.f32 ? (const void*)aa.X32 : (const void*)aa.X[aa.ixn], ldx,
                 aa.f32 ? (void*)aa.AX32 : (void*)aa.AX, ld, Bcur, spp, aa.f32 ? aa.X32l : nullptr))
      return false;
    bf_resid<<<Bcur, BT, 0, ks>>>(aa);
    // g_next = A^T r_next into the g ring's free slot (speculative for retries)
    if (!gemm_AtR(ks, D, aa.f32 ? (const void*)aa.R32 : (const void*)aa.R[aa.irn], ld,
                  aa.f32 ? (void*)aa.G32r[aa.g32ring ? aa.ign : 0] : (void*)aa.G[aa.ign], aa.f32 ? D->n : ldx, Bcur, spp,
                  aa.f32 ? aa.R32l : nullptr))
      return false;
    // rotate the rings (shrinkage.py:283-284); bf_step undoes it for retrying instances
    { int t = aa.ixp; aa.ixp = aa.ix; aa.ix = aa.ixn; aa.ixn = t; }
    { int t = aa.irxp; aa.irxp = aa.irx; aa.irx = aa.irn; aa.irn = t; }
    { int t = aa.igxp; aa.igxp = aa.igx; aa.igx = aa.ign; aa.ign = t; }
    return cudaGetLastError() == cudaSuccess;
  };
  bool use_graph = true;
  if (const char* e = getenv("ELL1_BATCH_GRAPH")) use_graph = e[0] != '0';
  cudaGraphExec_t gexec = nullptr;
  struct ExecGuard {                                   // every exit path releases the graph
    cudaGraphExec_t& e;
    ~ExecGuard() { if (e) cudaGraphExecDestroy(e); }
  } gexec_guard{gexec};
  int gB = -1;
  for (;;) {
    if (cudaMemcpyAsync(h_ctr, ctr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ELL1_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ELL1_ERR_CUDA;
    const int nact = h_ctr[1];
    if (nact <= 0) break;
    if (nact < Bcur * 3 / 4 || (nact < Bcur && nact <= 64)) {
      // compact the active instances to the front of every state matrix
      bf_scan<<<1, 1024, 0, s>>>(a.inst, Bcur, perm, ctr + 2);
      bool cok = true;
      auto perm_mat = [&](double* M, int64_t rows, int64_t ldm) {
        dim3 g((unsigned)((rows + 255) / 256 < 64 ? (rows + 255) / 256 : 64), (unsigned)nact);
        gather_cols<double><<<g, 256, 0, s>>>(M, scratch, rows, ldm, perm, nact);
        cok = cok && cudaMemcpyAsync(M, scratch, ldm * nact * 8, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      };
      for (int k = 0; k < 3; ++k) perm_mat(a.X[k], N, ldx);
      if (!a.g32ring)
        for (int k = 0; k < 3; ++k) perm_mat(a.G[k], N, ldx);
      for (int k = 0; k < 3; ++k) perm_mat(a.R[k], ld, ld);
      perm_mat(Bm, ld, ld);
      // fp32 storage: g_next of the last round (the GEMM output) is still pending; without the
      // [A, sI] block all three slots of the fp32 gradient ring are state
      for (int k = 0; k < (a.g32ring ? 3 : a.f32 ? 1 : 0); ++k) {
        float* fs = reinterpret_cast<float*>(scratch);
        dim3 g((unsigned)((D->n + 255) / 256 < 64 ? (D->n + 255) / 256 : 64), (unsigned)nact);
        gather_cols<float><<<g, 256, 0, s>>>(a.G32r[k], fs, D->n, D->n, perm, nact);
        cok = cok && cudaMemcpyAsync(a.G32r[k], fs, D->n * nact * 4, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      }
      {
        const int64_t words = (int64_t)sizeof(BI) / 4;
        dim3 g(1, (unsigned)nact);
        gather_cols<int><<<g, 64, 0, s>>>((const int*)a.inst, (int*)inst2, words, words, perm, nact);
        cok = cok && cudaMemcpyAsync(a.inst, inst2, sizeof(BI) * nact, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
      }
      if (!cok || cudaGetLastError() != cudaSuccess) return ELL1_ERR_CUDA;
      Bcur = nact;
    }
    if (use_graph && gB != Bcur) {
      if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
      cudaStream_t cs = nullptr;
      cudaGraph_t g = nullptr;
      bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
      if (ok) {
        ks = cs;
        ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        if (ok) {
          BFArgs aa = a;
          for (int r = 0; r < R && ok; ++r) ok = one_round(aa);
          ok = cudaStreamEndCapture(cs, &g) == cudaSuccess && ok;
        }
        ks = s;
        cudaStreamDestroy(cs);
      }
      ok = ok && cudaGraphInstantiate(&gexec, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
      if (ok) {
        gB = Bcur;
      } else {
        gexec = nullptr;
        use_graph = false;
        cudaGetLastError();
      }
    }
    if (use_graph) {
      if (cudaGraphLaunch(gexec, s) != cudaSuccess) return ELL1_ERR_CUDA;
    } else {
      BFArgs aa = a;
      for (int r = 0; r < R; ++r)
        if (!one_round(aa)) return ELL1_ERR_CUDA;
    }
  }
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

