// factor.cuh — single-CTA dense factor kernels (upper Cholesky R^T R = G,
// row-major m x m with leading dimension ldr) shared by the Homotopy path
// (homotopy.cu), the numerics ABI (linalg.cu) and the batched Homotopy.
// numerics.py:47-158 / _fastkernels.pyx:46-78 semantics.
#pragma once
#include "engine.cuh"

namespace ell1 {

// Solve R^T z = z (in place, z in shared memory), R upper m x m row-major.
template <int NT = NTHR>
static __device__ void trsv_RT(const double* R, int ldr, int m, double* z, double* tile) {
  for (int kb = 0; kb < m; kb += 32) {
    const int nbk = min(32, m - kb);
    // stage the 32 x 32 diagonal block
    // diagonal staged as reciprocals: the serial chain multiplies instead of dividing
    for (int t = tix(); t < 32 * 32; t += NT) {
      const int i = t >> 5, j = t & 31;
      const double r = (i < nbk && j < nbk) ? R[(size_t)(kb + i) * ldr + kb + j] : 0.0;
      tile[t] = (i == j && i < nbk) ? 1.0 / r : r;
    }
    __syncthreads();
    if (wpx() == 0) {
      const int j = lnx();
      double zj = j < nbk ? z[kb + j] : 0.0;
      for (int k = 0; k < nbk; ++k) {
        double zk = __shfl_sync(0xffffffffu, zj, k);
        zk = zk * tile[k * 32 + k];
        if (j == k) zj = zk;
        if (j > k && j < nbk) zj = zj - tile[k * 32 + j] * zk;
      }
      if (j < nbk) z[kb + j] = zj;
    }
    __syncthreads();
    // trailing update: z_j -= sum_{k in block} R[k][j] z_k  (rows of R: coalesced)
    for (int j = kb + nbk + tix(); j < m; j += NT) {
      double acc = 0.0;
      for (int k = 0; k < nbk; ++k) acc = fma(R[(size_t)(kb + k) * ldr + j], z[kb + k], acc);
      z[j] = z[j] - acc;
    }
    __syncthreads();
  }
}

// Solve R d = z (in place), back substitution, blocked.
template <int NT = NTHR>
static __device__ void trsv_R(const double* R, int ldr, int m, double* z, double* tile) {
  const int nblk = (m + 31) / 32;
  for (int bb = nblk - 1; bb >= 0; --bb) {
    const int kb = bb * 32;
    const int nbk = min(32, m - kb);
    // z_B -= R[B, > B] d_{>B}: one warp per row, lanes over the row
    for (int k = wpx(); k < nbk; k += NT / 32) {
      double acc = 0.0;
      const double* row = R + (size_t)(kb + k) * ldr;
      int j = kb + nbk + lnx();
      for (; j + 96 < m; j += 128) {                          // 4 loads in flight per lane
        const double r0 = row[j], r1 = row[j + 32], r2 = row[j + 64], r3 = row[j + 96];
        acc = fma(r0, z[j], acc);
        acc = fma(r1, z[j + 32], acc);
        acc = fma(r2, z[j + 64], acc);
        acc = fma(r3, z[j + 96], acc);
      }
      for (; j < m; j += 32) acc = fma(row[j], z[j], acc);
      acc = warp_sum(acc);
      if (lnx() == 0) z[kb + k] = z[kb + k] - acc;
    }
    for (int t = tix(); t < 32 * 32; t += NT) {
      const int i = t >> 5, j = t & 31;
      const double r = (i < nbk && j < nbk) ? R[(size_t)(kb + i) * ldr + kb + j] : 0.0;
      tile[t] = (i == j && i < nbk) ? 1.0 / r : r;
    }
    __syncthreads();
    if (wpx() == 0) {
      const int i = lnx();
      double zi = i < nbk ? z[kb + i] : 0.0;
      for (int k = nbk - 1; k >= 0; --k) {
        double dk = __shfl_sync(0xffffffffu, zi, k);
        dk = dk * tile[k * 32 + k];
        if (i == k) zi = dk;
        if (i < k) zi = zi - tile[i * 32 + k] * dk;
      }
      if (i < nbk) z[kb + i] = zi;
    }
    __syncthreads();
  }
}

// LINPACK rank-1 update of the (mt x mt) trailing block read from (src row
// offset so, col offset so) and written shifted to (do, do); w consumed
// (_fastkernels.pyx:46-59 semantics).
template <int NT = NTHR>
static __device__ void chol_update_shift(double* R, int ldr, int so, int dof, int mt, double* w, double* sc) {
  for (int p = 0; p < mt; ++p) {
    if (tix() == 0) {
      const double rkk = R[(size_t)(so + p) * ldr + so + p];
      const double r = hypot(rkk, w[p]);
      sc[0] = r / rkk;
      sc[1] = w[p] / rkk;
      sc[2] = r;
    }
    __syncthreads();
    const double c = sc[0], s = sc[1];
    for (int j = p + tix(); j < mt; j += NT) {
      double row;
      if (j == p) row = sc[2];
      else {
        row = (R[(size_t)(so + p) * ldr + so + j] + s * w[j]) / c;
        w[j] = c * w[j] - s * row;
      }
      R[(size_t)(dof + p) * ldr + dof + j] = row;
    }
    __syncthreads();
  }
}

// dense Cholesky (upper, R^T R = G) of the m x m matrix in G (row-major), into R.
// Returns false when not positive definite (numpy.linalg.cholesky LinAlgError).
template <int NT = NTHR>
static __device__ bool dense_chol(const double* G, double* R, int ldr, int m, double* sc) {
  for (int k = 0; k < m; ++k) {
    // R[k][j] = (G[k][j] - sum_{i<k} R[i][k] R[i][j]) / R[k][k]
    if (tix() == 0) {
      double s = G[(size_t)k * ldr + k];
      for (int i = 0; i < k; ++i) s -= R[(size_t)i * ldr + k] * R[(size_t)i * ldr + k];
      sc[0] = s;
    }
    __syncthreads();
    if (!(sc[0] > 0.0)) return false;
    const double rkk = sqrt(sc[0]);
    for (int j = k + tix(); j < m; j += NT) {
      if (j == k) { R[(size_t)k * ldr + k] = rkk; continue; }
      double s = G[(size_t)k * ldr + j];
      for (int i = 0; i < k; ++i) s -= R[(size_t)i * ldr + k] * R[(size_t)i * ldr + j];
      R[(size_t)k * ldr + j] = s / rkk;
    }
    __syncthreads();
  }
  return true;
}

}  // namespace ell1
