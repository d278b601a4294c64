// kernels_misc.cu — dictionary build (layout conversion) and the device
// equivalents of the reference's native seam ell1._accel
// (_accel/_fastkernels.pyx:14-78): soft threshold, l-inf box projection,
// LINPACK rank-1 Cholesky update / downdate.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include "../../include/ell1_b200.h"

namespace {

// row-major float64 (d x n) -> column-major TA (ld x n), zero padded rows
template <class TA>
__global__ void dict_build_kernel(const double* __restrict__ in, int64_t d, int64_t n, int64_t ld,
                                  TA* __restrict__ out) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + tx;
    tile[r][tx] = (i < d && j < n) ? in[i * n + j] : 0.0;
  }
  __syncthreads();
  for (int c = ty; c < 32; c += 8) {
    const int64_t j = j0 + c, i = i0 + tx;
    if (j < n && i < ld) out[j * ld + i] = (TA)tile[tx][c];
  }
}

__global__ void soft_kernel(const double* __restrict__ u, double a, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = u[i];
    out[i] = x > a ? x - a : (x < -a ? x + a : 0.0);
  }
}

__global__ void box_kernel(const double* __restrict__ z, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = z[i];
    out[i] = x > 1.0 ? 1.0 : (x < -1.0 ? -1.0 : x);
  }
}

// One CTA walks the pivots in order; threads sweep the row to the right.
// sign > 0: update (hypot); sign < 0: downdate (status = pivot + 1 on loss of PD).
__global__ void chol_rank1_kernel(double* R, double* v, int64_t m, int sign, int32_t* status) {
  __shared__ double sc, ss;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  for (int64_t k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      const double rkk = R[k * m + k];
      const double vk = v[k];
      double r;
      if (sign > 0) {
        r = hypot(rkk, vk);
      } else {
        const double d2 = (rkk - vk) * (rkk + vk);
        if (d2 <= 0.0) { fail = (int)(k + 1); r = 0.0; }
        else r = sqrt(d2);
      }
      if (!fail) {
        sc = r / rkk;
        ss = vk / rkk;
        R[k * m + k] = r;
      }
    }
    __syncthreads();
    if (fail) break;
    const double c = sc, s = ss;
    for (int64_t j = k + 1 + threadIdx.x; j < m; j += blockDim.x) {
      const double vj = v[j];
      const double row = (sign > 0) ? (R[k * m + j] + s * vj) / c : (R[k * m + j] - s * vj) / c;
      R[k * m + j] = row;
      v[j] = c * vj - s * row;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && status) *status = fail;
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             const double* __restrict__ y, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + (y ? b * y[i] : 0.0);
}

// sum of squares, one CTA, fixed order (per-thread strided partials, tree)
__global__ void sumsq_kernel(int64_t n, const double* __restrict__ x, double* out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" int ell1_dict_build(const double* A, int64_t d, int64_t n, int64_t ld, int32_t dtype,
                               void* out, void* stream) {
  if (!A || !out || d < 1 || n < 1 || ld < d || ld % 32) return ELL1_ERR_ARG;
  if ((ld + 31) / 32 > 65535) return ELL1_ERR_ARG;
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((ld + 31) / 32));
  dim3 block(32, 8);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == ELL1_F64)
    dict_build_kernel<double><<<grid, block, 0, s>>>(A, d, n, ld, (double*)out);
  else if (dtype == ELL1_F32)
    dict_build_kernel<float><<<grid, block, 0, s>>>(A, d, n, ld, (float*)out);
  else
    return ELL1_ERR_ARG;
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_soft_threshold(const double* u, double a, double* out, int64_t n, void* stream) {
  if (!(a >= 0.0) || n < 0) return ELL1_ERR_ARG;
  if (n == 0) return ELL1_OK;
  soft_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(u, a, out, n);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_project_box_linf(const double* z, double* out, int64_t n, void* stream) {
  if (n < 0) return ELL1_ERR_ARG;
  if (n == 0) return ELL1_OK;
  box_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(z, out, n);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_chol_update(double* R, double* v, int64_t m, int32_t* status, void* stream) {
  if (m < 0) return ELL1_ERR_ARG;
  if (m == 0) return cudaMemsetAsync(status, 0, 4, (cudaStream_t)stream) == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  chol_rank1_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(R, v, m, 1, status);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_chol_downdate(double* R, double* v, int64_t m, int32_t* status, void* stream) {
  if (m < 0) return ELL1_ERR_ARG;
  if (m == 0) return cudaMemsetAsync(status, 0, 4, (cudaStream_t)stream) == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
  chol_rank1_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(R, v, m, -1, status);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out,
                          void* stream) {
  if (n < 0 || !x || !out) return ELL1_ERR_ARG;
  if (n == 0) return ELL1_OK;
  axpby_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, a, x, b, y, out);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_sumsq(int64_t n, const double* x, double* out, void* stream) {
  if (n < 0 || !out || (n > 0 && !x)) return ELL1_ERR_ARG;
  sumsq_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(n, x, out);
  return cudaGetLastError() == cudaSuccess ? ELL1_OK : ELL1_ERR_CUDA;
}

extern "C" int ell1_device_sms(int32_t device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

extern "C" const char* ell1_version(void) { return "ell1_b200 0.1.0 sm_100a"; }
