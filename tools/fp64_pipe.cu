// FP64-pipe throughput on the B200 (diagnostics): cvt.f64.f32 (F2F) and DFMA
// per SM per clock, alone and mixed, 1 CTA x 1024 threads per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_pipe.cu -o /tmp/fp64_pipe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024) k(int iters, float seed, double* out) {
  float f[8];
  double d[8];
  for (int i = 0; i < 8; ++i) { f[i] = seed + threadIdx.x + i; d[i] = f[i]; }
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { d[i] += (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }   // F2F (+DADD)
      if (MODE == 1) d[i] = fma(d[i], 1.0000001, 0.5);                                          // DFMA
      if (MODE == 2) d[i] = fma((double)f[i], d[i], 0.5);                                        // F2F + DFMA
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i] + f[i];
  if (s == 12345.0) out[1] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0);
}

// dependent-chain latency: one warp, each op waits on the previous result
template <int MODE>
__global__ void lat(int iters, double seed, double* out) {
  double d = seed + threadIdx.x;
  float f = (float)seed;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) d = d + 1.0000001;                    // DADD
    if (MODE == 1) d = fma(d, 1.0000001, 0.5);           // DFMA
    if (MODE == 2) { d = (double)f + d; f = (float)d; }  // F2F + DADD + F2F back
    if (MODE == 3) d += __shfl_xor_sync(0xffffffffu, d, 1);   // SHFL + DADD
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / iters; out[1] = d; }
}

int main() {
  double* out;
  cudaMalloc(&out, 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  const char* names[3] = {"F2F.F64.F32 (+DADD)", "DFMA", "F2F + DFMA"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<sms, 1024>>>(iters, 1.5f, out);
      if (m == 1) k<1><<<sms, 1024>>>(iters, 1.5f, out);
      if (m == 2) k<2><<<sms, 1024>>>(iters, 1.5f, out);
    }
    cudaDeviceSynchronize();
    double cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    const double ops = 1024.0 * iters * 8;                       // per SM (one CTA per SM)
    printf("%-22s %6.2f lane-ops / clk / SM (x%s per element)\n", names[m], ops / cyc, m == 0 ? "2: F2F+DADD" : m == 2 ? "2" : "1");
  }
  const char* ln[4] = {"DADD", "DFMA", "F2F.F64+DADD+F2F.F32", "SHFL.BFLY x2 + DADD"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) lat<0><<<1, 32>>>(100000, 1.5, out);
      if (m == 1) lat<1><<<1, 32>>>(100000, 1.5, out);
      if (m == 2) lat<2><<<1, 32>>>(100000, 1.5, out);
      if (m == 3) lat<3><<<1, 32>>>(100000, 1.5, out);
    }
    cudaDeviceSynchronize();
    double c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("latency %-24s %6.1f cycles per dependent step\n", ln[m], c);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
