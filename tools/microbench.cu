// Calibration of the persistent-grid primitives on the B200 (diagnostics only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. tools/microbench.cu -o build/microbench
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1007_3753_b200/csrc/engine.cuh"

using namespace ell1;

__global__ void __launch_bounds__(NTHR, 1) k_sync(int iters, double* out) {
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) { __syncthreads(); acc += 1.0; }
  if (acc < 0) out[0] = acc;
}

__global__ void __launch_bounds__(NTHR, 1) k_breduce(int iters, double* out) {
  __shared__ Ctx E;
  __shared__ double sh[1024];
  if (threadIdx.x == 0) E.sh = sh;
  __syncthreads();
  double v[7];
  for (int k = 0; k < 7; ++k) v[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
    block_reduce<7>(E, v, 1u << 3);
    for (int k = 0; k < 7; ++k) v[k] = v[k] * 1e-3 + threadIdx.x;
  }
  if (v[0] < 0) out[0] = v[0];
}

__global__ void __launch_bounds__(NTHR, 1) k_grid(int iters, unsigned long long* bar, int* abort, double* out) {
  __shared__ Ctx E;
  if (threadIdx.x == 0) { E.nb = gridDim.x; E.b = blockIdx.x; E.epoch = 0; E.nbar = 0; E.bar = bar; E.abort = abort; }
  __syncthreads();
  for (int i = 0; i < iters; ++i)
    if (!grid_sync(E)) break;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)E.nbar;
}

// dependent chain of L2 loads (pointer chase through a buffer written earlier)
__global__ void k_chase(const int* nxt, int iters, int* out) {
  int p = threadIdx.x * 33;
  for (int i = 0; i < iters; ++i) p = __ldcg(nxt + p);
  out[threadIdx.x] = p;
}

__global__ void k_timer(int iters, unsigned long long* out) {
  unsigned long long t0 = gtimer(), t = t0, mn = ~0ull;
  for (int i = 0; i < iters; ++i) {
    unsigned long long t1 = gtimer();
    if (t1 != t && t1 - t < mn) mn = t1 - t;
    t = t1;
  }
  out[0] = t - t0;
  out[1] = mn;
}

static float timeit(void (*launch)(void*), void* ctx) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch(ctx);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  launch(ctx);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  const int N = 20000;
  double* out; cudaMalloc(&out, 64);
  unsigned long long* bar; cudaMalloc(&bar, 64);
  int* abort_; cudaMalloc(&abort_, 64);
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

  struct C { int n; double* out; unsigned long long* bar; int* ab; int nb; } c{N, out, bar, abort_, sms};
  float ms;
  ms = timeit([](void* p) { C* c = (C*)p; k_sync<<<c->nb, NTHR>>>(c->n, c->out); }, &c);
  printf("__syncthreads (512 thr)      : %7.1f ns\n", ms * 1e6 / N);
  ms = timeit([](void* p) { C* c = (C*)p; k_breduce<<<c->nb, NTHR>>>(c->n, c->out); }, &c);
  printf("block_reduce<7>              : %7.1f ns\n", ms * 1e6 / N);
  for (int nb : {148, 64, 16}) {
    c.nb = nb;
    ms = timeit([](void* p) {
      C* c = (C*)p;
      cudaMemset(c->bar, 0, 64); cudaMemset(c->ab, 0, 64);
      void* args[] = {&c->n, &c->bar, &c->ab, &c->out};
      cudaLaunchCooperativeKernel((const void*)k_grid, dim3(c->nb), dim3(NTHR), args, 0, 0);
    }, &c);
    printf("grid_sync (%3d CTAs)         : %7.1f ns\n", nb, ms * 1e6 / N);
  }
  // L2 latency
  const int M = 1 << 20;
  int* nxt; cudaMalloc(&nxt, M * 4);
  int* h = (int*)malloc(M * 4);
  for (int i = 0; i < M; ++i) h[i] = (int)(((long long)i * 7919 + 4099) % M);
  cudaMemcpy(nxt, h, M * 4, cudaMemcpyHostToDevice);
  int* o2; cudaMalloc(&o2, 4096);
  struct D { int* nxt; int* o; } dd{nxt, o2};
  ms = timeit([](void* p) { D* d = (D*)p; k_chase<<<1, 32>>>(d->nxt, 20000, d->o); }, &dd);
  printf("dependent L2 load (ldcg)     : %7.1f ns\n", ms * 1e6 / 20000);
  unsigned long long* t; cudaMalloc(&t, 64);
  k_timer<<<1, 1>>>(100000, t);
  unsigned long long ht[2];
  cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
  printf("globaltimer read             : %7.1f ns (min nonzero delta %llu ns)\n", (double)ht[0] / 100000, ht[1]);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("clock rate attr %d kHz, SMs %d, err %s\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
