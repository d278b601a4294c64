// Grid-barrier variants on the B200 (diagnostics only): the engine's counter
// barrier (one release-add on a shared word, acquire polls) vs a flag array
// (each CTA release-stores its epoch in its own word; one warp acquire-polls
// all nb words).  Each round also writes an 8 KB partial per CTA and reads a
// 148 x 8-double region after the barrier, like the panel GEMV exchange.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bar_bench.cu -o build/bar_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1007_3753_b200/csrc/engine.cuh"

using namespace ell1;

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>   // 0 counter, 1 flags (acquire polls), 2 flags (relaxed polls + one fence)
__device__ __forceinline__ void bar(unsigned long long* ctr, unsigned* flags, unsigned epoch, int nb) {
  __syncthreads();
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      red_release_add(ctr, 1ULL);
      const unsigned long long target = (unsigned long long)epoch * nb;
      while (ld_acquire(ctr) < target) {}
    }
  } else {
    if (threadIdx.x == 0) st_release_u32(flags + blockIdx.x, epoch);
    if (threadIdx.x < 32) {
      bool done = false;
      while (!done) {
        bool mine = true;
        for (int c = threadIdx.x; c < nb; c += 32) {
          const unsigned f = MODE == 1 ? ld_acquire_u32(flags + c) : ld_relaxed_u32(flags + c);
          mine = mine && (f >= epoch);
        }
        done = __all_sync(0xffffffffu, mine);
      }
      if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}

template <int MODE, bool DATA>
__global__ void __launch_bounds__(NTHR, 1) k_bar(int iters, unsigned long long* ctr, unsigned* flags, double* part,
                                                 double* out) {
  const int nb = gridDim.x, b = blockIdx.x;
  double acc = 0.0;
  for (int i = 1; i <= iters; ++i) {
    if (DATA) {
      // 1024 partial rows of this CTA, slice-major: owner o gets rows [8o, 8o+8)
      double* dst = part + (size_t)(i & 1) * nb * nb * 8;
      for (int r = threadIdx.x; r < 8 * nb; r += NTHR) {
        const int o = r >> 3, k = r & 7;
        dst[(size_t)o * nb * 8 + b * 8 + k] = acc + r;
      }
    }
    bar<MODE>(ctr, flags, (unsigned)i, nb);
    if (DATA) {
      const double* src = part + (size_t)(i & 1) * nb * nb * 8 + (size_t)b * nb * 8;
      double s = 0.0;
      for (int t = threadIdx.x; t < nb * 8; t += NTHR) s += __ldcg(src + t);
      acc += warp_sum(s) * 1e-30;
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int MODE, bool DATA>
float run(int nb, int iters, unsigned long long* ctr, unsigned* flags, double* part, double* out) {
  cudaMemset(ctr, 0, 64);
  cudaMemset(flags, 0, 4096);
  k_bar<MODE, DATA><<<nb, NTHR>>>(10, ctr, flags, part, out);
  cudaDeviceSynchronize();
  cudaMemset(ctr, 0, 64);
  cudaMemset(flags, 0, 4096);
  cudaEvent_t a, e;
  cudaEventCreate(&a); cudaEventCreate(&e);
  cudaEventRecord(a);
  k_bar<MODE, DATA><<<nb, NTHR>>>(iters, ctr, flags, part, out);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, a, e);
  return ms * 1e6f / iters;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* ctr; cudaMalloc(&ctr, 64);
  unsigned* flags; cudaMalloc(&flags, 4096);
  double* part; cudaMalloc(&part, (size_t)2 * 160 * 160 * 8 * 8);
  double* out; cudaMalloc(&out, 64);
  const int N = 20000;
  for (int nb : {32, 74, 148}) {
    if (nb > sms) continue;
    printf("nb=%3d  barrier only: counter %6.0f ns  flags/acq %6.0f ns  flags/relaxed+fence %6.0f ns\n", nb,
           run<0, false>(nb, N, ctr, flags, part, out), run<1, false>(nb, N, ctr, flags, part, out),
           run<2, false>(nb, N, ctr, flags, part, out));
    printf("nb=%3d  with exchange: counter %6.0f ns  flags/acq %6.0f ns  flags/relaxed+fence %6.0f ns\n", nb,
           run<0, true>(nb, N, ctr, flags, part, out), run<1, true>(nb, N, ctr, flags, part, out),
           run<2, true>(nb, N, ctr, flags, part, out));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
