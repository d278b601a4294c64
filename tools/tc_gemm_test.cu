// Standalone check of the 3xTF32 tcgen05 GEMM (csrc/tc_gemm.cu) against an fp64
// host reference and cuBLAS SIMT SGEMM, with timings at the batched shapes.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1007_3753_b200/csrc \
//        tools/tc_gemm_test.cu paper_1007_3753_b200/csrc/tc_gemm.cu -lcublas -o tools/tc_gemm_test
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "tc_gemm.cuh"
#ifdef TC3_TIMING
namespace ell1 { void tc3_debug(unsigned long long* out, bool reset); }
#endif

static float rna(float x) {  // host tf32 round-to-nearest-away
  unsigned u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

// device time per call with the launches replayed from a CUDA graph (as the solvers
// run them): no host enqueue cost in the figure
template <class F>
static float graph_ms(int reps, F&& call) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int r = 0; r < reps; ++r) call(st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(st);
  cudaEventDestroy(a); cudaEventDestroy(b);
  return ms / reps;
}

int main(int argc, char** argv) {
  cublasHandle_t h;
  cublasCreate(&h);
  const int shapes[][3] = {{100, 37, 50},     {128, 64, 32},     {1024, 1024, 1216}, {1216, 1024, 1024},
                           {1024, 2048, 1216}, {512, 1024, 2048}, {2048, 1024, 512},  {1024, 1024, 2240},
                           {1216, 300, 1024}, {8192, 8192, 8192}};
  int bad = 0;
  int si = -1;
  for (auto& sh : shapes) {
    ++si;
    if (argc > 1 && atoi(argv[1]) != si) continue;
    const int M = sh[0], N = sh[1], K = sh[2];
    const int64_t lda = (K + 3) / 4 * 4, ldb = lda, ldc = getenv("TC3_LDC_ODD") ? M + 5 : (M + 31) / 32 * 32;
    std::vector<float> A((size_t)M * lda, 0.f), B((size_t)N * ldb, 0.f);
    srand(M * 7 + N * 13 + K);
    for (int i = 0; i < M; ++i)
      for (int k = 0; k < K; ++k) A[(size_t)i * lda + k] = (float)rand() / RAND_MAX - 0.5f;
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < K; ++k) B[(size_t)j * ldb + k] = (float)rand() / RAND_MAX - 0.3f;
    std::vector<float> Ah(A.size()), Al(A.size()), Bh(B.size()), Bl(B.size());
    for (size_t i = 0; i < A.size(); ++i) { Ah[i] = rna(A[i]); Al[i] = rna(A[i] - Ah[i]); }
    for (size_t i = 0; i < B.size(); ++i) { Bh[i] = rna(B[i]); Bl[i] = rna(B[i] - Bh[i]); }
    float *dA, *dAh, *dAl, *dB, *dBh, *dBl, *dC, *dC2;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dAh, A.size() * 4); cudaMalloc(&dAl, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dBh, B.size() * 4); cudaMalloc(&dBl, B.size() * 4);
    cudaMalloc(&dC, (size_t)ldc * N * 4); cudaMalloc(&dC2, (size_t)ldc * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dAh, Ah.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dAl, Al.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBh, Bh.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBl, Bl.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xFF, (size_t)ldc * N * 4);
#ifdef TC3_TIMING
    {
      unsigned long long dbg[16];
      ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dB, ldb, dC, ldc, 0);
      cudaDeviceSynchronize();
      ell1::tc3_debug(dbg, true);
      for (int r = 0; r < 5; ++r) ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dB, ldb, dC, ldc, 0);
      cudaDeviceSynchronize();
      ell1::tc3_debug(dbg, true);
      const double ctas = (double)dbg[6], nkb = (K + 31) / 32;
      printf("timing per CTA per k-block (cycles): prod-wait-empty %.0f mma-wait-tempty %.0f mma-wait-conv %.0f "
             "drain-wait-tfull %.0f split-wait-full %.0f | CTA total %.0f cyc (%.0f per kb)\n",
             dbg[0] / ctas / nkb, dbg[1] / ctas / nkb, dbg[2] / ctas / nkb, dbg[3] / ctas / nkb, dbg[4] / ctas / nkb,
             dbg[5] / ctas, dbg[5] / ctas / nkb);
      for (int r = 0; r < 5; ++r) ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dBh, ldb, dC, ldc, 0, dBl);
      cudaDeviceSynchronize();
      ell1::tc3_debug(dbg, true);
      const double ctp = (double)dbg[6];
      printf("pre-split: prod-wait-empty %.0f mma-wait-tempty %.0f mma-wait-full %.0f drain-wait-tfull %.0f "
             "| CTA total %.0f cyc (%.0f per kb) ctas/launch %.0f\n",
             dbg[0] / ctp / nkb, dbg[1] / ctp / nkb, dbg[2] / ctp / nkb, dbg[3] / ctp / nkb, dbg[5] / ctp,
             dbg[5] / ctp / nkb, ctp / 5);
    }
#endif
    bool ok = ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dB, ldb, dC, ldc, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (!ok || e != cudaSuccess) {
      printf("%dx%dx%d: launch ok=%d err=%s\n", M, N, K, ok, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> Cg((size_t)ldc * N);
    cudaMemcpy(Cg.data(), dC, Cg.size() * 4, cudaMemcpyDeviceToHost);
    // SIMT reference: C2 = A (row-major => op T on a K x M column-major) * B
    const float one = 1.f, zero = 0.f;
    cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, dA, (int)lda, dB, (int)ldb, &zero, dC2, (int)ldc);
    cudaDeviceSynchronize();
    std::vector<float> Cs((size_t)ldc * N);
    cudaMemcpy(Cs.data(), dC2, Cs.size() * 4, cudaMemcpyDeviceToHost);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    double etc = 0, esimt = 0;
    const int samples = (M * (int64_t)N <= 200000) ? M * N : 4000;
    for (int t = 0; t < samples; ++t) {
      int i, j;
      if (samples == M * N) { i = t % M; j = t / M; }
      else { i = (int)(((int64_t)t * 7919) % M); j = (int)(((int64_t)t * 104729) % N); }
      double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) {
        double p = (double)A[(size_t)i * lda + k] * B[(size_t)j * ldb + k];
        s += p; sa += fabs(p);
      }
      etc = fmax(etc, fabs(Cg[(size_t)j * ldc + i] - s) / sa);
      esimt = fmax(esimt, fabs(Cs[(size_t)j * ldc + i] - s) / sa);
    }
    // timings
    const int reps = M >= 8192 ? 5 : 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dB, ldb, dC, ldc, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float mt; cudaEventElapsedTime(&mt, e0, e1); mt /= reps;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
      cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, dA, (int)lda, dB, (int)ldb, &zero, dC2, (int)ldc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    // producer-split B (b = hi, b_lo = lo): must give the same bits as the in-kernel split
    std::vector<float> Cp((size_t)ldc * N);
    ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dBh, ldb, dC2, ldc, 0, dBl);
    cudaDeviceSynchronize();
    cudaMemcpy(Cp.data(), dC2, Cp.size() * 4, cudaMemcpyDeviceToHost);
    size_t ndiff = 0;
    double maxd = 0;
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < M; ++i) {
        ndiff += Cp[(size_t)j * ldc + i] != Cg[(size_t)j * ldc + i];
        maxd = fmax(maxd, fabs((double)Cp[(size_t)j * ldc + i] - Cg[(size_t)j * ldc + i]));
      }
    double epre = 0;
    for (int t = 0; t < samples; ++t) {
      int i, j;
      if (samples == M * N) { i = t % M; j = t / M; }
      else { i = (int)(((int64_t)t * 7919) % M); j = (int)(((int64_t)t * 104729) % N); }
      double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) {
        double p = (double)A[(size_t)i * lda + k] * B[(size_t)j * ldb + k];
        s += p; sa += fabs(p);
      }
      epre = fmax(epre, fabs(Cp[(size_t)j * ldc + i] - s) / sa);
    }
    const float mp = graph_ms(reps, [&](cudaStream_t st) {
      ell1::tc3_gemm(M, N, K, dAh, dAl, lda, dBh, ldb, dC2, ldc, st, dBl);
    });
    printf("        pre-split B: %8.4f ms %6.1f TF/s err %.2e, %zu entries differ from the in-kernel split (max %.2e)\n",
           mp, 2.0 * M * N * K / mp / 1e9, epre, ndiff, maxd);
    const bool pass = etc < 5e-7 && epre < 5e-7;
    bad += !pass;
    printf("%5dx%5dx%5d  tc3 %8.4f ms %6.1f TF/s err %.2e | simt %8.4f ms %6.1f TF/s err %.2e  %s\n", M, N, K, mt,
           2.0 * M * N * K / mt / 1e9, etc, ms, 2.0 * M * N * K / ms / 1e9, esimt, pass ? "OK" : "FAIL");
    cudaFree(dA); cudaFree(dAh); cudaFree(dAl); cudaFree(dB); cudaFree(dBh); cudaFree(dBl);
    cudaFree(dC); cudaFree(dC2);
  }
  printf(bad ? "FAILURES %d\n" : "ALL OK\n", bad);
  return bad != 0;
}
