// Probe: fp32 GEMM throughput / accuracy at the batched-solver shapes
// (SIMT SGEMM vs cuBLAS BF16x9 emulation vs TF32), standalone (system cuBLAS).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/gemm_probe.cu -lcublas -o gemm_probe
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

static void fill(std::vector<float>& v, unsigned seed) {
  srand(seed);
  for (auto& x : v) x = (float)rand() / RAND_MAX - 0.5f;
}

int main() {
  int ver = 0;
  cublasHandle_t h;
  cublasCreate(&h);
  cublasGetVersion(h, &ver);
  printf("cublas version %d\n", ver);
  const int shapes[][3] = {{1024, 1024, 1216}, {1216, 1024, 1024}, {1024, 2048, 1216}, {512, 1024, 2048},
                           {2048, 1024, 512}, {8192, 8192, 8192}};
  for (auto& sh : shapes) {
    int m = sh[0], n = sh[1], k = sh[2];
    std::vector<float> hA((size_t)m * k), hB((size_t)k * n), hC((size_t)m * n), hR((size_t)m * n);
    fill(hA, 1);
    fill(hB, 2);
    float *A, *B, *C;
    cudaMalloc(&A, hA.size() * 4);
    cudaMalloc(&B, hB.size() * 4);
    cudaMalloc(&C, hC.size() * 4);
    cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
    // fp64 reference on a few entries
    const float one = 1.f, zero = 0.f;
    cublasComputeType_t modes[3] = {CUBLAS_COMPUTE_32F, CUBLAS_COMPUTE_32F_EMULATED_16BFX9,
                                    CUBLAS_COMPUTE_32F_FAST_TF32};
    const char* names[3] = {"simt", "bf16x9", "tf32"};
    for (int mi = 0; mi < 3; ++mi) {
      cublasStatus_t st = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, A, CUDA_R_32F, m, B, CUDA_R_32F,
                                       k, &zero, C, CUDA_R_32F, m, modes[mi], CUBLAS_GEMM_DEFAULT);
      if (st != CUBLAS_STATUS_SUCCESS) {
        printf("%dx%dx%d %s: status %d\n", m, n, k, names[mi], (int)st);
        continue;
      }
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      int reps = (m >= 8192) ? 5 : 50;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r)
        cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, A, CUDA_R_32F, m, B, CUDA_R_32F, k, &zero, C,
                     CUDA_R_32F, m, modes[mi], CUBLAS_GEMM_DEFAULT);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
      double maxrel = 0;
      for (int t = 0; t < 200; ++t) {
        int i = (t * 7919) % m, j = (t * 104729) % n;
        double s = 0, sa = 0;
        for (int p = 0; p < k; ++p) {
          double prod = (double)hA[(size_t)p * m + i] * hB[(size_t)j * k + p];
          s += prod;
          sa += fabs(prod);
        }
        double e = fabs(hC[(size_t)j * m + i] - s) / sa;
        if (e > maxrel) maxrel = e;
      }
      printf("%5dx%5dx%5d %-7s %8.3f ms %7.1f TF/s  max rel err (vs sum|ab|) %.2e\n", m, n, k, names[mi], ms,
             2.0 * m * n * k / ms / 1e9, maxrel);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}
