// Time cuSOLVER symmetric eigensolvers on the preconditioner's small problems.
// nvcc -O3 eig_bench.cu -lcusolver -lcublas -o eig_bench
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include <cusolverDn.h>

int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  for (int n : {256, 266, 522, 1034}) {
    std::vector<double> A(n * n);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    std::vector<double> G(n * n); for (auto& x : G) x = nd(g);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += G[i*n+k]*G[j*n+k]; A[i*n+j] = s; }
    double *dA, *dB, *dW, *work; int* info;
    cudaMalloc(&dA, 8*n*n); cudaMalloc(&dB, 8*n*n); cudaMalloc(&dW, 8*n); cudaMalloc(&info, 4);
    cudaMemcpy(dB, A.data(), 8*n*n, cudaMemcpyHostToDevice);
    int lw = 0;
    cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw);
    syevjInfo_t params; cusolverDnCreateSyevjInfo(&params); cusolverDnXsyevjSetTolerance(params, 1e-14); cusolverDnXsyevjSetMaxSweeps(params, 20);
    int lw2 = 0; cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw2, params);
    cudaMalloc(&work, 8 * (size_t)std::max(lw, lw2));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int alg = 0; alg < 2; ++alg) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaMemcpy(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        if (alg == 0) cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info);
        else cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw2, info, params);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      int sweeps = 0; if (alg == 1) cusolverDnXsyevjGetSweeps(h, params, &sweeps);
      printf("n=%d %s: %.3f ms %s\n", n, alg ? "syevj" : "syevd", best, alg ? (std::to_string(sweeps) + " sweeps").c_str() : "");
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dW); cudaFree(work); cudaFree(info);
  }
  return 0;
}
