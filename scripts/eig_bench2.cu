// cuSOLVER small symmetric eigensolvers / Cholesky at the preconditioner's sizes (warm, best of 5).
// nvcc -O3 -arch=sm_100a eig_bench2.cu -lcusolver -lcublas -o eig_bench2
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#include <cusolverDn.h>

static std::vector<double> decaying(int n, unsigned seed) {
  // A = V diag(lam) V^T, lam_i = 10^(7 - 10 i / n), V from Gram-Schmidt of a Gaussian block
  std::mt19937_64 g(seed); std::normal_distribution<double> nd;
  std::vector<double> V((size_t)n * n);
  for (auto& x : V) x = nd(g);
  for (int j = 0; j < n; ++j) {
    double* vj = &V[(size_t)j * n];
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < j; ++i) {
        const double* vi = &V[(size_t)i * n]; double d = 0; for (int r = 0; r < n; ++r) d += vi[r] * vj[r];
        for (int r = 0; r < n; ++r) vj[r] -= d * vi[r];
      }
    double s = 0; for (int r = 0; r < n; ++r) s += vj[r] * vj[r]; s = 1 / std::sqrt(s);
    for (int r = 0; r < n; ++r) vj[r] *= s;
  }
  std::vector<double> A((size_t)n * n, 0.0);
  for (int k = 0; k < n; ++k) {
    const double lam = std::pow(10.0, 7.0 - 10.0 * k / n);
    const double* v = &V[(size_t)k * n];
    for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) A[(size_t)j * n + i] += lam * v[i] * v[j];
  }
  return A;
}

int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cusolverDnParams_t p; cusolverDnCreateParams(&p);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int n : {256, 266, 522, 1034}) {
    std::vector<double> A = decaying(n, 1);
    double *dA, *dB, *dW; int* info;
    cudaMalloc(&dA, 8 * (size_t)n * n); cudaMalloc(&dB, 8 * (size_t)n * n); cudaMalloc(&dW, 8 * n); cudaMalloc(&info, 4);
    cudaMemcpy(dB, A.data(), 8 * (size_t)n * n, cudaMemcpyHostToDevice);
    size_t dws = 0, hws = 0, d2 = 0, h2 = 0, d3 = 0, h3 = 0;
    cusolverDnXsyevd_bufferSize(h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW,
                                CUDA_R_64F, &dws, &hws);
    cusolverStatus_t sb = cusolverDnXsyevBatched_bufferSize(h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n,
                                      CUDA_R_64F, dW, CUDA_R_64F, &d2, &h2, 1);
    int64_t meig = 0; double vl = 0, vu = 0; const int64_t k = n - 10;
    cusolverDnXsyevdx_bufferSize(h, p, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n,
                                 &vl, &vu, n - k + 1, n, &meig, CUDA_R_64F, dW, CUDA_R_64F, &d3, &h3);
    size_t dmax = std::max({dws, d2, d3, (size_t)8}), hmax = std::max({hws, h2, h3, (size_t)8});
    void* dwork; cudaMalloc(&dwork, dmax); std::vector<char> hwork(hmax);
    int lwp = 0; cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, &lwp);
    double* pw; cudaMalloc(&pw, 8 * (size_t)std::max(lwp, 1));
    std::vector<double> ref(n);
    const char* names[] = {"Xsyevd", "XsyevBatched(1)", "Xsyevdx(top n-10)", "Dpotrf", "Xpotrf"};
    for (int alg = 0; alg < 5; ++alg) {
      if (alg == 1 && sb != CUSOLVER_STATUS_SUCCESS) { printf("n=%d XsyevBatched unsupported (%d)\n", n, (int)sb); continue; }
      float best = 1e9; cusolverStatus_t st = CUSOLVER_STATUS_SUCCESS;
      for (int r = 0; r < 5; ++r) {
        cudaMemcpy(dA, dB, 8 * (size_t)n * n, cudaMemcpyDeviceToDevice);
        if (alg >= 3) {  // make it SPD-ish: A + I already SPD (lam >= 1e-3)
        }
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        if (alg == 0) st = cusolverDnXsyevd(h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW,
                                       CUDA_R_64F, dwork, dmax, hwork.data(), hmax, info);
        else if (alg == 1) st = cusolverDnXsyevBatched(h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n,
                                             CUDA_R_64F, dW, CUDA_R_64F, dwork, dmax, hwork.data(), hmax, info, 1);
        else if (alg == 2) st = cusolverDnXsyevdx(h, p, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F,
                                        dA, n, &vl, &vu, n - k + 1, n, &meig, CUDA_R_64F, dW, CUDA_R_64F, dwork, dmax, hwork.data(), hmax, info);
        else if (alg == 3) st = cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, pw, lwp, info);
        else st = cusolverDnXpotrf(h, p, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dwork, dmax, hwork.data(), hmax, info);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
      }
      int hinfo = 0; cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
      double err = 0;
      if (alg <= 2) {
        std::vector<double> w(n); cudaMemcpy(w.data(), dW, 8 * n, cudaMemcpyDeviceToHost);
        if (alg == 0) ref = w;
        const int off = alg == 2 ? n - (int)meig : 0;
        for (int i = 0; i < (alg == 2 ? (int)meig : n); ++i) err = std::max(err, std::fabs(w[i] - ref[i + off]) / std::fabs(ref[n - 1]));
      }
      printf("n=%d %-20s %8.3f ms  status %d info %d  eig diff/max %.2e\n", n, names[alg], best, (int)st, hinfo, err);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dW); cudaFree(dwork); cudaFree(info); cudaFree(pw);
  }
  return 0;
}
