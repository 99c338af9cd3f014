// Time the cuSOLVER / cuBLAS small dense calls of the preconditioner build at the
// config-2 sizes (w = 266, k = 256) in their alternatives.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a small_dense_bench.cu -lcusolver -lcublas -o small_dense_bench
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#define T0 cudaEventRecord(e0, st)
#define T1(name) do { cudaEventRecord(e1, st); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); \
  printf("%-40s n=%d  %.3f ms\n", name, n, ms / reps); } while (0)

int main() {
  cudaStream_t st; cudaStreamCreate(&st);
  cusolverDnHandle_t h; cusolverDnCreate(&h); cusolverDnSetStream(h, st);
  cublasHandle_t cb; cublasCreate(&cb); cublasSetStream(cb, st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  for (int n : {256, 266, 522}) {
    std::vector<double> A(n * n), G(n * n);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    for (auto& x : G) x = nd(g);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += G[i*n+k]*G[j*n+k]; A[i*n+j] = s + (i == j ? n : 0); }
    double *dA, *dB, *dW, *work, *dY; int* info;
    const long rows = 16384;
    cudaMalloc(&dA, 8*n*n); cudaMalloc(&dB, 8*n*n); cudaMalloc(&dW, 8*n); cudaMalloc(&info, 4 * 64);
    cudaMalloc(&dY, 8 * rows * n); cudaMemset(dY, 0, 8 * rows * n);
    cudaMemcpy(dB, A.data(), 8*n*n, cudaMemcpyHostToDevice);
    int lw = 0, lw2 = 0, lw3 = 0;
    cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, &lw);
    cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw2);
    int meig = 0;
    cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n,
                                 0, 0, 11, n, &meig, dW, &lw3);
    cudaMalloc(&work, 8 * (size_t)std::max(lw, std::max(lw2, lw3)));
    // potrf
    cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, work, lw, info);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, work, lw, info); } T1("potrf (incl. copy)");
    // copy only
    T0; for (int r = 0; r < reps; ++r) cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st); T1("copy only");
    // potrfBatched (batch 1)
    double** dptrs; cudaMalloc(&dptrs, sizeof(double*)); cudaMemcpy(dptrs, &dA, sizeof(double*), cudaMemcpyHostToDevice);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDpotrfBatched(h, CUBLAS_FILL_MODE_UPPER, n, dptrs, n, info, 1); } T1("potrfBatched(1) (incl. copy)");
    // Xpotrf
    cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
    size_t dws = 0, hws = 0;
    cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, dA, n, CUDA_R_64F, &dws, &hws);
    void* dwork; cudaMalloc(&dwork, dws + 8); std::vector<char> hwork(hws + 8);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dwork, dws, hwork.data(), hws, info); } T1("Xpotrf (incl. copy)");
    // trsm right on rows x n
    const double one = 1.0;
    T0; for (int r = 0; r < reps; ++r) cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, rows, n, &one, dA, n, dY, rows); T1("trsm right 16384 x n");
    // explicit inverse (Xtrtri) + TRMM, the TRSM alternative
    {
      cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, dA, n, work, lw, info);
      double* dR; cudaMalloc(&dR, 8*n*n);
      size_t tws = 0, thws = 0;
      cusolverDnXtrtri_bufferSize(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, dR, n, &tws, &thws);
      void* tw; cudaMalloc(&tw, tws + 8); std::vector<char> thw(thws + 8);
      double* dO; cudaMalloc(&dO, 8 * rows * n);
      T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dR, dA, 8*n*n, cudaMemcpyDeviceToDevice, st);
        cusolverDnXtrtri(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, dR, n, tw, tws, thw.data(), thws, info); } T1("Xtrtri (incl. copy)");
      T0; for (int r = 0; r < reps; ++r) cublasDtrmm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, rows, n, &one, dR, n, dY, rows, dO, rows); T1("trmm right 16384 x n");
      const double zero = 0.0;
      T0; for (int r = 0; r < reps; ++r) cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, rows, n, n, &one, dY, rows, dR, n, &zero, dO, rows); T1("gemm 16384 x n x n");
      cudaFree(dR); cudaFree(tw); cudaFree(dO);
    }
    // syevd
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw2, info); } T1("syevd (incl. copy)");
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n, 0, 0, 11, n, &meig, dW, work, lw3, info); } T1("syevdx top n-10 (incl. copy)");
    // Xsyevd
    size_t dws2 = 0, hws2 = 0;
    cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &dws2, &hws2);
    void* dwork2; cudaMalloc(&dwork2, dws2 + 8); std::vector<char> hwork2(hws2 + 8);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwork2, dws2, hwork2.data(), hws2, info); } T1("Xsyevd (incl. copy)");
    // sytrd only
    double *d, *e, *tau; cudaMalloc(&d, 8*n); cudaMalloc(&e, 8*n); cudaMalloc(&tau, 8*n);
    int lw4 = 0; cusolverDnDsytrd_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, d, e, tau, &lw4);
    double* work4; cudaMalloc(&work4, 8 * (size_t)lw4 + 8);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDsytrd(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, d, e, tau, work4, lw4, info); } T1("sytrd only (incl. copy)");
    // syevj with loose tolerance
    syevjInfo_t sj; cusolverDnCreateSyevjInfo(&sj); cusolverDnXsyevjSetTolerance(sj, 1e-13); cusolverDnXsyevjSetMaxSweeps(sj, 15);
    int lw5 = 0; cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw5, sj);
    double* work5; cudaMalloc(&work5, 8 * (size_t)lw5 + 8);
    T0; for (int r = 0; r < reps; ++r) { cudaMemcpyAsync(dA, dB, 8*n*n, cudaMemcpyDeviceToDevice, st);
      cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work5, lw5, info, sj); } T1("syevj (incl. copy)");
    cudaFree(dA); cudaFree(dB); cudaFree(dW); cudaFree(work); cudaFree(dY);
  }
  return 0;
}
