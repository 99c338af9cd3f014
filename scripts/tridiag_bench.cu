// Exploration for the eigensolver: Householder tridiagonalisation of a symmetric n x n (n <= 288)
// float64 matrix on one 16-CTA cluster, rows distributed over the CTAs, ONE cluster barrier per
// column (the next column is rebuilt redundantly from the broadcast old column and w).
// Prints the time and checks trace / Frobenius invariants (eigenvalues of T are those of A).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tridiag_bench.cu -o tridiag_bench
#include <cooperative_groups.h>
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int CL = 16, T = 256, NMAX = 288, RPC = NMAX / CL;   // rows per CTA (18)

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// A row-major n x n (symmetric).  Outputs d (n), e (n-1).  Each CTA r owns rows i = r, r + CL, ...
__global__ void __launch_bounds__(T) tridiag_kernel(int n, const double* __restrict__ A, double* d, double* e) {
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double rows_raw[];    // this CTA's rows of the trailing matrix, [RPC][NMAX]
  double (*rows)[NMAX] = reinterpret_cast<double (*)[NMAX]>(rows_raw);
  __shared__ double col[2][NMAX];         // broadcast: column j (old values), double-buffered by j parity
  __shared__ double pv[2][NMAX];          // broadcast: p = A v entries (by row owner)
  __shared__ double v[NMAX], w[NMAX];
  __shared__ double red[T / 32];
  const int nr = (n - r + CL - 1) / CL;   // rows owned
  for (int q = 0; q < nr; ++q)
    for (int c = tid; c < n; c += T) rows[q][c] = A[(size_t)(r + q * CL) * n + c];
  // column 0 broadcast: every CTA writes its rows' entries of column 0 into everyone's col[0]
  __syncthreads();
  for (int q = tid; q < nr; q += T) {
    const int i = r + q * CL;
    for (int dst = 0; dst < CL; ++dst) *cl.map_shared_rank(&col[0][i], dst) = rows[q][0];
  }
  cl.sync();
  for (int j = 0; j < n - 2; ++j) {
    const int b = j & 1;
    // ---- Householder vector of col[b][j+1..n-1] (redundant in every CTA)
    double s = 0.0;
    for (int i = j + 1 + tid; i < n; i += T) s = fma(col[b][i], col[b][i], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double sig = 0.0;
    for (int k = 0; k < T / 32; ++k) sig += red[k];
    const double x0 = col[b][j + 1];
    const double alpha = -copysign(sqrt(sig), x0);
    const double vtv = sig - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    const double tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
    for (int i = tid; i < n; i += T) v[i] = (i <= j) ? 0.0 : (i == j + 1 ? x0 - alpha : col[b][i]);
    if (r == 0 && tid == 0) {
      d[j] = col[b][j];
      e[j] = alpha;
    }
    __syncthreads();
    // ---- p = tau A' v for my rows (A' = trailing rows/cols > j), and my rows' old column j+2 entries
    for (int q = warp; q < nr; q += T / 32) {
      const int i = r + q * CL;
      double acc = 0.0;
      if (i > j)
        for (int c = j + 1 + lane; c < n; c += 32) acc = fma(rows[q][c], v[c], acc);
      acc = warp_sum(acc);
      if (lane < CL && i > j) *cl.map_shared_rank(&pv[b][i], lane) = tau * acc;   // to every CTA
    }
    // old column j+1 entries are needed next step: broadcast my rows' column j+1
    for (int q = tid; q < nr; q += T) {
      const int i = r + q * CL;
      if (i > j)
        for (int dst = 0; dst < CL; ++dst) *cl.map_shared_rank(&col[b ^ 1][i], dst) = rows[q][j + 1];
    }
    cl.sync();   // the one barrier of this column
    // ---- w = p - (tau/2)(p.v) v ; new column j+1 = old - v w_{j+1} - w v_{j+1}; rank-2 update of my rows
    double kap = 0.0;
    for (int i = j + 1 + tid; i < n; i += T) kap = fma(pv[b][i], v[i], kap);
    kap = warp_sum(kap);
    __syncthreads();
    if (lane == 0) red[warp] = kap;
    __syncthreads();
    double kk = 0.0;
    for (int k = 0; k < T / 32; ++k) kk += red[k];
    kk *= 0.5 * tau;
    for (int i = tid; i < n; i += T) w[i] = (i <= j) ? 0.0 : pv[b][i] - kk * v[i];
    __syncthreads();
    for (int i = j + 1 + tid; i < n; i += T) col[b ^ 1][i] -= v[i] * w[j + 1] + w[i] * v[j + 1];
    for (int q = warp; q < nr; q += T / 32) {
      const int i = r + q * CL;
      if (i <= j) continue;
      const double vi = v[i], wi = w[i];
      for (int c = j + 1 + lane; c < n; c += 32) rows[q][c] -= vi * w[c] + wi * v[c];
    }
    __syncthreads();
  }
  if (r == 0 && tid == 0) {
    const int b = (n - 2) & 1;
    d[n - 2] = col[b][n - 2];
    e[n - 2] = col[b][n - 1];
  }
  // d[n-1]: owner of row n-1
  if ((n - 1) % CL == r && tid == 0) d[n - 1] = rows[(n - 1) / CL][n - 1];
}

int main() {
  for (int n : {64, 256, 266, 288}) {
    std::mt19937_64 g(n);
    std::normal_distribution<double> nd;
    std::vector<double> X((size_t)(n + 4) * n), A((size_t)n * n, 0.0);
    for (auto& x : X) x = nd(g);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) {
        double s = 0;
        for (int t = 0; t < n + 4; ++t) s += X[(size_t)t * n + i] * X[(size_t)t * n + k];
        A[(size_t)i * n + k] = s;
      }
    double *dA, *dd, *de;
    cudaMalloc(&dA, 8 * (size_t)n * n);
    cudaMalloc(&dd, 8 * n);
    cudaMalloc(&de, 8 * n);
    cudaMemcpy(dA, A.data(), 8 * (size_t)n * n, cudaMemcpyHostToDevice);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(T);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * RPC * NMAX));
    cfg.dynamicSmemBytes = 8 * RPC * NMAX;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, tridiag_kernel, n, (const double*)dA, dd, de);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<double> d(n), e(n);
    cudaMemcpy(d.data(), dd, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(e.data(), de, 8 * n, cudaMemcpyDeviceToHost);
    double trA = 0, frA = 0, trT = 0, frT = 0;
    for (int i = 0; i < n; ++i) trA += A[(size_t)i * n + i];
    for (auto x : A) frA += x * x;
    for (int i = 0; i < n; ++i) trT += d[i], frT += d[i] * d[i];
    for (int i = 0; i < n - 1; ++i) frT += 2 * e[i] * e[i];
    printf("n=%d: %.3f ms  (%s)  trace rel %.2e  frobenius rel %.2e\n", n, best, cudaGetErrorString(err),
           fabs(trT - trA) / fabs(trA), fabs(frT - frA) / frA);
    cudaFree(dA);
    cudaFree(dd);
    cudaFree(de);
  }
  return 0;
}
