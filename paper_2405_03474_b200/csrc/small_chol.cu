// Small dense Cholesky G = R^T R (upper, float64, column-major, in place) on one thread-block
// cluster -- the w x w Gram factorisations of CholQR (src/linalg.py:159-180 restated as
// Cholesky-QR) and the k x k inner factor of the preconditioner
// (src/precond.py:75-80).  cuSOLVER's potrf at these sizes is a chain of ~20 small kernels
// (0.21 ms at n = 256, 0.27 ms at 266); this is one launch.
//
// Right-looking, 32-column panels, CL = 16 CTAs of one cluster; column j belongs to CTA j % CL.
// Per panel p (rows/cols [k0, k1)):
//   1. every CTA loads the diagonal block from global, applies the previous panel's update to
//      it redundantly (owners skip those columns), and factors it in one warp with the columns
//      in registers (identical arithmetic in every CTA, so a non-positive pivot is seen by all
//      and they leave together);
//   2. each CTA solves R_pp^T x = G[k0:k1, j] for its columns j >= k1 (forward substitution,
//      one warp per column) and writes the panel row R[k0:k1, j] over G;
//   3. one cluster barrier, then every CTA pulls the whole panel row into shared memory and
//      applies the rank-32 update G[k1:j, j] -= R[p, k1:j]^T R[p, j] to its columns.
// The matrix stays in global memory (L2-resident at these sizes); data other CTAs wrote is read
// with ld.global.cg after the barrier (release / acquire at cluster scope, plus a gpu fence).
// info = first failing pivot (1-based), 0 on success, as LAPACK's potrf.
#include "rld_internal.cuh"
#include "rld_device.cuh"

namespace rld {

namespace {

// CTAs per cluster: 16 (non-portable; RLD_CHOL_CL=8 for the portable size)
constexpr int NB = 32;           // panel width
constexpr int THREADS = 256;
constexpr int SMALL_CHOL_MAX = 640;

// Global-memory writes of one CTA become visible to the others: gpu-scope fence, then the
// cluster barrier (release / acquire); the reads after it go to L2 (ld.global.cg).
__device__ __forceinline__ void cluster_sync_all() {
  __threadfence();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Pivot J of the register-resident 32 x 32 factorisation (lane c holds column c); templated so
// every a[] index is a compile-time constant (the array stays in registers).
__device__ __forceinline__ double rsqrt_nr(double d) {
  // MUFU approximation + two Newton steps (relative error ~1 ulp); the IEEE sqrt and division
  // sequences are several times longer on the serial pivot chain
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

// Pivot J of the register-resident 32 x 32 factorisation (lane c holds column c); templated so
// every a[] index is a compile-time constant.  d = the (already updated) pivot, broadcast.
// The serial chain is d -> 1/sqrt(d) -> scale -> next pivot (lane J+1 updates its own two
// entries and broadcasts the result); the rank-1 update of the other entries goes through a
// shared-memory row broadcast off that chain.  No per-lane predicates: lane c's entries below
// its diagonal (a[i], i > c) are scratch that is never read.
template <int J>
__device__ __forceinline__ void chol_pivot(double (&a)[NB], double d, int lane, int& bad, double* Ri,
                                           double* rowbuf) {
  if (!(d > 0.0) && bad < 0) bad = J;   // warp-uniform; finish on dummies
  if (bad >= 0) d = 1.0;
  const double ri = rsqrt_nr(d);
  const double r = d * ri;
  a[J] = (lane == J) ? r : a[J] * ri;
  double dn = 0.0;
  if constexpr (J + 1 < NB) dn = __shfl_sync(0xffffffffu, fma(-a[J], a[J], a[J + 1]), J + 1);
  if (lane == 0) Ri[J] = ri;
  double* rb = rowbuf + (J & 1) * NB;   // double-buffered row J of R
  rb[lane] = a[J];
  __syncwarp();
#pragma unroll
  for (int i = J + 1; i < NB; ++i) a[i] = fma(-rb[i], a[J], a[i]);
  if constexpr (J + 1 < NB) chol_pivot<J + 1>(a, dn, lane, bad, Ri, rowbuf);
}


// Warp 0: factor the diagonal block in Ds (upper part valid, lower part zero / identity pad) into
// R_pp (upper part of Ds), 1/R_ii (Ri) and R_pp^-1 (upper part of Rv).  Returns via Ri[0] < 0 a
// failure marker -1 - j for a non-positive pivot j.
__device__ __forceinline__ void factor_block(double* Ds, double* Ri, double* Rv, double* rowbuf, int lane) {
  double a[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) a[i] = Ds[i * (NB + 1) + lane];
  int bad = -1;
  chol_pivot<0>(a, __shfl_sync(0xffffffffu, a[0], 0), lane, bad, Ri, rowbuf);
#pragma unroll
  for (int i = 0; i < NB; ++i) Ds[i * (NB + 1) + lane] = a[i];
  __syncwarp();
  // R^-1, column c = lane, by column-oriented back substitution: x_m = 1/R_mm (m == c) or
  // s_m / R_mm (m < c), then s_i -= R_im x_m for i < m (independent updates, short chains)
  double x[NB], sacc[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) sacc[i] = 0.0;
#pragma unroll
  for (int m = NB - 1; m >= 0; --m) {
    x[m] = (m > lane) ? 0.0 : Ri[m] * ((m == lane) ? 1.0 : sacc[m]);
#pragma unroll
    for (int i = 0; i < m; ++i) sacc[i] = fma(-Ds[i * (NB + 1) + m], x[m], sacc[i]);
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) Rv[i * (NB + 1) + lane] = x[i];
  if (bad >= 0 && lane == 0) Ri[0] = -1.0 - (double)bad;
}

template <int CL>
__global__ void __launch_bounds__(THREADS)
chol_upper_kernel(int n, double* __restrict__ G, int ld, int* __restrict__ info, double* __restrict__ X,
                  long long* __restrict__ prof) {
  extern __shared__ double sm[];
  constexpr int LDB = NB + 1;
  double* Ds = sm;                  // NB x LDB: diagonal block / its factor R_pp (upper part)
  double* Rv = Ds + NB * LDB;       // NB x LDB: R_pp^-1 (upper part)
  double* Dn = Rv + NB * LDB;       // NB x LDB: next diagonal block as loaded from global
  double* Ri = Dn + NB * LDB;       // NB: 1 / R_ii
  double* rowbuf = Ri + NB;         // 2 x NB: pivot-row broadcast of the diagonal factorisation
  double* Gs = rowbuf + 2 * NB;     // CMAX x LDB: this CTA's columns of the panel rows (step 2 input)
  constexpr int CMAX = (SMALL_CHOL_MAX + CL - 1) / CL;
  double* Pt = Gs + CMAX * LDB;     // n x LDB: panel row, Pt[j * LDB + m] = R[k0 + m, j]
  const int cta = (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npanels = (n + NB - 1) / NB;
  long long t_prev = clock64();
  auto mark = [&](int slot) {   // RLD_CHOL_PROFILE: per-phase cycles of CTA 0
    if (prof && cta == 0) {
      __syncthreads();
      const long long t = clock64();
      if (tid == 0) prof[slot] += t - t_prev;
      t_prev = t;
    }
  };

  // ---- prologue: the first diagonal block straight from global
  {
    const int kb = min(NB, n);
    for (int e = tid; e < NB * NB; e += THREADS) {
      const int i = e % NB, c = e / NB;
      Ds[i * LDB + c] = (i < kb && c < kb) ? ((i <= c) ? __ldcg(G + (size_t)c * ld + i) : 0.0) : (i == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (warp == 0) factor_block(Ds, Ri, Rv, rowbuf, lane);
    __syncthreads();
  }
  mark(0);

  for (int p = 0; p < npanels; ++p) {
    const int k0 = p * NB, kb = min(NB, n - k0), k1 = k0 + kb;
    if (Ri[0] < 0.0) {   // identical in every CTA: leave together
      if (cta == 0 && tid == 0) *info = k0 + (int)(-Ri[0] - 1.0) + 1;
      return;
    }
    // R_pp goes over the diagonal block only after the cluster barrier: until then the other CTAs
    // may still be reading that block
    auto write_rpp = [&]() {   // also R_pp^-1 into X's diagonal block when R^-1 is wanted
      if (cta == 0)
        for (int e = tid; e < kb * kb; e += THREADS) {
          const int i = e % kb, c = e / kb;
          if (i <= c) {
            G[(size_t)(k0 + c) * ld + k0 + i] = Ds[i * LDB + c];
            if (X) X[(size_t)(k0 + c) * n + k0 + i] = Rv[i * LDB + c];
          }
        }
    };
    if (k1 >= n) {
      cluster_sync_all();
      write_rpp();
      break;
    }
    // ---- 2. panel row for this CTA's columns j >= k1: R[p, j] = R_pp^-T g_j
    const int jstart = k1 + ((cta - k1 % CL) + CL) % CL;   // first column j >= k1 with j % CL == cta
    const int ncol = jstart < n ? (n - 1 - jstart) / CL + 1 : 0;
    for (int e = tid; e < ncol * NB; e += THREADS) {   // this CTA's own columns: plain loads are coherent
      const int m = e % NB, q = e / NB;
      Gs[q * LDB + m] = (m < kb) ? G[(size_t)(jstart + q * CL) * ld + k0 + m] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < ncol * NB; e += THREADS) {
      const int m = e % NB, q = e / NB;
      double x4[4] = {0.0, 0.0, 0.0, 0.0};   // four short chains instead of one of length 32
#pragma unroll
      for (int l = 0; l < NB; ++l) x4[l & 3] = fma(Rv[l * LDB + m], Gs[q * LDB + l], x4[l & 3]);   // Rv lower part is 0
      if (m < kb) G[(size_t)(jstart + q * CL) * ld + k0 + m] = (x4[0] + x4[1]) + (x4[2] + x4[3]);
    }
    mark(1);
    cluster_sync_all();
    mark(2);
    write_rpp();
    // ---- 3. panel row (all columns) and the next diagonal block into shared memory
    const int k2 = min(n, k1 + NB), kb2 = k2 - k1;
    // other CTAs wrote these: L2 loads (ld.global.cg), never a possibly stale L1 line (a column's
    // 128-byte lines straddle panels, so this SM may hold an old copy from the previous panel)
    {
      const int tot = NB * (n - k1);
      constexpr int UNR = 16;
      for (int e0 = tid; e0 < tot; e0 += THREADS * UNR) {
        double v[UNR];
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          const int e = e0 + q * THREADS;
          const int m = e % NB, j = k1 + e / NB;
          v[q] = (e < tot && m < kb) ? __ldcg(G + (size_t)j * ld + k0 + m) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          const int e = e0 + q * THREADS;
          if (e < tot) Pt[(k1 + e / NB) * LDB + e % NB] = v[q];
        }
      }
    }
    for (int e = tid; e < NB * NB; e += THREADS) {
      const int i = e % NB, c = e / NB;
      Dn[i * LDB + c] = (i < kb2 && c < kb2) ? ((i <= c) ? __ldcg(G + (size_t)(k1 + c) * ld + k1 + i) : 0.0)
                                             : (i == c ? 1.0 : 0.0);
    }
    __syncthreads();
    mark(3);
    // ---- 4a. next diagonal block = Dn - panel-row update (all threads), then warp 0 factors it
    for (int e = tid; e < NB * NB; e += THREADS) {
      const int i = e % NB, c = e / NB;
      double v = Dn[i * LDB + c];
      if (i <= c && c < kb2) {
        double u4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < NB; ++m) u4[m & 3] = fma(Pt[(k1 + i) * LDB + m], Pt[(k1 + c) * LDB + m], u4[m & 3]);
        v -= (u4[0] + u4[1]) + (u4[2] + u4[3]);
      }
      Ds[i * LDB + c] = v;
    }
    __syncthreads();
    if (warp == 0) {
      const long long tf = clock64();
      factor_block(Ds, Ri, Rv, rowbuf, lane);
      if (prof && cta == 0 && lane == 0) prof[5] += clock64() - tf;
    } else {
      // ---- 4b. rank-kb update of this CTA's columns beyond the next diagonal block
      const int js2 = k2 + ((cta - k2 % CL) + CL) % CL;
      for (int j = js2 + (warp - 1) * CL; j < n; j += CL * (THREADS / 32 - 1)) {
        double pj[NB];
#pragma unroll
        for (int m = 0; m < NB; ++m) pj[m] = Pt[j * LDB + m];
        // this column's rows in chunks of 8 per lane: all 8 L2 loads of G issued before the FMAs
        // (one round trip per chunk instead of one per row: the update was L2-latency bound)
        for (int ib = k1; ib <= j; ib += 256) {
          double g[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = ib + lane + 32 * u;
            g[u] = (i <= j) ? G[(size_t)j * ld + i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = ib + lane + 32 * u;
            if (i <= j) {
              const double* P1 = Pt + i * LDB;
              double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
              for (int m = 0; m < NB; ++m) s4[m & 3] = fma(P1[m], pj[m], s4[m & 3]);
              G[(size_t)j * ld + i] = g[u] - ((s4[0] + s4[1]) + (s4[2] + s4[3]));
            }
          }
        }
      }
    }
    __syncthreads();
    mark(4);
  }
  if (cta == 0 && tid == 0) *info = 0;
  if (!X) return;
  // ---- R^-1 (upper, n x n, ld n; lower part left as the caller's zeros), block column J by this
  // CTA (J % CL == cta): X_JJ = R_JJ^-1 is in place; X_IJ = -R_II^-1 sum_{K=I+1..J} R_IK X_KJ for
  // I = J-1 .. 0 (block back substitution), the column's blocks kept in shared memory
  cluster_sync_all();   // every panel row of R and every diagonal inverse is in global memory
  double* Xc = Pt;      // npanels x NB x NB: this column's blocks, Xc[K][m][c]
  double* S = Dn;       // NB x LDB
  const int ri = tid & 31, cg = tid >> 5;   // output row, 4-column group
  for (int J = cta; J < npanels; J += CL) {
    const int cJ = J * NB, wJ = min(NB, n - cJ);
    for (int e = tid; e < NB * NB; e += THREADS) {
      const int m = e % NB, c = e / NB;
      Xc[(size_t)J * NB * NB + m * NB + c] = (m < wJ && c < wJ && m <= c) ? __ldcg(X + (size_t)(cJ + c) * n + cJ + m) : 0.0;
    }
    __syncthreads();
    for (int I = J - 1; I >= 0; --I) {
      const int rI = I * NB;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int K = I + 1; K <= J; ++K) {
        const int cK = K * NB, wK = min(NB, n - cK);
        const double* Xk = Xc + (size_t)K * NB * NB;
        for (int m0 = 0; m0 < wK; m0 += 8) {   // 8 independent L2 loads in flight per thread
          double r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            r[u] = (m0 + u < wK) ? __ldcg(G + (size_t)(cK + m0 + u) * ld + rI + ri) : 0.0;   // R[rI + ri, cK + m]
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(r[u], Xk[(m0 + u) * NB + cg * 4 + q], acc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) S[ri * LDB + cg * 4 + q] = acc[q];
      __syncthreads();
      double x[4] = {0.0, 0.0, 0.0, 0.0};
      for (int m0 = 0; m0 < NB; m0 += 8) {   // R_II^-1 is upper: row ri, columns m >= ri (zeros below)
        double rv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rv[u] = (m0 + u >= ri) ? __ldcg(X + (size_t)(rI + m0 + u) * n + rI + ri) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = fma(rv[u], S[(m0 + u) * LDB + cg * 4 + q], x[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cg * 4 + q;
        Xc[(size_t)I * NB * NB + ri * NB + c] = -x[q];
        if (c < wJ) X[(size_t)(cJ + c) * n + rI + ri] = -x[q];
      }
      __syncthreads();
    }
  }
}

}  // namespace

bool small_potrf_upper(int n, double* G, int ld, int* info, cudaStream_t st, double* Rinv) {
  if (n < 1 || n > SMALL_CHOL_MAX) return false;
  // the panel-row buffer doubles as the R^-1 column blocks (ceil(n / 32) 32 x 32 blocks)
  auto smem_for = [](int nn, int cl) {
    const size_t cmax = (size_t)(SMALL_CHOL_MAX + cl - 1) / cl;
    const size_t tail = std::max((size_t)nn * (NB + 1), (size_t)NB * NB * ((nn + NB - 1) / NB));
    return sizeof(double) * ((size_t)3 * NB * (NB + 1) + 3 * NB + cmax * (NB + 1)) + sizeof(double) * tail;
  };
  static std::atomic<uint64_t> attr_set{0};
  once_per_device(attr_set, [&] {
    RLD_CUDA(cudaFuncSetAttribute(chol_upper_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem_for(SMALL_CHOL_MAX, 8)));
    RLD_CUDA(cudaFuncSetAttribute(chol_upper_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem_for(SMALL_CHOL_MAX, 16)));
    RLD_CUDA(cudaFuncSetAttribute(chol_upper_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  // RLD_CHOL_CL=8/16 forces the cluster size (measurement)
  static const int cl_env = getenv("RLD_CHOL_CL") ? atoi(getenv("RLD_CHOL_CL")) : 0;
  const int cl = cl_env == 8 || cl_env == 16 ? cl_env : 16;   // 16: 255 vs 314 us at n = 522, 120 vs 129 at 266
  const size_t smem = smem_for(n, cl);
  static const bool profile = getenv("RLD_CHOL_PROFILE") != nullptr;
  long long* prof = nullptr;
  if (profile) RLD_CUDA(cudaMallocAsync(&prof, 8 * sizeof(long long), st)), RLD_CUDA(cudaMemsetAsync(prof, 0, 64, st));
  if (Rinv) RLD_CUDA(cudaMemsetAsync(Rinv, 0, sizeof(double) * (size_t)n * n, st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cl == 16)
    RLD_CUDA(cudaLaunchKernelEx(&cfg, chol_upper_kernel<16>, n, G, ld, info, Rinv, prof));
  else
    RLD_CUDA(cudaLaunchKernelEx(&cfg, chol_upper_kernel<8>, n, G, ld, info, Rinv, prof));
  RLD_LAUNCH_CHECK();
  if (profile) {
    long long hp[8];
    RLD_CUDA(cudaMemcpyAsync(hp, prof, sizeof hp, cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    RLD_CUDA(cudaFree(prof));
    fprintf(stderr, "small_chol n=%d cycles: prologue %lld panel-row %lld barrier %lld load %lld factor||update %lld "
            "(factor alone %lld)\n", n, hp[0], hp[1], hp[2], hp[3], hp[4], hp[5]);
  }
  return true;
}

}  // namespace rld
