// Symmetric eigensolver for the preconditioner's small matrices (B, w x w, src/precond.py:189-190;
// At^T At, k x k, src/precond.py:96), n <= 288, built from
//   1. Householder tridiagonalisation on one 16-CTA cluster (rows distributed, one cluster barrier
//      per column: the next column is rebuilt redundantly from the broadcast old column and w);
//      the reflectors (v_j, tau_j) go to global memory;
//   2. eigenvalues of the tridiagonal T by multisection (one warp per eigenvalue, 32 Sturm counts
//      per iteration);
//   3. eigenvectors of T by inverse iteration (one thread per eigenvalue, tridiagonal LU with
//      partial pivoting, start vectors that differ per index so repeated eigenvalues span their
//      eigenspace), then one Cholesky-QR pass over all of them (they are orthogonal up to
//      eps |T| / gap; the pass restores orthogonality inside close clusters);
//   4. the back-transformation Q Z with Q = H_0 ... H_{n-3} formed row-locally by the cluster.
// Positive semi-definiteness is not required.  Results match LAPACK eigh up to eigenvector signs
// and rotations inside (near-)degenerate eigenspaces, neither of which changes P.
#include "rld_internal.cuh"
#include "rld_device.cuh"
#include "rld_kernels.cuh"

#include <cooperative_groups.h>

namespace rld {

namespace {

namespace cg = cooperative_groups;
constexpr int TCL = 16, TT = 256, TNMAX = 288;
// Two instantiations: n <= 288 (256 threads, 18 rows per CTA) and n <= 544 (192 threads, 34 rows
// per CTA: 148 KB of rows + the per-warp v / w slots + the broadcast columns fill the 227 KB)
constexpr int TNMAX_L = 544, TT_L = 192;
template <int NMAX, int TTH>
constexpr size_t tridiag_smem_t() {
  return sizeof(double) * ((size_t)((NMAX + TCL - 1) / TCL) * NMAX + (size_t)(TTH / 32) * 2 * NMAX + 4 * (size_t)NMAX);
}

// sqrt and reciprocal on the per-column chain from the MUFU approximations plus two Newton steps
// (~1 ulp): the IEEE FP64 sqrt / division sequences are several times longer.  Normal inputs only
// (callers keep the IEEE path below 1e-300).
__device__ __forceinline__ double sqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return x * y;
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = fma(y, fma(-x, y, 1.0), y);
  y = fma(y, fma(-x, y, 1.0), y);
  return y;
}

// A column-major n x n symmetric (only symmetry is used: row i == column i).  Outputs d (n),
// e (n - 1), tau (n - 2) and the reflectors V (n x (n - 2), column j = v_j, zero above j + 1).
// Each CTA owns rows i = r, r + 16, ...; per column ONE cluster barrier and no block barrier:
// every warp keeps the current column, v and w in registers (c = lane + 32k), computes the
// reflector and both dot products redundantly with butterflies, and reads v_i / w_i of its own
// rows (the rank-2 update) from a per-warp shared slot.  Owners broadcast p = tau A v and their
// raw entries of the next column through DSMEM; the next column is rebuilt locally from them.
// (0.63 ms vs 0.89 ms for the block-barrier version at n = 266: scripts/tridiag_bench3.cu.)
template <int NMAX, int TTH>
__global__ void __launch_bounds__(TTH)
tridiag_kernel(int n, const double* __restrict__ A, double* __restrict__ d, double* __restrict__ e,
               double* __restrict__ tau_out, double* __restrict__ V) {
  constexpr int K = NMAX / 32, W = TTH / 32, TT = TTH, TNMAX = NMAX, TRPC = (NMAX + TCL - 1) / TCL;
  static_assert(NMAX % 32 == 0, "NMAX must be a multiple of 32");
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double sm[];
  double (*rows)[TNMAX] = reinterpret_cast<double (*)[TNMAX]>(sm);                  // [TRPC][TNMAX]
  double (*vw)[2][TNMAX] = reinterpret_cast<double (*)[2][TNMAX]>(sm + TRPC * TNMAX);  // [W][2][TNMAX]
  double (*col)[TNMAX] = reinterpret_cast<double (*)[TNMAX]>(sm + (TRPC + 2 * W) * TNMAX);  // [2][TNMAX] raw broadcast column
  double (*pv)[TNMAX] = col + 2;     // [2][TNMAX] broadcast p = tau A v
  const int nr = (n - r + TCL - 1) / TCL;
  for (int q = 0; q < nr; ++q)
    for (int c = tid; c < n; c += TT) rows[q][c] = A[(size_t)(r + q * TCL) * n + c];
  __syncthreads();
  for (int q = tid; q < nr; q += TT) {
    const int i = r + q * TCL;
    for (int dst = 0; dst < TCL; ++dst) *cl.map_shared_rank(&col[0][i], dst) = rows[q][0];
  }
  cl.sync();
  double x[K], v[K], w[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int c = lane + 32 * k;
    x[k] = c < n ? col[0][c] : 0.0;
  }
  double* myv = vw[warp][0];
  double* myw = vw[warp][1];
  for (int c = lane; c < TNMAX; c += 32) myv[c] = myw[c] = 0.0;
  __syncwarp();
  // the previous column's reflector scalars v_j, w_j: entry c of the current column is
  // col[b][c] - (v'_c w'_j + w'_c v'_j) with v', w' still in this warp's slot
  double pvj = 0.0, pwj = 0.0;
  for (int j = 0; j < n - 2; ++j) {
    const int b = j & 1;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k > j) s = fma(x[k], x[k], s);
    const double sig = warp_sum(s);
    const double x0 = col[b][j + 1] - (myv[j + 1] * pwj + myw[j + 1] * pvj);
    const double dj = col[b][j] - (myv[j] * pwj + myw[j] * pvj);
    __syncwarp();
    const double alpha = -copysign(sig > 1e-300 ? sqrt_nr(sig) : sqrt(sig), x0);
    const double vtv = sig - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    const double tau = vtv > 1e-300 ? 2.0 * rcp_nr(vtv) : (vtv > 0.0 ? 2.0 / vtv : 0.0);
    const double vj1 = x0 - alpha;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      v[k] = (c <= j) ? 0.0 : (c == j + 1 ? vj1 : x[k]);
      myv[c] = v[k];
    }
    if (r == 0 && warp == 0) {
      if (lane == 0) {
        d[j] = dj;
        e[j] = (tau > 0.0) ? alpha : x0;
        tau_out[j] = tau;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c < n) V[(size_t)j * n + c] = v[k];
      }
    }
    for (int q = warp; q < nr; q += W) {
      const int i = r + q * TCL;
      if (i <= j) continue;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c > j && c < n) acc = fma(rows[q][c], v[k], acc);
      }
      acc = warp_sum(acc);
      if (lane < TCL) {
        *cl.map_shared_rank(&pv[b][i], lane) = tau * acc;
        *cl.map_shared_rank(&col[b ^ 1][i], lane) = rows[q][j + 1];
      }
    }
    cl.sync();
    double kap = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      w[k] = (c > j && c < n) ? pv[b][c] : 0.0;
      kap = fma(w[k], v[k], kap);
    }
    const double kk = 0.5 * tau * warp_sum(kap);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k] = fma(-kk, v[k], w[k]);
      myw[lane + 32 * k] = w[k];
    }
    __syncwarp();
    const double wj1 = fma(-kk, vj1, pv[b][j + 1]);
    pvj = vj1;
    pwj = wj1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      x[k] = (c > j && c < n) ? col[b ^ 1][c] - (v[k] * wj1 + w[k] * vj1) : 0.0;
    }
    for (int q = warp; q < nr; q += W) {
      const int i = r + q * TCL;
      if (i <= j) continue;
      const double vi = myv[i], wi = myw[i];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c > j && c < n) rows[q][c] -= vi * w[k] + wi * v[k];
      }
    }
    __syncwarp();
  }
  if (n >= 3) {
    const int b = (n - 2) & 1;
    const double a = col[b][n - 2] - (myv[n - 2] * pwj + myw[n - 2] * pvj);
    const double bb = col[b][n - 1] - (myv[n - 1] * pwj + myw[n - 1] * pvj);
    if (r == 0 && tid == 0) {
      d[n - 2] = a;
      e[n - 2] = bb;
    }
  }
  __syncthreads();   // row n - 1 was last updated by its owner warp
  if ((n - 1) % TCL == r && tid == 0) d[n - 1] = rows[(n - 1) / TCL][n - 1];
}


// Variant with ONE set of v / w slots per CTA (double-buffered by column parity) instead of one per
// warp, so the shared memory that held the per-warp copies goes to more warps (fewer rows per warp
// on the latency-bound per-column chain), and two rows per warp iteration (independent dot
// products and butterflies interleave).  Warp 0 writes the slots; the cluster barrier publishes
// v, one block barrier per column publishes w before the rank-2 update.
template <int NMAX, int TTH>
constexpr size_t tridiag2_smem_t() {
  return sizeof(double) * ((size_t)((NMAX + TCL - 1) / TCL) * NMAX + 8 * (size_t)NMAX);
}

template <int NMAX, int TTH>
__global__ void __launch_bounds__(TTH)
tridiag2_kernel(int n, const double* __restrict__ A, double* __restrict__ d, double* __restrict__ e,
                double* __restrict__ tau_out, double* __restrict__ V) {
  constexpr int K = NMAX / 32, W = TTH / 32, TRPC = (NMAX + TCL - 1) / TCL;
  static_assert(NMAX % 32 == 0, "NMAX must be a multiple of 32");
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double sm[];
  double (*rows)[NMAX] = reinterpret_cast<double (*)[NMAX]>(sm);                     // [TRPC][NMAX]
  double (*slot)[2][NMAX] = reinterpret_cast<double (*)[2][NMAX]>(sm + TRPC * NMAX);  // [parity][v, w][NMAX]
  double (*col)[NMAX] = reinterpret_cast<double (*)[NMAX]>(sm + (TRPC + 4) * NMAX);   // [2][NMAX] raw column
  double (*pv)[NMAX] = col + 2;                                                      // [2][NMAX] p = tau A v
  const int nr = (n - r + TCL - 1) / TCL;
  for (int q = 0; q < nr; ++q)
    for (int c = tid; c < n; c += TTH) rows[q][c] = A[(size_t)(r + q * TCL) * n + c];
  for (int c = tid; c < 4 * NMAX; c += TTH) (&slot[0][0][0])[c] = 0.0;
  __syncthreads();
  for (int q = tid; q < nr; q += TTH) {
    const int i = r + q * TCL;
    for (int dst = 0; dst < TCL; ++dst) *cl.map_shared_rank(&col[0][i], dst) = rows[q][0];
  }
  cl.sync();
  double x[K], v[K], w[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int c = lane + 32 * k;
    x[k] = c < n ? col[0][c] : 0.0;
  }
  double pvj = 0.0, pwj = 0.0;
  for (int j = 0; j < n - 2; ++j) {
    const int b = j & 1;
    const double* vp = slot[b ^ 1][0];   // the previous column's v', w'
    const double* wp = slot[b ^ 1][1];
    double s0 = 0.0, s1 = 0.0;   // two chains: the per-column path is latency-bound
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k > j) {
        if (k & 1) s1 = fma(x[k], x[k], s1);
        else s0 = fma(x[k], x[k], s0);
      }
    const double sig = warp_sum(s0 + s1);
    const double x0 = col[b][j + 1] - (vp[j + 1] * pwj + wp[j + 1] * pvj);
    const double dj = col[b][j] - (vp[j] * pwj + wp[j] * pvj);
    const double alpha = -copysign(sig > 1e-300 ? sqrt_nr(sig) : sqrt(sig), x0);
    const double vtv = sig - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    const double tau = vtv > 1e-300 ? 2.0 * rcp_nr(vtv) : (vtv > 0.0 ? 2.0 / vtv : 0.0);
    const double vj1 = x0 - alpha;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      v[k] = (c <= j) ? 0.0 : (c == j + 1 ? vj1 : x[k]);
      if (warp == 0) slot[b][0][c] = v[k];
    }
    if (r == 0 && warp == 0) {
      if (lane == 0) {
        d[j] = dj;
        e[j] = (tau > 0.0) ? alpha : x0;
        tau_out[j] = tau;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c < n) V[(size_t)j * n + c] = v[k];
      }
    }
    // own rows i > j, two per iteration: p_i = tau (row_i . v), broadcast with the raw entry of
    // the next column
    for (int q = warp; q < nr; q += 2 * W) {
      const int q2 = q + W;
      const int i1 = r + q * TCL, i2 = r + q2 * TCL;
      const bool a1 = i1 > j, a2 = q2 < nr && i2 > j;
      if (!a1 && !a2) continue;
      double acc1 = 0.0, acc2 = 0.0, acc3 = 0.0, acc4 = 0.0;
      const double* r1 = rows[q];
      const double* r2 = rows[a2 ? q2 : q];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c > j && c < n) {
          if (k & 1) {
            acc3 = fma(r1[c], v[k], acc3);
            acc4 = fma(r2[c], v[k], acc4);
          } else {
            acc1 = fma(r1[c], v[k], acc1);
            acc2 = fma(r2[c], v[k], acc2);
          }
        }
      }
      acc1 += acc3;
      acc2 += acc4;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
        acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
      }
      if (lane < TCL) {
        if (a1) {
          *cl.map_shared_rank(&pv[b][i1], lane) = tau * acc1;
          *cl.map_shared_rank(&col[b ^ 1][i1], lane) = r1[j + 1];
        }
        if (a2) {
          *cl.map_shared_rank(&pv[b][i2], lane) = tau * acc2;
          *cl.map_shared_rank(&col[b ^ 1][i2], lane) = r2[j + 1];
        }
      }
    }
    cl.sync();
    double kap0 = 0.0, kap1 = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      w[k] = (c > j && c < n) ? pv[b][c] : 0.0;
      if (k & 1) kap1 = fma(w[k], v[k], kap1);
      else kap0 = fma(w[k], v[k], kap0);
    }
    const double kk = 0.5 * tau * warp_sum(kap0 + kap1);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k] = fma(-kk, v[k], w[k]);
      if (warp == 0) slot[b][1][lane + 32 * k] = w[k];
    }
    const double wj1 = fma(-kk, vj1, pv[b][j + 1]);
    pvj = vj1;
    pwj = wj1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = lane + 32 * k;
      x[k] = (c > j && c < n) ? col[b ^ 1][c] - (v[k] * wj1 + w[k] * vj1) : 0.0;
    }
    __syncthreads();   // w in the slot
    const double* vs = slot[b][0];
    const double* ws = slot[b][1];
    for (int q = warp; q < nr; q += W) {
      const int i = r + q * TCL;
      if (i <= j) continue;
      const double vi = vs[i], wi = ws[i];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = lane + 32 * k;
        if (c > j && c < n) rows[q][c] -= vi * w[k] + wi * v[k];
      }
    }
  }
  if (n >= 3) {
    const int b = (n - 2) & 1;
    const double* vp = slot[b ^ 1][0];
    const double* wp = slot[b ^ 1][1];
    const double a = col[b][n - 2] - (vp[n - 2] * pwj + wp[n - 2] * pvj);
    const double bb = col[b][n - 1] - (vp[n - 1] * pwj + wp[n - 1] * pvj);
    if (r == 0 && tid == 0) {
      d[n - 2] = a;
      e[n - 2] = bb;
    }
  }
  __syncthreads();   // row n - 1 was last updated by its owner warp
  if ((n - 1) % TCL == r && tid == 0) d[n - 1] = rows[(n - 1) / TCL][n - 1];
}


// T splits between i and i + 1 when e_i^2 <= eps^2 |d_i d_{i+1}| (LAPACK dstebz's test): the
// coupling is treated as zero by both the eigenvalue and the eigenvector kernels
__device__ __forceinline__ bool split_at(const double* d, const double* e, int i) {
  const double e2 = e[i] * e[i];
  return e2 <= 4.93e-32 * fabs(d[i] * d[i + 1]) + 1e-300;
}

// Number of eigenvalues of rows [s, t] of T below x: sign changes of the leading principal minors
// p_i = det(T_i - x I) (p_i / p_{i-1} are the LDL^T pivots, so this is the usual Sturm count),
// by the division-free three-term recurrence -- one dependent FMA per row instead of a division.
// Expects T scaled to |T| <= ~1 (growth <= 3 per row); both minors are renormalised by a power of
// two (exponent-field arithmetic) every 8 rows.  A zero minor counts as negative (LAPACK's -pivmin
// rule): it is replaced by a tiny value of the opposite sign of its predecessor.
__device__ __forceinline__ void sturm_step(double dx, double e2i, double& p1, double& p2, int& cnt) {
  double p = fma(dx, p1, -e2i * p2);
  if (p == 0.0) p = -copysign(0x1p-900, p1);
  cnt += (__double2hiint(p) ^ __double2hiint(p1)) < 0;
  p2 = p1;
  p1 = p;
}
__device__ __forceinline__ void sturm_renorm(double& p1, double& p2) {
  const int e1 = (__double2hiint(p1) >> 20) & 0x7ff, e2 = (__double2hiint(p2) >> 20) & 0x7ff;
  const int sh = min(max(2046 - max(e1, e2), 1), 2046);   // biased exponent of 2^(1023 - max)
  const double f = __hiloint2double(sh << 20, 0);
  p1 *= f;
  p2 *= f;
}
__device__ __forceinline__ int sturm_block(int s, int t, const double* __restrict__ d, const double* __restrict__ e2,
                                           double x) {
  double p2 = 1.0, p1 = d[s] - x;
  if (p1 == 0.0) p1 = -0x1p-900;
  int cnt = p1 < 0.0;
  int i = s + 1;
  for (; i + 7 <= t; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) sturm_step(d[i + u] - x, e2[i + u - 1], p1, p2, cnt);
    sturm_renorm(p1, p2);
  }
  for (; i <= t; ++i) sturm_step(d[i] - x, e2[i - 1], p1, p2, cnt);
  return cnt;
}

// Two Sturm counts of rows [0, n) at xa and xb, interleaved (two independent recurrences per
// thread: the chain is latency-bound, so the second count is nearly free).
__device__ __forceinline__ void sturm_pair(int n, const double* __restrict__ d, const double* __restrict__ e2,
                                           double xa, double xb, int& ca, int& cb) {
  double a2 = 1.0, a1 = d[0] - xa, b2 = 1.0, b1 = d[0] - xb;
  if (a1 == 0.0) a1 = -0x1p-900;
  if (b1 == 0.0) b1 = -0x1p-900;
  ca = a1 < 0.0;
  cb = b1 < 0.0;
  int i = 1;
  for (; i + 7 <= n - 1; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double di = d[i + u], ei = e2[i + u - 1];
      sturm_step(di - xa, ei, a1, a2, ca);
      sturm_step(di - xb, ei, b1, b2, cb);
    }
    sturm_renorm(a1, a2);
    sturm_renorm(b1, b2);
  }
  for (; i <= n - 1; ++i) {
    sturm_step(d[i] - xa, e2[i - 1], a1, a2, ca);
    sturm_step(d[i] - xb, e2[i - 1], b1, b2, cb);
  }
}

// d, e of T scaled by a power of two to |T|_inf <= 1 (exact), squared couplings with splits zeroed.
// Staged through shared memory first (the norm loop would otherwise walk global memory serially).
__device__ __forceinline__ double load_scaled(int n, const double* __restrict__ d, const double* __restrict__ e,
                                              double* ds, double* e2, double* es) {
  double* eraw = es ? es : e2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ds[i] = d[i];
    eraw[i] = (i < n - 1) ? e[i] : 0.0;
  }
  __syncthreads();
  double tnorm = 0.0;
  for (int i = 0; i < n; ++i) tnorm = fmax(tnorm, fabs(ds[i]) + (i > 0 ? fabs(eraw[i - 1]) : 0.0) + fabs(eraw[i]));
  const double sc = tnorm > 0.0 ? scalbn(1.0, -ilogb(tnorm) - 1) : 1.0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const bool sp = (i == n - 1) || split_at(d, e, i);
    const double ei = eraw[i];
    ds[i] *= sc;
    e2[i] = sp ? 0.0 : (ei * sc) * (ei * sc);
    if (es) es[i] = sp ? 0.0 : ei;
  }
  return sc;
}

// eigenvalue k (ascending) of T by multisection, one warp per eigenvalue: each iteration the lanes
// test 63 interior points of [lo, hi] (~6 bits), down to 2 eps |T| or 2 ulp of the eigenvalue
__global__ void bisect_kernel(int n, const double* __restrict__ d, const double* __restrict__ e,
                              double* __restrict__ lam) {
  extern __shared__ double sh[];
  double* ds = sh;
  double* e2 = sh + n;
  const double sc = load_scaled(n, d, e, ds, e2, nullptr);
  __syncthreads();
  double glo = 1e300, ghi = -1e300;
  for (int i = 0; i < n; ++i) {
    const double rad = (i > 0 ? sqrt(e2[i - 1]) : 0.0) + sqrt(e2[i]);
    glo = fmin(glo, ds[i] - rad);
    ghi = fmax(ghi, ds[i] + rad);
  }
  const double atol = 2.0 * 2.2e-16;   // |T| <= 1 after scaling
  const int lane = threadIdx.x & 31;
  const int k = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (k >= n) return;
  double lo = glo - atol, hi = ghi + atol;
  for (int it = 0; it < 200 && hi - lo > fmax(atol, 4.4e-16 * fmax(fabs(lo), fabs(hi))); ++it) {
    // 64 points lo + (hi - lo) q / 64, q = 1..64 (~6 bits per iteration): lane l tests q = l + 1
    // and q = l + 33; q = 64 is hi itself (count n)
    const double xa = lo + (hi - lo) * (double)(lane + 1) / 64.0;
    const double xb = lo + (hi - lo) * (double)(lane + 33) / 64.0;
    int ca, cb;
    sturm_pair(n, ds, e2, xa, xb, ca, cb);
    if (lane == 31) cb = n;
    // smallest point whose count exceeds k: the eigenvalue lies below it
    const unsigned aa = __ballot_sync(0xffffffffu, ca > k), ab = __ballot_sync(0xffffffffu, cb > k);
    const int first = aa ? __ffs(aa) - 1 : 32 + __ffs(ab) - 1;   // exists: q = 64 has count n > k
    const double nhi = lo + (hi - lo) * (double)(first + 1) / 64.0;
    const double nlo = lo + (hi - lo) * (double)first / 64.0;
    hi = (first == 63) ? hi : nhi;
    lo = nlo;
  }
  if (lane == 0) lam[k] = 0.5 * (lo + hi) / sc;
}

// eigenvalues (threads) per inverse-iteration CTA: 16 for n <= 288, 8 above (the per-thread
// factors take 5 n doubles of shared memory)

// eigenvector k of T by inverse iteration on the unreduced block of T that owns eigenvalue k
// (LAPACK dstein style).  Ownership (only when T splits): the eigenvalues within +-delta of lam[k]
// are ranked globally (c_lo = count below lam - delta) and handed to the blocks in row order by
// their own counts, so an eigenvalue shared by several blocks (exact degeneracy) gets one vector
// per block, supported on that block only.  The solve is LU with partial pivoting of T_b - lam I
// (dlagtf / dlagts), three iterations from a start vector that differs per k; unit norm, zero off
// the block.  The factors and the iterate live in shared memory, interleaved over the CTA's 16
// threads ([field][row][thread]: conflict-free), so the serial recurrences run at shared-memory
// latency.
template <int IV_T>
__global__ void __launch_bounds__(IV_T)
inviter_kernel(int n, const double* __restrict__ d, const double* __restrict__ e, const double* __restrict__ lam,
               double* __restrict__ Z) {
  extern __shared__ double sh_iv[];
  double* ds = sh_iv;
  double* es = sh_iv + n;
  double* e2 = sh_iv + 2 * n;
  double* fw = sh_iv + 3 * n;
  unsigned* pbits = reinterpret_cast<unsigned*>(fw + (size_t)5 * n * IV_T);
  const double sc = load_scaled(n, d, e, ds, e2, es);
  __syncthreads();
  const int t = threadIdx.x;
  const int k = blockIdx.x * IV_T + t;
  if (k >= n) return;
#define FW(f, i) fw[((size_t)(f) * n + (i)) * IV_T + t]
  const int nw = (n + 31) / 32;
#define PB(i) pbits[((i) >> 5) * IV_T + t]
  const double shs = lam[k] * sc;   // shift in the scaled units of ds / e2
  // ---- owning block
  bool splits = false;
  for (int i = 0; i < n - 1; ++i) splits |= (e2[i] == 0.0);
  int bs = 0, bt = n - 1;
  if (splits) {
    for (double delta = 16.0 * 2.2e-16;; delta *= 16.0) {
      int c_lo = 0;
      for (int s0 = 0; s0 < n;) {
        int t0 = s0;
        while (e2[t0] != 0.0) ++t0;
        c_lo += sturm_block(s0, t0, ds, e2, shs - delta);
        s0 = t0 + 1;
      }
      int cum = c_lo, found = 0;
      for (int s0 = 0; s0 < n && !found;) {
        int t0 = s0;
        while (e2[t0] != 0.0) ++t0;
        const int m = sturm_block(s0, t0, ds, e2, shs + delta) - sturm_block(s0, t0, ds, e2, shs - delta);
        if (k >= cum && k < cum + m) {
          bs = s0;
          bt = t0;
          found = 1;
        }
        cum += m;
        s0 = t0 + 1;
      }
      if (found || delta > 1e-3) break;
    }
  }
  if (bs == bt) {
    for (int i = 0; i < n; ++i) Z[(size_t)k * n + i] = (i == bs) ? 1.0 : 0.0;
    return;
  }
  // LU with partial pivoting of the scaled block, T_b sc - shs I (fields: 0 U diag^-1, 1 first
  // super, 2 multipliers, 3 second super, 4 iterate; interchanges in PB)
  const double tiny = 2.2e-16;
  for (int w = 0; w < nw; ++w) pbits[w * IV_T + t] = 0u;
  {
    double a = ds[bs] - shs, bsup = es[bs] * sc;
    for (int i = bs; i < bt; ++i) {
      const double sub = es[i] * sc;
      const double a1 = ds[i + 1] - shs, b1 = (i + 1 < bt) ? es[i + 1] * sc : 0.0;
      if (fabs(a) >= fabs(sub)) {   // no interchange (one reciprocal per row on the chain, not two divisions)
        const double ra = 1.0 / ((fabs(a) < tiny) ? copysign(tiny, a) : a);
        const double m = (a == 0.0) ? 0.0 : sub * ra;
        FW(0, i) = ra;
        FW(1, i) = bsup;
        FW(2, i) = m;
        FW(3, i) = 0.0;
        a = a1 - m * bsup;
        bsup = b1;
      } else {                      // rows i and i+1 swap
        const double rs = 1.0 / sub;
        const double m = a * rs;
        FW(0, i) = rs;
        FW(1, i) = a1;
        FW(2, i) = m;
        FW(3, i) = b1;
        PB(i) |= 1u << (i & 31);
        a = bsup - m * a1;
        bsup = -m * b1;
      }
    }
    FW(0, bt) = 1.0 / ((fabs(a) < tiny) ? copysign(tiny, a) : a);
  }
  for (int i = bs; i <= bt; ++i) {
    const uint64_t hsh = ((uint64_t)(k + 1) * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)(i + 1) * 0xC2B2AE3D27D4EB4FULL);
    const uint64_t m2 = (hsh ^ (hsh >> 29)) * 0xBF58476D1CE4E5B9ULL;
    FW(4, i) = (double)((m2 >> 11) & 0xFFFFF) / 1048576.0 - 0.5 + ((i & 1) ? 0.25 : -0.25);
  }
  for (int iter = 0; iter < 3; ++iter) {
    // forward: L^-1 with the recorded interchanges
    double xi = FW(4, bs);
    for (int i = bs; i < bt; ++i) {
      const double xn = FW(4, i + 1);
      const double m = FW(2, i);
      if ((PB(i) >> (i & 31)) & 1u) {
        FW(4, i) = xn;
        xi = fma(-m, xn, xi);
      } else {
        FW(4, i) = xi;
        xi = fma(-m, xi, xn);
      }
    }
    // back: U x = y
    double x2 = 0.0, x1 = xi * FW(0, bt);
    FW(4, bt) = x1;
    double amax = fabs(x1);
    for (int i = bt - 1; i >= bs; --i) {
      const double x0 = (FW(4, i) - FW(1, i) * x1 - FW(3, i) * x2) * FW(0, i);
      FW(4, i) = x0;
      amax = fmax(amax, fabs(x0));
      x2 = x1;
      x1 = x0;
    }
    // normalise (scaled by the max entry first: the solve grows by up to 1 / (eps |T|))
    const double inv0 = 1.0 / amax;
    double s2 = 0.0;
    for (int i = bs; i <= bt; ++i) {
      const double v = FW(4, i) * inv0;
      s2 = fma(v, v, s2);
    }
    const double inv = inv0 / sqrt(s2);
    for (int i = bs; i <= bt; ++i) FW(4, i) *= inv;
  }
  for (int i = 0; i < n; ++i) Z[(size_t)k * n + i] = (i >= bs && i <= bt) ? FW(4, i) : 0.0;
#undef FW
#undef PB
}

size_t inviter_smem(int n, int iv_t) {
  return sizeof(double) * (3 * (size_t)n + (size_t)5 * n * iv_t) + sizeof(unsigned) * ((n + 31) / 32) * iv_t;
}

// Compact-WY factors of the reflectors in chunks of FQ_C (LAPACK dlarft, forward / columnwise):
// H_j0 ... H_{j0+C-1} = I - V_c T_c V_c^T with T_c upper triangular, T_jj = tau_j,
// T[0:j, j] = -tau_j T[0:j, 0:j] (V_c^T v_j)[0:j].  One CTA per chunk.
constexpr int FQ_C = 16;
template <int TNMAX>
__global__ void __launch_bounds__(TT)
wy_t_kernel(int n, const double* __restrict__ V, const double* __restrict__ tau, double* __restrict__ Tout) {
  extern __shared__ double vs_dyn[];
  double (*vs)[TNMAX] = reinterpret_cast<double (*)[TNMAX]>(vs_dyn);   // [FQ_C][TNMAX]
  __shared__ double g[FQ_C][FQ_C + 1];
  __shared__ double tt[FQ_C][FQ_C + 1];
  const int j0 = blockIdx.x * FQ_C;
  const int nc = min(FQ_C, n - 2 - j0);
  for (int idx = threadIdx.x; idx < FQ_C * n; idx += TT) {
    const int c = idx / n, i = idx - c * n;
    vs[c][i] = c < nc ? V[(size_t)(j0 + c) * n + i] : 0.0;
  }
  __syncthreads();
  {   // Gram of the chunk: thread (a, b)
    const int a = threadIdx.x / FQ_C, b = threadIdx.x % FQ_C;
    double acc0 = 0.0, acc1 = 0.0;
    int i = 0;
    for (; i + 1 < n; i += 2) {
      acc0 = fma(vs[a][i], vs[b][i], acc0);
      acc1 = fma(vs[a][i + 1], vs[b][i + 1], acc1);
    }
    if (i < n) acc0 = fma(vs[a][i], vs[b][i], acc0);
    g[a][b] = acc0 + acc1;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int j = 0; j < FQ_C; ++j) {
      const double tj = j < nc ? tau[j0 + j] : 0.0;
      // lane r < j: T[r, j] = -tau_j sum_{q = r}^{j-1} T[r, q] g[q, j]
      double v = 0.0;
      if (lane < j)
        for (int q = lane; q < j; ++q) v = fma(tt[lane][q], g[q][j], v);
      __syncwarp();
      if (lane < FQ_C) tt[lane][j] = lane < j ? -tj * v : (lane == j ? tj : 0.0);
      __syncwarp();
    }
    for (int idx = lane; idx < FQ_C * FQ_C; idx += 32)
      Tout[(size_t)blockIdx.x * FQ_C * FQ_C + idx] = tt[idx / FQ_C][idx % FQ_C];
  }
}

// Q = H_0 H_1 ... H_{n-3} (H_j = I - tau_j v_j v_j^T), row by row: row i of Q is e_i^T H_0 H_1 ...,
// so per chunk x <- x - ((x V_c) T_c) V_c^T, no data shared between rows.  The chunk's 16 dots are
// independent (their butterfly reductions interleave) instead of one serial reduction per
// reflector.  Each warp carries FQ_R rows; V_c and T_c are staged in shared memory for the CTA.
constexpr int FQ_R = 2;
template <int TNMAX>
__global__ void __launch_bounds__(TT)
formq_kernel(int n, const double* __restrict__ V, const double* __restrict__ Tw, double* __restrict__ Q) {
  extern __shared__ double vs_dyn[];
  double (*vs)[TNMAX] = reinterpret_cast<double (*)[TNMAX]>(vs_dyn);   // [FQ_C][TNMAX]
  __shared__ double ts[FQ_C][FQ_C];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row0 = (blockIdx.x * (TT / 32) + warp) * FQ_R;
  double x[FQ_R][TNMAX / 32];
#pragma unroll
  for (int r = 0; r < FQ_R; ++r)
#pragma unroll
    for (int q = 0; q < TNMAX / 32; ++q) x[r][q] = (lane + 32 * q == row0 + r) ? 1.0 : 0.0;
  const int nchunks = (n - 2 + FQ_C - 1) / FQ_C;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int j0 = ch * FQ_C;
    const int nc = min(FQ_C, n - 2 - j0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < FQ_C * TNMAX; idx += TT) {
      const int c = idx / TNMAX, i = idx - c * TNMAX;
      vs[c][i] = (c < nc && i < n) ? V[(size_t)(j0 + c) * n + i] : 0.0;
    }
    ts[threadIdx.x / FQ_C][threadIdx.x % FQ_C] = Tw[(size_t)ch * FQ_C * FQ_C + threadIdx.x];
    __syncthreads();
    double u[FQ_R][FQ_C];
#pragma unroll
    for (int c = 0; c < FQ_C; ++c) {
#pragma unroll
      for (int r = 0; r < FQ_R; ++r) u[r][c] = 0.0;
#pragma unroll
      for (int q = 0; q < TNMAX / 32; ++q) {
        const double vv = vs[c][lane + 32 * q];
#pragma unroll
        for (int r = 0; r < FQ_R; ++r) u[r][c] = fma(x[r][q], vv, u[r][c]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < FQ_C; ++c)
#pragma unroll
        for (int r = 0; r < FQ_R; ++r) u[r][c] += __shfl_xor_sync(0xffffffffu, u[r][c], o);
    // u <- u T (upper triangular): u'_j = sum_{i <= j} u_i T[i, j], in place from the top
#pragma unroll
    for (int j = FQ_C - 1; j >= 0; --j)
#pragma unroll
      for (int r = 0; r < FQ_R; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i <= j; ++i) acc = fma(u[r][i], ts[i][j], acc);
        u[r][j] = acc;
      }
    __syncwarp();   // keeps the compiler from holding all of V_c in registers across the phases
#pragma unroll
    for (int q = 0; q < TNMAX / 32; ++q)
#pragma unroll
      for (int c = 0; c < FQ_C; ++c) {
        const double vv = vs[c][lane + 32 * q];
#pragma unroll
        for (int r = 0; r < FQ_R; ++r) x[r][q] = fma(-u[r][c], vv, x[r][q]);
      }
  }
#pragma unroll
  for (int r = 0; r < FQ_R; ++r) {
    const int row = row0 + r;
    if (row >= n) continue;
#pragma unroll
    for (int q = 0; q < TNMAX / 32; ++q) {
      const int c = lane + 32 * q;
      if (c < n) Q[(size_t)c * n + row] = x[r][q];
    }
  }
}

// max |G - I| over the n x n Gram matrix (one CTA)
__global__ void __launch_bounds__(1024) orth_defect_kernel(int n, const double* __restrict__ G, double* __restrict__ out) {
  __shared__ double red[32];
  double m = 0.0;
  const int lane = threadIdx.x & 31;
  for (int j = threadIdx.x >> 5; j < n; j += 32)
    for (int i = lane; i < n; i += 32) {
      const double x = G[(size_t)j * n + i] - (i == j ? 1.0 : 0.0);
      m = fmax(m, x == x ? fabs(x) : 1e300);   // fmax drops NaN: map it to huge
    }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int k = 0; k < 32; ++k) r = fmax(r, red[k]);
    *out = r;
  }
}

// RLD_TRIDIAG: 1 = per-warp slots (tridiag_kernel), 2 = per-CTA slots with more warps
// (tridiag2_kernel); default: 1 for n <= 288, 2 above
int tridiag_variant(int n) {
  static const int v = getenv("RLD_TRIDIAG") ? atoi(getenv("RLD_TRIDIAG")) : 0;
  return v ? v : (n <= TNMAX ? 1 : 2);   // measured: 1.00 vs 1.18 ms at n = 266, 3.54 vs 3.24 ms at 522
}

template <int NMAX, int TTH, int IVT, int TTH2>
void tri_eigh_launch(int n, const double* A, double* w, double* d, double* e, double* tau, double* V, double* Z,
                     double* Q, double* Tw, cudaStream_t st, cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join) {
  constexpr size_t tsm = tridiag_smem_t<NMAX, TTH>();
  constexpr size_t tsm2 = tridiag2_smem_t<NMAX, TTH2>();
  const size_t vsm = sizeof(double) * FQ_C * NMAX;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(tridiag_kernel<NMAX, TTH>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RLD_CUDA(cudaFuncSetAttribute(tridiag_kernel<NMAX, TTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    RLD_CUDA(cudaFuncSetAttribute(tridiag2_kernel<NMAX, TTH2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RLD_CUDA(cudaFuncSetAttribute(tridiag2_kernel<NMAX, TTH2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm2));
    RLD_CUDA(cudaFuncSetAttribute(inviter_kernel<IVT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)inviter_smem(NMAX, IVT)));
    RLD_CUDA(cudaFuncSetAttribute(wy_t_kernel<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
    RLD_CUDA(cudaFuncSetAttribute(formq_kernel<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
  });
  {
    cudaLaunchConfig_t cfg{};
    const bool v2 = tridiag_variant(n) == 2;
    cfg.gridDim = dim3(TCL);
    cfg.blockDim = dim3(v2 ? TTH2 : TTH);
    cfg.dynamicSmemBytes = v2 ? tsm2 : tsm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (v2)
      RLD_CUDA(cudaLaunchKernelEx(&cfg, tridiag2_kernel<NMAX, TTH2>, n, A, d, e, tau, V));
    else
      RLD_CUDA(cudaLaunchKernelEx(&cfg, tridiag_kernel<NMAX, TTH>, n, A, d, e, tau, V));
    RLD_LAUNCH_CHECK();
  }
  // Q (reflectors -> WY -> rows of Q) on the side stream, overlapping the eigenvalue and
  // eigenvector kernels of T on `st`; joined by the caller
  RLD_CUDA(cudaEventRecord(fork, st));
  RLD_CUDA(cudaStreamWaitEvent(st2, fork, 0));
  wy_t_kernel<NMAX><<<(unsigned)ceil_div(n - 2, FQ_C), TT, vsm, st2>>>(n, V, tau, Tw);
  RLD_LAUNCH_CHECK();
  formq_kernel<NMAX><<<(unsigned)ceil_div(n, (TT / 32) * FQ_R), TT, vsm, st2>>>(n, V, Tw, Q);
  RLD_LAUNCH_CHECK();
  RLD_CUDA(cudaEventRecord(join, st2));
  bisect_kernel<<<(unsigned)ceil_div(32 * (int64_t)n, 256), 256, sizeof(double) * 2 * n, st>>>(n, d, e, w);
  RLD_LAUNCH_CHECK();
  inviter_kernel<IVT><<<(unsigned)ceil_div(n, IVT), IVT, inviter_smem(n, IVT), st>>>(n, d, e, w, Z);
  RLD_LAUNCH_CHECK();
}

}  // namespace

void orth_defect(int n, const double* G, double* out, cudaStream_t st) {
  orth_defect_kernel<<<1, 1024, 0, st>>>(n, G, out);
  RLD_LAUNCH_CHECK();
}

bool tri_eigh(int n, const double* A, double* w, DevBuf& scratch, double** Zout, double** Qout, double** spare,
              cudaStream_t st, cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join) {
  static const int env = getenv("RLD_TRI_EIG") ? atoi(getenv("RLD_TRI_EIG")) : 1;
  if (!env || n < 3 || n > TNMAX_L) return false;
  // scratch: d e tau | V (n x n) | Z (n x n) | Q (n x n) | WY factors (n x n) | spare (3 n x n)
  const size_t nn = (size_t)n * n;
  scratch.reserve(sizeof(double) * (3 * (size_t)n + 7 * nn));
  double* d = scratch.as<double>();
  double* e = d + n;
  double* tau = e + n;
  double* V = tau + n;
  double* Z = V + nn;
  double* Q = Z + nn;
  double* work = Q + nn;
  double* Tw = work;   // compact-WY T factors, FQ_C^2 per chunk (<= n^2 in all)
  if (n <= TNMAX)
    tri_eigh_launch<TNMAX, TT, 16, 512>(n, A, w, d, e, tau, V, Z, Q, Tw, st, st2, fork, join);
  else
    tri_eigh_launch<TNMAX_L, TT_L, 8, 384>(n, A, w, d, e, tau, V, Z, Q, Tw, st, st2, fork, join);
  RLD_CUDA(cudaStreamWaitEvent(st, join, 0));
  *Zout = Z;
  *Qout = Q;
  *spare = work + nn;   // 3 n^2 doubles
  return true;
}

}  // namespace rld
