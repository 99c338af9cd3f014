// Symmetric positive semi-definite eigensolver for the preconditioner's small matrices
// (B = Q K Q^T, w x w, src/precond.py:189-190, and C = At^T At, k x k, src/precond.py:96) on one
// thread-block cluster: one-sided (Hestenes) block Jacobi.  cuSOLVER's DSYEVD at these sizes is
// ~2.3-2.7 ms of latency-bound tridiagonalisation; this is a single launch plus a sort -- but it
// measured ~10x slower (see small_eigh), so it is opt-in and DSYEVD stays the default.
//
// For symmetric PSD A, rotating columns until they are mutually orthogonal gives A V = U S with
// V orthogonal (the eigenvectors) and S the column norms (the eigenvalues).  Columns are cut into
// 2 CL blocks of BW columns; CTA r holds two blocks ("top", "bottom") in shared memory, the A
// columns and the matching V columns.  A sweep is 2 CL - 1 steps of the circle-method tournament
// over blocks: in a step every CTA orthogonalises all column pairs inside its two blocks (a
// circle-method tournament over its 2 BW columns, one warp per pair, rows over the lanes), then
// the blocks move one seat round the table through DSMEM.  Sweeps repeat until no pair in a sweep
// has |a_p . a_q| > tol |a_p| |a_q|.  Deterministic: fixed orders everywhere.
// Parity with LAPACK eigh is up to eigenvector signs (all uses are sign-invariant) and rotations
// inside (near-)degenerate eigenspaces, which do not change P.
#include "rld_internal.cuh"
#include "rld_device.cuh"
#include "rld_kernels.cuh"

#include <cooperative_groups.h>

namespace rld {

namespace {

constexpr int ECL = 16;            // CTAs per cluster (non-portable size)
constexpr int BW = 9;              // columns per block: 2 ECL BW = 288 >= n
constexpr int EIG_MAX = 2 * ECL * BW;
constexpr int ET = 32 * BW;        // one warp per column pair of a round
constexpr int NPAD = 288;          // rows per stored column (n <= 288)
constexpr int MAX_SWEEPS = 40;

__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// circle method over M = 2 BW players: round r, pair i -> (x, y)
__device__ __forceinline__ void circle_pair(int M, int r, int i, int& x, int& y) {
  if (i == 0) {
    x = r;
    y = M - 1;
  } else {
    x = (r + i) % (M - 1);
    y = (r - i + (M - 1)) % (M - 1);
  }
}

// block tournament over 2 ECL blocks: seat arrays top[ECL], bot[ECL], top[0] fixed
__device__ __forceinline__ void seats(int step, int r, int& top_blk, int& bot_blk) {
  // seat s holds player (s + step) in the rotating ring of 2 ECL - 1 players plus the fixed one;
  // ring order: top[1..ECL-1] then bot[ECL-1..0] (clockwise)
  const int R = 2 * ECL - 1;
  auto ring = [&](int pos) {   // player in ring position pos after `step` rotations
    return ((pos - step) % R + R) % R + 1;   // players 1..R
  };
  // ring positions: top seat s (s >= 1) -> pos s - 1; bottom seat s -> pos (ECL - 1) + (ECL - 1 - s)
  top_blk = (r == 0) ? 0 : ring(r - 1);
  bot_blk = ring((ECL - 1) + (ECL - 1 - r));
}

__global__ void __launch_bounds__(ET)
eig_jacobi_kernel(int n, const double* __restrict__ A, double tol, double* __restrict__ Vout,
                  double* __restrict__ sig, int* __restrict__ sweeps_out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  // two buffers (the blocks of this step, and those of the next pulled in through DSMEM), each
  // [2 (top, bottom)][BW][NPAD] for A and for V
  constexpr int SLOTS = 2 * BW * NPAD;
  auto bufA = [&](int b) { return sm + (size_t)b * 2 * SLOTS; };
  auto bufV = [&](int b) { return sm + (size_t)b * 2 * SLOTS + SLOTS; };
  int cur = 0;
  __shared__ int s_rot;        // rotations this sweep (this CTA)
  __shared__ int s_total;      // cluster total (CTA 0 gathers)
  const int r = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int tb, bb;
  seats(0, r, tb, bb);
  // load this CTA's blocks: A columns, V = identity columns
  for (int slot = 0; slot < 2; ++slot) {
    const int blk = slot == 0 ? tb : bb;
    for (int e = tid; e < BW * NPAD; e += ET) {
      const int c = e / NPAD, i = e % NPAD;
      const int j = blk * BW + c;
      const bool ok = j < n && i < n;
      bufA(0)[slot * BW * NPAD + e] = ok ? A[(size_t)j * n + i] : 0.0;
      bufV(0)[slot * BW * NPAD + e] = (ok && i == j) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int step = 0; step < 2 * ECL - 1; ++step) {
      double* cA = bufA(cur);
      double* cV = bufV(cur);
      // ---- all pairs of the 2 BW local columns: circle method, one warp per pair
      constexpr int M = 2 * BW;
      for (int rr = 0; rr < M - 1; ++rr) {
        for (int pi = warp; pi < BW; pi += ET / 32) {
          int x, y;
          circle_pair(M, rr, pi, x, y);
          double* ap = cA + x * NPAD;   // local column x: slot x / BW, column x % BW (contiguous)
          double* aq = cA + y * NPAD;
          double* vp = cV + x * NPAD;
          double* vq = cV + y * NPAD;
          double al = 0.0, be = 0.0, ga = 0.0;
          for (int i = lane; i < n; i += 32) {
            const double u = ap[i], w = aq[i];
            al = fma(u, u, al);
            be = fma(w, w, be);
            ga = fma(u, w, ga);
          }
          al = warp_sum(al);
          be = warp_sum(be);
          ga = warp_sum(ga);
          if (al > 0.0 && be > 0.0 && fabs(ga) > tol * sqrt(al * be)) {
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
            for (int i = lane; i < n; i += 32) {
              const double u = ap[i], w = aq[i];
              ap[i] = c * u - s * w;
              aq[i] = s * u + c * w;
              const double vu = vp[i], vw = vq[i];
              vp[i] = c * vu - s * vw;
              vq[i] = s * vu + c * vw;
            }
            if (lane == 0) atomicAdd(&s_rot, 1);
          }
        }
        __syncthreads();
      }
      // ---- move the blocks one seat (after the sweep's last step they are back at step 0's seats):
      // pull the new ones from their current holders into the other buffer
      int ntb, nbb;
      seats(step + 1, r, ntb, nbb);
      // find who holds ntb / nbb now
      int src_t = -1, slot_t = 0, src_b = -1, slot_b = 0;
      for (int q = 0; q < ECL; ++q) {
        int t2, b2;
        seats(step, q, t2, b2);
        if (t2 == ntb) { src_t = q; slot_t = 0; }
        if (b2 == ntb) { src_t = q; slot_t = 1; }
        if (t2 == nbb) { src_b = q; slot_b = 0; }
        if (b2 == nbb) { src_b = q; slot_b = 1; }
      }
      csync();   // every CTA finished its rotations of this step
      {
        double* rA = bufA(cur ^ 1);
        double* rV = bufV(cur ^ 1);
        const double2* sA_t = reinterpret_cast<const double2*>(cl.map_shared_rank(cA, src_t) + slot_t * BW * NPAD);
        const double2* sV_t = reinterpret_cast<const double2*>(cl.map_shared_rank(cV, src_t) + slot_t * BW * NPAD);
        const double2* sA_b = reinterpret_cast<const double2*>(cl.map_shared_rank(cA, src_b) + slot_b * BW * NPAD);
        const double2* sV_b = reinterpret_cast<const double2*>(cl.map_shared_rank(cV, src_b) + slot_b * BW * NPAD);
        double2* dA = reinterpret_cast<double2*>(rA);
        double2* dV = reinterpret_cast<double2*>(rV);
        constexpr int H = BW * NPAD / 2;
        for (int e = tid; e < H; e += ET) {
          const double2 a0 = sA_t[e], v0 = sV_t[e], a1 = sA_b[e], v1 = sV_b[e];
          dA[e] = a0;
          dV[e] = v0;
          dA[H + e] = a1;
          dV[H + e] = v1;
        }
      }
      csync();   // all pulls done: the buffers swap
      cur ^= 1;
    }
    // ---- convergence: any rotation anywhere in this sweep?
    csync();
    if (tid == 0) {
      int* tot0 = cl.map_shared_rank(&s_total, 0);
      if (r == 0) *tot0 = 0;
    }
    csync();
    if (tid == 0) atomicAdd(cl.map_shared_rank(&s_total, 0), s_rot);
    csync();
    const int total = *cl.map_shared_rank(&s_total, 0);
    csync();
    if (total == 0) break;
  }
  // ---- eigenvalues = column norms of A V, eigenvectors = V columns; after a full sweep the blocks
  // are back at step 0's seats
  double* cA = bufA(cur);
  double* cV = bufV(cur);
  int ftb, fbb;
  seats(0, r, ftb, fbb);
  for (int slot = 0; slot < 2; ++slot) {
    const int blk = slot == 0 ? ftb : fbb;
    for (int c = warp; c < BW; c += ET / 32) {
      const int j = blk * BW + c;
      if (j >= n) continue;
      const double* a = cA + (slot * BW + c) * NPAD;
      double s2 = 0.0;
      for (int i = lane; i < n; i += 32) s2 = fma(a[i], a[i], s2);
      s2 = warp_sum(s2);
      if (lane == 0) sig[j] = sqrt(s2);
      const double* v = cV + (slot * BW + c) * NPAD;
      for (int i = lane; i < n; i += 32) Vout[(size_t)j * n + i] = v[i];
    }
  }
  if (r == 0 && tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
}

// ascending order of the eigenvalues (ties by index), eigenvectors permuted with them
__global__ void eig_sort_kernel(int n, const double* __restrict__ sig, const double* __restrict__ V,
                                double* __restrict__ w, double* __restrict__ A) {
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    __shared__ int pos;
    if (threadIdx.x == 0) pos = 0;
    __syncthreads();
    const double sj = sig[j];
    int cnt = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double si = sig[i];
      cnt += (si < sj || (si == sj && i < j)) ? 1 : 0;
    }
    atomicAdd(&pos, cnt);
    __syncthreads();
    const int p = pos;
    if (threadIdx.x == 0) w[p] = sj;
    for (int i = threadIdx.x; i < n; i += blockDim.x) A[(size_t)p * n + i] = V[(size_t)j * n + i];
    __syncthreads();
  }
}

}  // namespace

bool small_eigh(int n, double* A, double* w, DevBuf& scratch, int* sweeps, cudaStream_t st) {
  // Opt-in (RLD_SMALL_EIG=1): correct (tests vs LAPACK pass) but ~10x slower than DSYEVD at
  // n = 256-288 (25-27 ms vs 2.3-2.8 ms): every round of the column tournament costs a warp
  // reduction and a sqrt/divide chain plus a block barrier, and a sweep is 31 steps x 17 rounds.
  static const bool on = getenv("RLD_SMALL_EIG") && getenv("RLD_SMALL_EIG")[0] == '1';
  if (!on || n < 2 || n > EIG_MAX || n > NPAD) return false;
  scratch.reserve(sizeof(double) * ((size_t)n * n + n));
  double* V = scratch.as<double>();
  double* sig = V + (size_t)n * n;
  const size_t smem = sizeof(double) * 8 * BW * NPAD;   // 2 buffers x (A, V) x 2 blocks
  static bool attr = false;
  if (!attr) {
    RLD_CUDA(cudaFuncSetAttribute(eig_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RLD_CUDA(cudaFuncSetAttribute(eig_jacobi_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ECL);
  cfg.blockDim = dim3(ET);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ECL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double tol = 4e-16 * n;   // relative orthogonality of converged columns
  RLD_CUDA(cudaLaunchKernelEx(&cfg, eig_jacobi_kernel, n, (const double*)A, tol, V, sig, sweeps));
  RLD_LAUNCH_CHECK();
  eig_sort_kernel<<<std::min(n, 148), 128, 0, st>>>(n, sig, V, w, A);
  RLD_LAUNCH_CHECK();
  return true;
}

}  // namespace rld
