// Float64 "reduce over n" products on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
//   C[c, i] = sum_j A[i, j] B[c, j]        A: p x n, B: q x n, C: q x p   (all rows layout)
//
// This one shape covers every float64 product of the estimate whose reduction runs over the n
// points:
//   * K x V with stored float64 K (src/estimators.py:72; src/precond.py:186, 189): A = K's local
//     rows, B = the m vectors, C = the m x rows result;
//   * the Gram matrices of the preconditioner build (src/precond.py:75-76, 94-99; the CholQR of
//     src/linalg.py:159-180): A = B = the w x n block, C = w x w;
//   * the projections B = Q K Q^T (src/precond.py:189) and U^T W (src/precond.py:102-115).
// tcgen05 has no f64 kind, so this is the B200's float64 tensor path.
//
// Kernel design (one CTA = BM x BN outputs over a k range):
//   * warp 8 is the producer: one elected lane streams BK = 16-double (128-byte) k-steps of A and
//     of B into a 4-stage shared-memory ring with TMA (cp.async.bulk.tensor, 128-byte swizzle,
//     out-of-range rows and columns zero-filled by the copy engine), full/empty mbarriers; a
//     stage is released one step late (after the DMMAs that consumed its shared loads issued);
//   * warps 0-7 each own a WM x WN slice of the tile and issue (WM/8) x (WN/8) DMMAs per 4-deep
//     k slice; the m8n8k4 A and B fragments (8 rows x 4 consecutive k of a row-major tile) are
//     single 8-byte shared loads, conflict-free under the 128-byte swizzle (two wavefronts per
//     warp load, the minimum for 256 bytes);
//   * the k range is split across CTAs so that every shape fills the 148 SMs; partial tiles land
//     in a [split][q][p] buffer that split_reduce sums in fixed order (deterministic, no atomics).
#include <cuda.h>

#include <algorithm>
#include <climits>
#include <mutex>

#include "rld_internal.cuh"
#include "rld_kernels.cuh"
#include "tc_ptx.cuh"

namespace rld {

namespace {

constexpr int DM_BK = 16;         // doubles per k-step: one 128-byte swizzle row
constexpr int DM_STAGES = 4;
constexpr int DM_MMA_WARPS = 8;
constexpr int DM_THREADS = (DM_MMA_WARPS + 1) * 32;

template <int BM, int BN>
struct DmmaShape {
  static constexpr int WARPS_N = (BN >= 64 && BN % 16 == 0) ? 2 : 1;
  static constexpr int WARPS_M = DM_MMA_WARPS / WARPS_N;
  static constexpr int WM = BM / WARPS_M;
  static constexpr int WN = BN / WARPS_N;
  static constexpr int MT = WM / 8;
  static constexpr int NT = WN / 8;
  static constexpr int A_BYTES = BM * DM_BK * 8;
  static constexpr int B_BYTES = BN * DM_BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = DM_STAGES * STAGE_BYTES + 1024 + 2 * DM_STAGES * 8;
  static constexpr int MIN_BLOCKS = (MT * NT <= 16) ? 2 : 1;
  static_assert(WM % 8 == 0 && WN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "stage tiles must keep 1024-byte alignment");
};

// byte offset of element (r, k) of a [rows][16] float64 tile written by TMA with SWIZZLE_128B:
// 16-byte granule g = k / 2 of row r lands at granule g ^ (r % 8)
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3));
}

__device__ __forceinline__ double lds_f64(uint32_t saddr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(saddr));
  return v;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN>
__global__ void __launch_bounds__(DM_THREADS, DmmaShape<BM, BN>::MIN_BLOCKS)
gemm_nt_dmma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t p,
                    int64_t q, int64_t n, int64_t kchunk, double* __restrict__ out, int64_t ldo,
                    int64_t split_stride, int sym) {
  using S = DmmaShape<BM, BN>;
  // symmetric (A == B, a Gram): tiles wholly above the diagonal (every c > i) are mirrored by the
  // reduce instead of computed
  if (sym && (int64_t)blockIdx.x * BN >= (int64_t)blockIdx.y * BM + BM) return;
  extern __shared__ __align__(1024) unsigned char dm_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dm_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DM_STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + DM_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = (int64_t)blockIdx.x * BN;   // B rows (vectors): fastest, so CTAs sharing
  const int64_t row0 = (int64_t)blockIdx.y * BM;   // an A tile run together and share it in L2
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min64(n, kbeg + kchunk);
  const int steps = (int)ceil_div(max64(kend - kbeg, 0), DM_BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < DM_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], DM_MMA_WARPS);
    }
    ptx::fence_mbarrier_init();
  }
  __syncthreads();

  if (warp == DM_MMA_WARPS) {   // ---- producer
    if (ptx::elect_one()) {
      ptx::tma_prefetch_desc(&mapA);
      ptx::tma_prefetch_desc(&mapB);
      for (int s = 0; s < steps; ++s) {
        const int st = s % DM_STAGES;
        if (s >= DM_STAGES) ptx::mbar_wait(&empty[st], ((s / DM_STAGES) - 1) & 1);
        unsigned char* a_dst = smem + st * S::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full[st], S::STAGE_BYTES);
        const int32_t kc = (int32_t)(kbeg + (int64_t)s * DM_BK);
        ptx::tma_load_2d(a_dst, &mapA, &full[st], kc, (int32_t)row0);
        ptx::tma_load_2d(a_dst + S::A_BYTES, &mapB, &full[st], kc, (int32_t)col0);
      }
    }
    return;
  }

  // ---- DMMA warps
  const int wm0 = (warp / S::WARPS_N) * S::WM;
  const int wn0 = (warp % S::WARPS_N) * S::WN;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[S::MT][S::NT][2];
#pragma unroll
  for (int i = 0; i < S::MT; ++i)
#pragma unroll
    for (int j = 0; j < S::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t sbase = ptx::smem_u32(smem);
  for (int s = 0; s < steps; ++s) {
    const int st = s % DM_STAGES;
    ptx::mbar_wait(&full[st], (s / DM_STAGES) & 1);
    // Release the PREVIOUS stage only now.  An mbarrier arrive does not wait for this warp's
    // outstanding shared loads (ptxas schedules it among the DMMAs that consume them), so an
    // arrive right after the loads let the next TMA overwrite a row before its LDS had read it
    // (rare single-row errors, worst with concurrent kernels).  Every DMMA of step s-1 -- and so
    // every LDS it consumed -- has issued before the loop back-edge, i.e. before this point.
    if (s > 0 && lane == 0) ptx::mbar_arrive(&empty[(s - 1) % DM_STAGES]);
    const uint32_t a_s = sbase + st * S::STAGE_BYTES;
    const uint32_t b_s = a_s + S::A_BYTES;
#pragma unroll
    for (int kk = 0; kk < DM_BK / 4; ++kk) {
      const int k = kk * 4 + fk;
      double a[S::MT], b[S::NT];
#pragma unroll
      for (int i = 0; i < S::MT; ++i) a[i] = lds_f64(a_s + sw128(wm0 + i * 8 + fr, k));
#pragma unroll
      for (int j = 0; j < S::NT; ++j) b[j] = lds_f64(b_s + sw128(wn0 + j * 8 + fr, k));
#pragma unroll
      for (int i = 0; i < S::MT; ++i)
#pragma unroll
        for (int j = 0; j < S::NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }

  // ---- epilogue: C[c, i] (+ split offset); lane holds rows fr, columns 2 fk + {0, 1}
  double* o = out + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < S::MT; ++i) {
    const int64_t r = row0 + wm0 + i * 8 + fr;
    if (r >= p) continue;
#pragma unroll
    for (int j = 0; j < S::NT; ++j) {
      const int64_t c = col0 + wn0 + j * 8 + 2 * fk;
      if (c < q) o[c * ldo + r] = acc[i][j][0];
      if (c + 1 < q) o[(c + 1) * ldo + r] = acc[i][j][1];
    }
  }
}

// out[c * ldo + r] = beta * out + sum_{s < splits} part[s * stride + c * p + r]   (fixed order);
// sym_bm > 0: entries of the skipped tiles (c >= (r / sym_bm + 1) sym_bm, column tiles of sym_bn)
// come from their mirror (r, c)
__global__ void dmma_split_reduce_kernel(const double* __restrict__ part, int splits, int64_t stride, int64_t q,
                                         int64_t p, double* __restrict__ out, int64_t ldo, double beta, int sym_bm,
                                         int sym_bn) {
  const int64_t total = q * p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / p, r = e % p;
    int64_t src = e;
    if (sym_bm > 0 && (c / sym_bn) * sym_bn >= (r / sym_bm + 1) * sym_bm) src = r * p + c;
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += part[k * stride + src];
    double* d = out + c * ldo + r;
    *d = beta == 0.0 ? s : beta * *d + s;
  }
}

// ---------------------------------------------------------------------------------------------
// "Expand" products: C (q x N) = beta C + S^T X, S: p x q column-major (small), X: p x N rows layout
// (long N = the points).  The basis changes / low-rank expansions of the preconditioner
// (Q R^-1 of the CholQR, A = Q^T U_top, U = A W / sqrt(lambda): src/precond.py:96-99, 191-193;
// src/linalg.py:159-180) and the Woodbury apply w += U (h o U^T w) (src/precond.py:102-115).
// m8n8k4 with M = the q side (fragment rows of the S tile, 128-byte swizzle as above) and N = the
// long side; the X tile arrives as 8-column TMA boxes [BK][8] (64-byte rows, no swizzle), so a
// B fragment (4 consecutive k rows x 8 consecutive columns) is 256 contiguous bytes: conflict-free.
// No split over p (p <= a few thousand): deterministic, one pass.
constexpr int EX_BN = 128;   // columns of X / C per CTA

template <int BQ>
struct ExShape {
  static constexpr int WARPS_Q = BQ >= 64 ? 2 : 1;
  static constexpr int WARPS_N = DM_MMA_WARPS / WARPS_Q;
  static constexpr int WQ = BQ / WARPS_Q;           // 32
  static constexpr int WN = EX_BN / WARPS_N;        // 32 (BQ 64) or 16 (BQ 32)
  static constexpr int MT = WQ / 8, NT = WN / 8;
  static constexpr int S_BYTES = BQ * DM_BK * 8;
  static constexpr int X_BYTES = EX_BN * DM_BK * 8;
  static constexpr int STAGE_BYTES = S_BYTES + X_BYTES;
  static constexpr int SMEM = DM_STAGES * STAGE_BYTES + 1024 + 2 * DM_STAGES * 8;
  static_assert(S_BYTES % 1024 == 0, "S tile must keep 1024-byte alignment");
};

template <int BQ>
__global__ void __launch_bounds__(DM_THREADS, 2)
gemm_expand_dmma_kernel(const __grid_constant__ CUtensorMap mapS, const __grid_constant__ CUtensorMap mapX, int64_t p,
                        int64_t q, int64_t N, double* __restrict__ C, int64_t ldc, double alpha, double beta, int tri) {
  using S = ExShape<BQ>;
  extern __shared__ __align__(1024) unsigned char ex_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(ex_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DM_STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + DM_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j0 = (int64_t)blockIdx.x * EX_BN;
  const int64_t b0 = (int64_t)blockIdx.y * BQ;
  // tri: S is upper triangular (S[k][b] = 0 for k > b, the R^-1 of CholQR): this tile of output rows
  // b0 .. b0 + BQ - 1 only needs k < b0 + BQ
  const int steps = (int)ceil_div(tri ? min64(p, b0 + BQ) : p, DM_BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < DM_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], DM_MMA_WARPS);
    }
    ptx::fence_mbarrier_init();
  }
  __syncthreads();

  if (warp == DM_MMA_WARPS) {   // ---- producer: one S box + EX_BN / 8 X boxes per k-step
    if (ptx::elect_one()) {
      ptx::tma_prefetch_desc(&mapS);
      ptx::tma_prefetch_desc(&mapX);
      for (int s = 0; s < steps; ++s) {
        const int st = s % DM_STAGES;
        if (s >= DM_STAGES) ptx::mbar_wait(&empty[st], ((s / DM_STAGES) - 1) & 1);
        unsigned char* dst = smem + st * S::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full[st], S::STAGE_BYTES);
        const int32_t kc = s * DM_BK;
        ptx::tma_load_2d(dst, &mapS, &full[st], kc, (int32_t)b0);
#pragma unroll 1
        for (int g = 0; g < EX_BN / 8; ++g)
          ptx::tma_load_2d(dst + S::S_BYTES + g * DM_BK * 64, &mapX, &full[st], (int32_t)(j0 + 8 * g), kc);
      }
    }
    return;
  }

  const int wq0 = (warp / S::WARPS_N) * S::WQ;
  const int wn0 = (warp % S::WARPS_N) * S::WN;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[S::MT][S::NT][2];
#pragma unroll
  for (int i = 0; i < S::MT; ++i)
#pragma unroll
    for (int j = 0; j < S::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const uint32_t sbase = ptx::smem_u32(smem);
  for (int s = 0; s < steps; ++s) {
    const int st = s % DM_STAGES;
    ptx::mbar_wait(&full[st], (s / DM_STAGES) & 1);
    if (s > 0 && lane == 0) ptx::mbar_arrive(&empty[(s - 1) % DM_STAGES]);   // see gemm_nt_dmma_kernel
    const uint32_t s_s = sbase + st * S::STAGE_BYTES;
    const uint32_t x_s = s_s + S::S_BYTES;
#pragma unroll
    for (int kk = 0; kk < DM_BK / 4; ++kk) {
      const int k = kk * 4 + fk;
      double a[S::MT], b[S::NT];
#pragma unroll
      for (int i = 0; i < S::MT; ++i) a[i] = lds_f64(s_s + sw128(wq0 + i * 8 + fr, k));
#pragma unroll
      for (int j = 0; j < S::NT; ++j) {
        const int g = (wn0 + j * 8) >> 3;   // 8-column box
        b[j] = lds_f64(x_s + (uint32_t)(g * DM_BK * 64 + k * 64 + fr * 8));
      }
#pragma unroll
      for (int i = 0; i < S::MT; ++i)
#pragma unroll
        for (int j = 0; j < S::NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  // C[b][j]: lane holds row fr, columns 2 fk + {0, 1}
#pragma unroll
  for (int i = 0; i < S::MT; ++i) {
    const int64_t b = b0 + wq0 + i * 8 + fr;
    if (b >= q) continue;
#pragma unroll
    for (int j = 0; j < S::NT; ++j) {
      const int64_t c = j0 + wn0 + j * 8 + 2 * fk;
      double* o = C + b * ldc + c;
      if (c < N) o[0] = beta == 0.0 ? alpha * acc[i][j][0] : fma(beta, o[0], alpha * acc[i][j][0]);
      if (c + 1 < N) o[1] = beta == 0.0 ? alpha * acc[i][j][1] : fma(beta, o[1], alpha * acc[i][j][1]);
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  if (!fn) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// rows x cols float64 row-major (row stride ld elements), box {16, box_rows}, 128-byte swizzle
CUtensorMap map_f64(const double* base, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)DM_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled (f64) failed (" + std::to_string((int)r) + ")");
  return m;
}

int dm_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    RLD_CUDA(cudaGetDevice(&dev));
    RLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

// Split count: every split at least 16 k-steps; the fewest splits whose CTA count fills whole
// waves of the resident slots to >= 95 % (at least 2 waves), else the best fill found.
int64_t choose_splits(int64_t tiles, int64_t n, int64_t slots) {
  const int64_t max_s = std::max<int64_t>(1, n / (DM_BK * 16));
  int64_t best = 1;
  double best_eff = 0.0;
  for (int64_t s = 1; s <= std::min<int64_t>(max_s, 256); ++s) {
    const int64_t units = tiles * s;
    const int64_t waves = ceil_div(units, slots);
    const double eff = (double)units / (double)(waves * slots);
    if (waves >= 2 && eff >= 0.95) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
    if (units >= 64 * slots) break;
  }
  return best;
}

template <int BM, int BN>
void launch_nt(const double* A, int64_t lda, int64_t p, const double* B, int64_t ldb, int64_t q, int64_t n,
               double* C, int64_t ldc, double beta, DevBuf& partial, cudaStream_t st, bool sym) {
  using S = DmmaShape<BM, BN>;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(gemm_nt_dmma_kernel<BM, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM));
  });
  const CUtensorMap ma = map_f64(A, n, p, lda, BM);
  const CUtensorMap mb = map_f64(B, n, q, ldb, BN);
  int64_t tiles = ceil_div(p, BM) * ceil_div(q, BN);
  if (sym) {   // computed tiles only
    tiles = 0;
    for (int64_t ty = 0; ty < ceil_div(p, BM); ++ty)
      for (int64_t tx = 0; tx < ceil_div(q, BN); ++tx) tiles += (tx * BN < ty * BM + BM);
  }
  const int64_t splits_req = choose_splits(tiles, n, (int64_t)dm_sms() * S::MIN_BLOCKS);
  const int64_t kchunk = ceil_div(ceil_div(n, splits_req), DM_BK) * DM_BK;
  const int64_t splits = ceil_div(n, kchunk);
  dim3 grid((unsigned)ceil_div(q, BN), (unsigned)ceil_div(p, BM), (unsigned)splits);
  if (grid.y > 65535u) fail(RLD_ERR_NOT_SUPPORTED, "gemm_nt_f64: too many row tiles");
  if (splits == 1 && beta == 0.0 && !sym) {
    gemm_nt_dmma_kernel<BM, BN><<<grid, DM_THREADS, S::SMEM, st>>>(ma, mb, p, q, n, kchunk, C, ldc, 0, 0);
    RLD_LAUNCH_CHECK();
    return;
  }
  const int64_t stride = q * p;
  partial.reserve(sizeof(double) * stride * splits);
  gemm_nt_dmma_kernel<BM, BN><<<grid, DM_THREADS, S::SMEM, st>>>(ma, mb, p, q, n, kchunk, partial.as<double>(), p,
                                                                   stride, sym ? 1 : 0);
  RLD_LAUNCH_CHECK();
  const int blocks = (int)std::min<int64_t>(ceil_div(stride, 256), (int64_t)dm_sms() * 8);
  dmma_split_reduce_kernel<<<blocks, 256, 0, st>>>(partial.as<double>(), (int)splits, stride, q, p, C, ldc, beta,
                                                   sym ? BM : 0, BN);
  RLD_LAUNCH_CHECK();
}

bool aligned16(const void* ptr, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (ld & 1) == 0;
}

}  // namespace

// rows x cols float64 row-major, box {8, box_rows}, no swizzle (64-byte rows)
CUtensorMap map_f64_b8(const double* base, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {8, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled (f64 x8) failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int BQ>
void launch_expand(const double* Sm, int64_t lds, int64_t p, int64_t q, const double* X, int64_t ldx, int64_t N,
                   double* C, int64_t ldc, double alpha, double beta, cudaStream_t st, bool tri) {
  using S = ExShape<BQ>;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(gemm_expand_dmma_kernel<BQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM));
  });
  const CUtensorMap ms = map_f64(Sm, p, q, lds, BQ);       // S^T as q rows of p
  const CUtensorMap mx = map_f64_b8(X, N, p, ldx, DM_BK);   // X: p rows of N
  dim3 grid((unsigned)ceil_div(N, EX_BN), (unsigned)ceil_div(q, BQ), 1);
  if (grid.y > 65535u) fail(RLD_ERR_NOT_SUPPORTED, "gemm_expand_f64: q too large");
  gemm_expand_dmma_kernel<BQ><<<grid, DM_THREADS, S::SMEM, st>>>(ms, mx, p, q, N, C, ldc, alpha, beta, tri ? 1 : 0);
  RLD_LAUNCH_CHECK();
}

bool gemm_nt_f64_ok(const double* A, int64_t lda, const double* B, int64_t ldb) {
  return aligned16(A, lda) && aligned16(B, ldb);
}

// C (q x p, ld ldc) = beta C + A B^T for A: p x n (ld lda), B: q x n (ld ldb), rows layout.
void gemm_nt_f64(const double* A, int64_t lda, int64_t p, const double* B, int64_t ldb, int64_t q, int64_t n,
                 double* C, int64_t ldc, double beta, DevBuf& partial, cudaStream_t st) {
  if (p <= 0 || q <= 0) return;
  if (n <= 0) {
    if (beta == 0.0)
      for (int64_t c = 0; c < q; ++c) RLD_CUDA(cudaMemsetAsync(C + c * ldc, 0, sizeof(double) * p, st));
    return;
  }
  if (!gemm_nt_f64_ok(A, lda, B, ldb)) fail(RLD_ERR_NOT_SUPPORTED, "gemm_nt_f64 needs 16-byte aligned rows");
  // column-tile width with the least padding of q (ties: the wider tile, fewer A re-reads)
  static const int widths[] = {128, 96, 64, 48, 32, 16};
  int bn = 128;
  int64_t best = INT64_MAX;
  for (int w : widths) {
    const int64_t padded = ceil_div(q, w) * w;
    if (padded < best) {
      best = padded;
      bn = w;
    }
  }
  // a Gram (the same block on both sides): skip the tiles above the diagonal (RLD_GRAM_SYM=0: off)
  static const bool sym_on = !(getenv("RLD_GRAM_SYM") && getenv("RLD_GRAM_SYM")[0] == '0');
  const bool sym = sym_on && A == B && lda == ldb && p == q;
  switch (bn) {
    case 128: launch_nt<128, 128>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
    case 96: launch_nt<128, 96>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
    case 64: launch_nt<128, 64>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
    case 48: launch_nt<128, 48>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
    case 32: launch_nt<128, 32>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
    default: launch_nt<128, 16>(A, lda, p, B, ldb, q, n, C, ldc, beta, partial, st, sym); break;
  }
}

// C (q x N, ld ldc, rows layout) = beta C + alpha S^T X; S: p x q column-major (ld lds), X: p x N
// rows layout (ld ldx).  S and X rows 16-byte aligned (gemm_nt_f64_ok(S, lds, X, ldx)).
void gemm_expand_f64(const double* Sm, int64_t lds, int64_t p, int64_t q, const double* X, int64_t ldx, int64_t N,
                     double* C, int64_t ldc, double alpha, double beta, cudaStream_t st, bool tri_upper) {
  if (q <= 0 || N <= 0) return;
  if (p <= 0) {
    if (beta != 1.0) fail(RLD_ERR_NOT_SUPPORTED, "gemm_expand_f64 with p = 0 needs beta = 1");
    return;
  }
  if (!gemm_nt_f64_ok(Sm, lds, X, ldx)) fail(RLD_ERR_NOT_SUPPORTED, "gemm_expand_f64 needs 16-byte aligned rows");
  if (q <= 32)
    launch_expand<32>(Sm, lds, p, q, X, ldx, N, C, ldc, alpha, beta, st, tri_upper);
  else
    launch_expand<64>(Sm, lds, p, q, X, ldx, N, C, ldc, alpha, beta, st, tri_upper);
}

}  // namespace rld
