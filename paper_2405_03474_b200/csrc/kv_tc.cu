// K x block products on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Y[c, i] = sum_j K[i, j] V[c, j] for a stored float32 K (the HBM-streaming
// path of BASELINE configs 2-3; reference call sites src/estimators.py:72 and
// src/precond.py:186, 189).
//
// Per CTA (one per SM, persistent, 8 warps):
//   warp 0      TMA producer: K tile (128 rows x 32 fp32, 128B-swizzled) and the
//               B tiles (NT vectors x 32 fp32: hi, and lo for 3xTF32) per k-step,
//               into an S-stage shared-memory ring guarded by full/empty mbarriers.
//   warps 4-7   converters: each thread owns one K row; it reads its 32 values
//               from the swizzled tile, splits them into tf32 hi + lo (lo exact
//               in fp32), and tcgen05.st's them into a double-buffered TMEM
//               A-operand region (the tensor core never re-reads A from shared
//               memory).  The same warps drain the accumulators (below).
//   warp 1      MMA issuer (one thread): per 8-wide k chunk, D += Ahi*Bhi +
//               Ahi*Blo + Alo*Bhi (3xTF32, ~fp32 accuracy) or D += A*B (1xTF32),
//               A from TMEM, B from SMEM descriptors; tcgen05.commit releases
//               the SMEM stage and the TMEM A buffer.
//   warp 2      TMEM allocation owner.
//
// Accuracy: the tensor core rounds its fp32 accumulator toward zero, so a long
// accumulation drifts (measured -2e-4 relative at n = 16384, -9e-4 at 65536).
// The MMA therefore accumulates only GROUP k-steps into one of two TMEM
// accumulators; the converter warps add each finished group into fp32
// registers with round-to-nearest, one group behind (double buffering keeps
// the tensor core busy meanwhile).
//
// Work split: "stream-K" -- the tiles x k-steps space is cut into gridDim.x
// contiguous ranges of equal length, so every SM streams the same number of K
// bytes; a tile shared by several CTAs leaves per-CTA partial sums that
// kv_tc_reduce adds in fixed CTA order, in float64 (deterministic).
#include <cuda.h>

#include <mutex>

#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"

namespace rld {

namespace {

constexpr int TC_BM = 128;          // K rows per tile (UMMA M)
constexpr int TC_BK = 32;           // fp32 k-elements per step (one 128-byte swizzle row)
constexpr int TC_THREADS = 256;
constexpr int GROUP = 4;            // k-steps accumulated in TMEM before the register flush
constexpr int NABUF = 4;            // TMEM A-operand buffers (converter runs up to 3 steps ahead)
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;  // 16 KB

// A launch covers `npass` column passes of NT vectors each: CTA b works on pass
// b % npass over stream-K range b / npass, so the CTAs that need the same K rows
// run concurrently and K streams from HBM about once (L2 serves the other passes).
struct TcParams {
  int64_t total;    // tiles * ks
  int ks;           // k-steps per tile
  int tiles;
  int npass;        // column passes in this launch
  int segs;         // partial slots per tile
  int stages;
  uint32_t tmem_cols;
  float* partial;   // [npass][tiles][segs][NT][128]
};

__host__ __device__ __forceinline__ int64_t cta_of_step(int64_t x, int64_t total, int64_t G) {
  // the CTA whose range [c*total/G, (c+1)*total/G) contains step x
  return ((x + 1) * G - 1) / total;
}

// Walks a CTA's contiguous range of (tile, k-step) pairs with running counters
// (no 64-bit divisions in the pipeline loops).
struct StepIter {
  int64_t g, end, j;
  int ks, kstep, tile, gpos, s, S;
  uint32_t ph;
  __device__ __forceinline__ StepIter(int64_t beg, int64_t end_, int ks_, int S_)
      : g(beg), end(end_), j(0), ks(ks_), gpos(0), s(0), S(S_), ph(0) {
    tile = (int)(beg / ks_);
    kstep = (int)(beg - (int64_t)tile * ks_);
  }
  __device__ __forceinline__ bool valid() const { return g < end; }
  __device__ __forceinline__ bool group_start() const { return gpos == 0; }
  __device__ __forceinline__ bool seg_end() const { return g + 1 == end || kstep + 1 == ks; }
  __device__ __forceinline__ bool group_end() const { return seg_end() || gpos + 1 == GROUP; }
  __device__ __forceinline__ int abuf() const { return (int)(j & (NABUF - 1)); }
  __device__ __forceinline__ uint32_t aphase() const { return (uint32_t)((j / NABUF) & 1); }
  __device__ __forceinline__ void next() {
    gpos = group_end() ? 0 : gpos + 1;
    ++g;
    ++j;
    if (++kstep == ks) {
      kstep = 0;
      ++tile;
    }
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }
};

template <int MODE, int NT>
__global__ void __launch_bounds__(TC_THREADS, 1)
kv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
             const __grid_constant__ CUtensorMap tmBlo, const TcParams p) {
  static_assert(NT % 32 == 0 && (MODE == 3 ? NT <= 64 : NT <= 128), "NT");
  // accumulator width: 3xTF32 multiplies [Bhi; Blo] (2 NT rows) in one instruction and
  // folds the two halves in the drain; 1xTF32 multiplies Bhi (NT rows)
  constexpr int DW = MODE == 3 ? 2 * NT : NT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t B_BYTES = (uint32_t)NT * 128;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES * (MODE == 3 ? 2 : 1);
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* afull = empty + S;       // [NABUF]
  uint64_t* aempty = afull + NABUF;  // [NABUF]
  uint64_t* accfull = aempty + NABUF;  // [2]
  uint64_t* accempty = accfull + 2;  // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pass = (int)(blockIdx.x % p.npass);
  const int64_t G = gridDim.x / p.npass, cta = blockIdx.x / p.npass;
  const int64_t beg = cta * p.total / G, end = (cta + 1) * p.total / G;
  const int b_row0 = pass * NT;
  float* const partial = p.partial + (size_t)pass * p.tiles * p.segs * NT * TC_BM;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmBhi);
    if (MODE == 3) ptx::tma_prefetch_desc(&tmBlo);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NABUF; ++b) {
      ptx::mbar_init(&afull[b], 4);
      ptx::mbar_init(&aempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&accfull[b], 1);
      ptx::mbar_init(&accempty[b], 4);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, p.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // TMEM columns: accumulators [0, DW) and [DW, 2DW); A buffer b at A_COL0 + ASTRIDE b: hi [+0, +32), lo [+32, +64)
  constexpr uint32_t A_COL0 = 2 * DW;
  constexpr uint32_t ASTRIDE = MODE == 3 ? 64 : 32;

  if (beg < end) {
    if (warp == 0) {
      if (lane == 0) {
        // ---------------- TMA producer
        for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
          const int s = it.s;
          ptx::mbar_wait(&empty[s], it.ph ^ 1);
          uint8_t* st = smem + (size_t)s * STAGE;
          ptx::mbar_arrive_expect_tx(&full[s], STAGE);
          ptx::tma_load_2d(st, &tmA, &full[s], it.kstep * TC_BK, it.tile * TC_BM);
          ptx::tma_load_2d(st + A_BYTES, &tmBhi, &full[s], it.kstep * TC_BK, b_row0);
          if (MODE == 3) ptx::tma_load_2d(st + A_BYTES + B_BYTES, &tmBlo, &full[s], it.kstep * TC_BK, b_row0);
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc = ptx::idesc_tf32(TC_BM, DW);
        int64_t gi = -1;  // group index
        for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
          const int s = it.s;
          const int b = it.abuf();
          const bool gstart = it.group_start(), gend = it.group_end();
          if (gstart) {
            ++gi;
            if (gi >= 2) ptx::mbar_wait(&accempty[gi & 1], (uint32_t)(((gi >> 1) - 1) & 1));
          }
          const uint32_t d = tmem + (uint32_t)(gi & 1) * DW;
          ptx::mbar_wait(&full[s], it.ph);
          ptx::mbar_wait(&afull[b], it.aphase());
          ptx::tc_fence_after();
          const uint32_t sB = ptx::smem_u32(smem + (size_t)s * STAGE + A_BYTES);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 8; ++kk) {
            const uint32_t a_hi = tmem + A_COL0 + ASTRIDE * b + 8 * kk;
            const uint64_t bd = ptx::smem_desc_sw128(sB + 32 * kk);   // [Bhi; Blo] rows (3xTF32) or Bhi
            const uint32_t acc = (gstart && kk == 0) ? 0u : 1u;
            ptx::mma_tf32_ts(d, a_hi, bd, idesc, acc);                 // D += Ahi [Bhi; Blo]
            if (MODE == 3) ptx::mma_tf32_ts(d, a_hi + 32, bd, idesc, 1u);  // D += Alo [Bhi; Blo]
          }
          ptx::tc_commit(&empty[s]);
          ptx::tc_commit(&aempty[b]);
          if (gend) ptx::tc_commit(&accfull[gi & 1]);
        }
      }
    } else if (warp >= 4) {
      // ---------------- converters + accumulator drain (warp q owns TMEM lanes 32q..32q+31)
      const int q = warp - 4;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      float acc[NT];
#pragma unroll
      for (int c = 0; c < NT; ++c) acc[c] = 0.f;
      // finished groups waiting to be drained (at most two in flight)
      int64_t pend_gi[2], pend_tile[2];
      bool pend_seg[2];
      int npend = 0;

      auto drain = [&](int64_t gi, bool seg_end, int64_t tile) {
        const int buf = (int)(gi & 1);
        ptx::mbar_wait(&accfull[buf], (uint32_t)((gi >> 1) & 1));
        ptx::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < NT; c0 += 32) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(buf * DW + c0), v);
          if (MODE == 3) {
            uint32_t w[32];
            ptx::tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(buf * DW + NT + c0), w);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[c0 + e] += __uint_as_float(v[e]) + __uint_as_float(w[e]);
          } else {
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[c0 + e] += __uint_as_float(v[e]);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&accempty[buf]);
        if (seg_end) {
          const int seg = (int)(cta - cta_of_step(tile * (int64_t)p.ks, p.total, G));
          float* P = partial + ((size_t)tile * p.segs + seg) * (size_t)NT * TC_BM;
#pragma unroll
          for (int c = 0; c < NT; ++c) {
            P[(size_t)c * TC_BM + row] = acc[c];
            acc[c] = 0.f;
          }
        }
      };

      int64_t gi = -1;
      for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
        const int s = it.s;
        const int b = it.abuf();
        const int64_t j = it.j;
        if (it.group_start()) ++gi;
        ptx::mbar_wait(&full[s], it.ph);
        const uint32_t rowp = ptx::smem_u32(smem + (size_t)s * STAGE + row * 128);
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = ptx::lds128(rowp + ((c ^ (row & 7)) << 4));
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t ub = __float_as_uint(vv[e]);
            if (MODE == 3) {
              const uint32_t hb = ub & 0xFFFFE000u;
              hi[4 * c + e] = hb;
              lo[4 * c + e] = __float_as_uint(vv[e] - __uint_as_float(hb));
            } else {
              hi[4 * c + e] = ub;
            }
          }
        }
        if (j >= NABUF) ptx::mbar_wait(&aempty[b], (uint32_t)(((j / NABUF) - 1) & 1));
        ptx::tc_fence_after();
        const uint32_t ta = tmem + lane_base + A_COL0 + ASTRIDE * b;
        ptx::tmem_st_32x32b_x32(ta, hi);
        if (MODE == 3) ptx::tmem_st_32x32b_x32(ta + 32, lo);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[b]);

        // drain groups that finished at earlier steps (their MMAs do not wait on this step)
        for (int k = 0; k < npend; ++k) drain(pend_gi[k], pend_seg[k], pend_tile[k]);
        npend = 0;
        if (it.group_end()) {
          pend_gi[npend] = gi;
          pend_seg[npend] = it.seg_end();
          pend_tile[npend] = it.tile;
          ++npend;
        }
      }
      for (int k = 0; k < npend; ++k) drain(pend_gi[k], pend_seg[k], pend_tile[k]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, p.tmem_cols);
}

// Y[c * ldy + i] = sum over the tile's segments of the partials (float64 accumulation, fixed order)
__global__ void kv_tc_reduce(const float* __restrict__ P, int64_t total, int64_t G, int ks, int tiles, int segs,
                             int nt, int64_t m, int64_t rows, double* __restrict__ Y, int64_t ldy) {
  const int64_t count = m * rows;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    const int64_t pass = c / nt, cc = c % nt;
    const int64_t tile = i / TC_BM, r = i % TC_BM;
    const int64_t x0 = tile * ks;
    const int nseg = (int)(cta_of_step(x0 + ks - 1, total, G) - cta_of_step(x0, total, G) + 1);
    const float* Pp = P + (size_t)pass * tiles * segs * nt * TC_BM;
    double s = 0.0;
    for (int k = 0; k < nseg; ++k) s += (double)Pp[(((size_t)tile * segs + k) * nt + cc) * TC_BM + r];
    Y[c * ldy + i] = s;
  }
}

// B operand rows from float64 V: hi = tf32(v) (3xTF32) or fp32(v) (1xTF32), lo = fp32(v - hi)
__global__ void kv_tc_split(const double* __restrict__ V, int64_t ldv, int64_t m, int64_t n, int64_t ldb, int mode,
                            float* __restrict__ Bhi, float* __restrict__ Blo) {
  const int64_t count = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, j = e % n;
    const double v = V[c * ldv + j];
    float h = (float)v;
    if (mode == 3) {
      h = __uint_as_float(__float_as_uint(h) & 0xFFFFE000u);
      Blo[c * ldb + j] = (float)(v - (double)h);
    }
    Bhi[c * ldb + j] = h;
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D fp32 row-major map: inner dim `cols`, outer `rows`, row stride `ld` elements, box {32, box_rows}
CUtensorMap make_map(const float* base, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

int sm_count() {
  int dev = 0, sms = 0;
  RLD_CUDA(cudaGetDevice(&dev));
  RLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

int max_smem_optin() {
  int dev = 0, v = 0;
  RLD_CUDA(cudaGetDevice(&dev));
  RLD_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return v;
}

template <int MODE, int NT>
void launch_tc(const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl, TcParams p, int64_t G,
               cudaStream_t st) {
  constexpr size_t stage = A_BYTES + (size_t)NT * 128 * (MODE == 3 ? 2 : 1);
  const size_t extra = 1024 + 8 * 64;
  const int smem_cap = max_smem_optin() - 1024;
  p.stages = (int)std::min<size_t>(8, (smem_cap - extra) / stage);
  constexpr int DW = MODE == 3 ? 2 * NT : NT;
  constexpr int cols = 2 * DW + NABUF * (MODE == 3 ? 64 : 32);
  static_assert(cols <= 512, "TMEM budget");
  p.tmem_cols = cols <= 256 ? 256 : 512;
  const size_t smem = p.stages * stage + extra;
  RLD_CUDA(cudaFuncSetAttribute(kv_tc_kernel<MODE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kv_tc_kernel<MODE, NT><<<(unsigned)G, TC_THREADS, smem, st>>>(mA, mBh, mBl, p);
  RLD_LAUNCH_CHECK();
}

void launch_tc_3(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl, const TcParams& p,
                 int64_t G, cudaStream_t st) {
  if (nt == 32)
    launch_tc<3, 32>(mA, mBh, mBl, p, G, st);
  else
    launch_tc<3, 64>(mA, mBh, mBl, p, G, st);
}

void launch_tc_1(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl, const TcParams& p,
                 int64_t G, cudaStream_t st) {
  switch (nt) {
    case 32: launch_tc<1, 32>(mA, mBh, mBl, p, G, st); break;
    case 64: launch_tc<1, 64>(mA, mBh, mBl, p, G, st); break;
    case 96: launch_tc<1, 96>(mA, mBh, mBl, p, G, st); break;
    default: launch_tc<1, 128>(mA, mBh, mBl, p, G, st); break;
  }
}

}  // namespace

bool kv_tc_supported(const KvOperand& op) {
  return op.dtype == RLD_FP32 && op.K != nullptr && (op.ldk % 4) == 0 &&
         (reinterpret_cast<uintptr_t>(op.K) % 16) == 0;
}

// Y (m x rows, float64, row stride ldy) = V (m x n float64 rows) K^T on the tensor cores.
void kv_product_tc(const KvOperand& op, int mode, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                   KvWorkspace& ws, cudaStream_t st) {
  const int64_t n = op.n, rows = op.rows;
  const int64_t ldb = ceil_div(n, 4) * 4;
  ws.bhi.reserve(sizeof(float) * ldb * m);
  if (mode == 3) ws.blo.reserve(sizeof(float) * ldb * m);
  {
    const int64_t count = m * n;
    const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
    kv_tc_split<<<blocks, 256, 0, st>>>(V, ldv, m, n, ldb, mode, ws.bhi.as<float>(),
                                        mode == 3 ? ws.blo.as<float>() : nullptr);
    RLD_LAUNCH_CHECK();
  }
  const int G = sm_count();
  const int ks = (int)ceil_div(n, TC_BK);
  const int tiles = (int)ceil_div(rows, TC_BM);
  const int64_t total = (int64_t)tiles * ks;
  // vectors per pass: <= 64 for 3xTF32 ([Bhi; Blo] is one N = 2 NT instruction), <= 128 for
  // 1xTF32 (register-resident fp32 accumulators of the drain warps)
  const int npass = (int)ceil_div(m, mode == 3 ? 64 : 128);
  const int width = (int)(ceil_div(ceil_div(m, npass), 32) * 32);
  const int64_t Gl = std::min<int64_t>(std::max(1, G / npass), total);
  int segs = 1;
  for (int t = 0; t < tiles; ++t) {
    const int64_t x0 = (int64_t)t * ks;
    segs = (int)std::max<int64_t>(segs, cta_of_step(x0 + ks - 1, total, Gl) - cta_of_step(x0, total, Gl) + 1);
  }
  const CUtensorMap mA = make_map(static_cast<const float*>(op.K), n, rows, op.ldk, TC_BM);
  TcParams p{};
  p.total = total;
  p.ks = ks;
  p.tiles = tiles;
  p.npass = npass;
  p.segs = segs;
  ws.tc_partial.reserve(sizeof(float) * (size_t)npass * tiles * segs * width * TC_BM);
  p.partial = ws.tc_partial.as<float>();
  const CUtensorMap mBh = make_map(ws.bhi.as<float>(), n, m, ldb, width);
  const CUtensorMap mBl = mode == 3 ? make_map(ws.blo.as<float>(), n, m, ldb, width) : mBh;
  if (mode == 3)
    launch_tc_3(width, mA, mBh, mBl, p, Gl * npass, st);
  else
    launch_tc_1(width, mA, mBh, mBl, p, Gl * npass, st);
  const int64_t count = m * rows;
  const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
  kv_tc_reduce<<<blocks, 256, 0, st>>>(p.partial, total, Gl, ks, tiles, segs, width, m, rows, Y, ldy);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
