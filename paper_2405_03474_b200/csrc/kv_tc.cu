// K x block products on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Y[c, i] = sum_j K[i, j] V[c, j] for a stored float32 K (the HBM-streaming
// path of BASELINE configs 2-3; reference call sites src/estimators.py:72 and
// src/precond.py:186, 189).
//
// One persistent CTA per SM, 20 warps:
//   warp 0       TMA producer: K tile (128 rows x 32 fp32, 128B-swizzled) plus the
//                B tiles (NT vectors x 32 fp32: tf32-hi, and lo for 3xTF32) per
//                k-step into an S-stage shared-memory ring (full/empty mbarriers).
//   warps 4-11   converters (two per TMEM lane quarter, 16 of the 32 k-columns each):
//                thread = one K row; it reads its values from the swizzled tile (or
//                generates them from the points), splits them into tf32 hi + lo
//                (lo exact in fp32) and tcgen05.st's them into one of NABUF TMEM
//                A-operand buffers, so the tensor core never re-reads A from SMEM.
//   warp 1       MMA issuer (whole warp walks the pipeline so every descriptor is
//                warp-uniform; one elected lane issues).  3xTF32 per 8-wide k chunk:
//                  NT == 32: D[2NT] += Ahi [Bhi; Blo] + Alo [Bhi; Blo] (two N = 64
//                            instructions -- small N costs the same ~45 cycles as
//                            N = 64, so stacking hi/lo B halves the issue count);
//                  NT >= 64: D[NT] += Ahi Bhi + Ahi Blo + Alo Bhi.
//                1xTF32 (optional sketch mode): D[NT] += A Bhi.
//   warps 12-19  accumulator drain (two warps per TMEM lane quarter, one half of
//                the result columns each).
//   warp 2       TMEM allocation owner.
//
// Accuracy: the tensor core rounds its fp32 accumulator toward zero, so a long
// accumulation drifts (measured -2e-4 relative at n = 16384, -9e-4 at 65536).
// The MMAs therefore accumulate only GROUP k-steps into one of two TMEM
// accumulators; the drain warps add each finished group into fp32 registers
// with round-to-nearest while the tensor core fills the other accumulator.
//
// Work split: "stream-K" -- the tiles x k-steps space is cut into equal
// contiguous ranges, so every SM streams the same number of K bytes; a tile
// shared by several CTAs leaves per-CTA partial sums that kv_tc_reduce adds in
// fixed CTA order, in float64 (deterministic).  Column passes (more vectors than
// one TMEM accumulator holds) run as concurrent CTA groups of the same launch so
// K streams from HBM about once.
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"

namespace rld {

namespace {

constexpr int TC_BM = 128;          // K rows per tile (UMMA M)
constexpr int TC_BK = 32;           // fp32 k-elements per step (one 128-byte swizzle row)
constexpr int TC_THREADS = 640;   // 20 warps: TMA, MMA, TMEM owner, idle, 8 converters, 8 drains
constexpr int GROUP = 4;            // k-steps accumulated in TMEM before the register flush
constexpr int NABUF = 4;            // TMEM A-operand buffers (converters run up to 3 steps ahead)
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;  // 16 KB

// CTA b works on column pass b % npass over stream-K range b / npass.
struct TcParams {
  int64_t total;    // tiles * ks
  int ks;           // k-steps per tile
  int tiles;
  int npass;        // column passes in this launch
  int segs;         // partial slots per tile
  int stages;
  uint32_t tmem_cols;
  float* partial;   // [npass][tiles][segs][NT][128]
  int debug;        // profiling knob (RLD_TC_DEBUG): 1 = skip A stores, 2 = skip MMAs, 4 = skip A loads
  // on-the-fly kernel tiles (src/kernels.py:40-46, 72)
  const float* pts;  // [8][ldp] float32: coordinate rows x,y,z,w (hi) then x,y,z,w (lo)
  int64_t ldp;
  int64_t n, row0, rows;
  int family;
  float a2, gscale, s5, diag;  // amplitude^2, log2(e) / (2 l^2), sqrt(5) / l, a^2 + jitter
  float la2;                   // log2(amplitude^2), folded into the exponent
};

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed FP32x2 helpers (sm_100 FADD2 / FMUL2 / FFMA2), lanes = (lo 32 bits, hi 32 bits)
__device__ __forceinline__ uint64_t pk(float a, float b) {
  return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ float pk_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float pk_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Two K entries from packed squared distances (src/kernels.py:40-46), float32.
template <int FAM>
__device__ __forceinline__ uint64_t kernel_pair(const TcParams& p, uint64_t r2) {
  if (FAM == RLD_RBF) {   // a^2 2^(-g r^2) = 2^(log2 a^2 - g r^2)
    const uint64_t t = fma2(r2, pk(-p.gscale, -p.gscale), pk(p.la2, p.la2));
    return pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t)));
  }
  const float a = pk_lo(r2), b = pk_hi(r2);
  const float ra = a > 0.f ? a * rsqrtf(a) : 0.f, rb = b > 0.f ? b * rsqrtf(b) : 0.f;
  const uint64_t u = mul2(pk(ra, rb), pk(p.s5, p.s5));
  const uint64_t poly = fma2(u, fma2(u, pk(1.0f / 3.0f, 1.0f / 3.0f), pk(1.f, 1.f)), pk(1.f, 1.f));
  const uint64_t t = fma2(u, pk(-1.4426950408889634f, -1.4426950408889634f), pk(p.la2, p.la2));
  return mul2(poly, pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t))));
}

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

// On-the-fly K: the stage carries the 32 column points of the k-step (TMA box of
// the coordinate-major point array [8][ldp]: rows x,y,z,w hi then x,y,z,w lo -- a
// double-float split of the float64 coordinates, so differences of close points
// keep ~48 bits) instead of a K tile; the converter warps generate the tile with
// packed FP32x2 arithmetic (FFMA2/FADD2/FMUL2) and MUFU ex2/rsqrt.
constexpr uint32_t PTS_BYTES = 1024;

template <int MODE, int NT, bool OTF = false>
struct TcShape {
  static constexpr bool STACK = MODE == 3 && NT == 32;  // [Bhi; Blo] as one N = 2 NT operand
  static constexpr int DW = STACK ? 2 * NT : NT;       // accumulator columns
  static constexpr uint32_t B_BYTES = (uint32_t)NT * 128;
  static constexpr uint32_t A_REGION = OTF ? PTS_BYTES : A_BYTES;
  static constexpr uint32_t STAGE = A_REGION + B_BYTES * (MODE == 3 ? 2 : 1);
  static constexpr uint32_t ASTRIDE = MODE == 3 ? 64 : 32;  // TMEM columns per A buffer (hi | lo)
  static constexpr uint32_t A_COL0 = 2 * DW;
  static constexpr int TMEM_NEED = 2 * DW + NABUF * (int)ASTRIDE;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(NT % 32 == 0 && NT <= 128, "NT");
};

template <int MODE, int NT, bool OTF, int DIM, int FAM>
__global__ void __launch_bounds__(TC_THREADS, 1)
kv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
             const __grid_constant__ CUtensorMap tmBlo, const TcParams p) {
  using Sh = TcShape<MODE, NT, OTF>;
  constexpr int DW = Sh::DW;
  constexpr uint32_t B_BYTES = Sh::B_BYTES, STAGE = Sh::STAGE, ASTRIDE = Sh::ASTRIDE, A_COL0 = Sh::A_COL0;
  constexpr uint32_t AR = Sh::A_REGION;   // K tile (stored) or column points (on the fly)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw so the compiler keeps the shared
  // address space (plain C++ loads compile to LDS and are ordered by the mbarrier asm)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* afull = empty + S;          // [NABUF]
  uint64_t* aempty = afull + NABUF;     // [NABUF]
  uint64_t* accfull = aempty + NABUF;   // [2]
  uint64_t* accempty = accfull + 2;     // [2]
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
      ptx::mbar_init(&afull[b], 8);
      ptx::mbar_init(&aempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&accfull[b], 1);
      ptx::mbar_init(&accempty[b], 8);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, Sh::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (beg < end) {
    if (warp == 0) {
      // ---------------- TMA producer (whole warp walks the ring; one elected lane issues)
      for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
        const int s = it.s;
        ptx::mbar_wait_sleep(&empty[s], it.ph ^ 1);
        if (ptx::elect_one()) {
          uint8_t* st = smem + (size_t)s * STAGE;
          if (OTF) {
            ptx::mbar_arrive_expect_tx(&full[s], STAGE);
            ptx::tma_load_2d(st, &tmA, &full[s], it.kstep * TC_BK, 0);   // 32 column points, 8 coordinate rows
          } else {
            ptx::mbar_arrive_expect_tx(&full[s], p.debug == 4 ? STAGE - AR : STAGE);
            if (p.debug != 4) ptx::tma_load_2d(st, &tmA, &full[s], it.kstep * TC_BK, it.tile * TC_BM);
          }
          ptx::tma_load_2d(st + AR, &tmBhi, &full[s], it.kstep * TC_BK, b_row0);
          if (MODE == 3) ptx::tma_load_2d(st + AR + B_BYTES, &tmBlo, &full[s], it.kstep * TC_BK, b_row0);
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = ptx::idesc_tf32(TC_BM, DW);
      const uint64_t desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smem + AR));
      constexpr uint64_t LO_OFF = (uint64_t)(B_BYTES >> 4);   // Blo rows, in descriptor units
      int64_t gi = -1;  // group index
      for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
        const int s = it.s;
        const int b = it.abuf();
        const bool gstart = it.group_start(), gend = it.group_end();
        if (gstart) {
          ++gi;
          if (gi >= 2) ptx::mbar_wait(&accempty[gi & 1], (uint32_t)(((gi >> 1) - 1) & 1));
        }
        ptx::mbar_wait(&full[s], it.ph);
        ptx::mbar_wait(&afull[b], it.aphase());
        ptx::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(gi & 1) * DW;
        const uint32_t a0 = tmem + A_COL0 + ASTRIDE * b;
        const uint64_t bdesc = desc0 + (uint64_t)((s * STAGE) >> 4);
        if (ptx::elect_one()) {
          if (p.debug != 2) {
#pragma unroll
            for (int kk = 0; kk < TC_BK / 8; ++kk) {
              const uint64_t bd = bdesc + 2 * kk;  // +32 bytes along k
              const uint32_t acc = (gstart && kk == 0) ? 0u : 1u;
              if (MODE == 1) {
                ptx::mma_tf32_ts(d, a0 + 8 * kk, bd, idesc, acc);
              } else if (Sh::STACK) {
                ptx::mma_tf32_ts(d, a0 + 8 * kk, bd, idesc, acc);        // D += Ahi [Bhi; Blo]
                ptx::mma_tf32_ts(d, a0 + 32 + 8 * kk, bd, idesc, 1u);    // D += Alo [Bhi; Blo]
              } else {
                ptx::mma_tf32_ts(d, a0 + 8 * kk, bd, idesc, acc);            // D += Ahi Bhi
                ptx::mma_tf32_ts(d, a0 + 8 * kk, bd + LO_OFF, idesc, 1u);    // D += Ahi Blo
                ptx::mma_tf32_ts(d, a0 + 32 + 8 * kk, bd, idesc, 1u);        // D += Alo Bhi
              }
            }
          }
          ptx::tc_commit(&empty[s]);
          ptx::tc_commit(&aempty[b]);
          if (gend) ptx::tc_commit(&accfull[gi & 1]);
        }
        __syncwarp();
      }
    } else if (warp >= 4 && warp < 12) {
      // ---------------- converters: warp 4 + q + 4h owns TMEM lanes 32q..32q+31 (K rows) and
      // the 16 k-columns [16h, 16h + 16) of every step
      const int q = (warp - 4) & 3, hsel = (warp - 4) >> 2;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      const int e0 = 16 * hsel;
      int cur_tile = -1;
      uint64_t xh2[4] = {0, 0, 0, 0}, xl2[4] = {0, 0, 0, 0};   // this row's point, packed twice (on the fly)
      int64_t grow = 0;
      for (StepIter it(beg, end, p.ks, S); it.valid(); it.next()) {
        const int s = it.s;
        const int b = it.abuf();
        const int64_t j = it.j;
        uint32_t hi[16], lo[16];
        if (OTF) {
          if (it.tile != cur_tile) {
            cur_tile = it.tile;
            const int64_t lr = (int64_t)cur_tile * TC_BM + row;
            grow = p.row0 + lr;
            if (lr < p.rows) {
#pragma unroll
              for (int k = 0; k < DIM; ++k) {
                const float h = p.pts[k * p.ldp + grow], l = p.pts[(4 + k) * p.ldp + grow];
                xh2[k] = pk(h, h);
                xl2[k] = pk(l, l);
              }
            }
          }
          ptx::mbar_wait(&full[s], it.ph);
          const float* pp = reinterpret_cast<const float*>(smem + (size_t)s * STAGE) + e0;   // [8][32] + half
          const int64_t j0 = (int64_t)it.kstep * TC_BK + e0;
          // warp-uniform: does this half step hold a diagonal entry of these rows, or columns >= n?
          const int64_t wrow0 = p.row0 + (int64_t)cur_tile * TC_BM + q * 32;
          const bool fix = (j0 < wrow0 + 32 && j0 + 16 > wrow0) || (j0 + 16 > p.n);
          const uint64_t neg1 = pk(-1.f, -1.f);
          if (p.debug == 6) {   // profiling: skip the generation math
#pragma unroll
            for (int e = 0; e < 16; ++e) hi[e] = lo[e] = __float_as_uint(pp[e]);
          } else
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            uint64_t r2a = 0, r2b = 0;   // entries (e, e+1) and (e+2, e+3)
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
              const uint4 ch = *reinterpret_cast<const uint4*>(pp + k * 32 + e);
              const uint4 cl = *reinterpret_cast<const uint4*>(pp + (4 + k) * 32 + e);
              const uint64_t cha = (uint64_t)ch.x | ((uint64_t)ch.y << 32), chb = (uint64_t)ch.z | ((uint64_t)ch.w << 32);
              const uint64_t cla = (uint64_t)cl.x | ((uint64_t)cl.y << 32), clb = (uint64_t)cl.z | ((uint64_t)cl.w << 32);
              const uint64_t da = add2(fma2(cha, neg1, xh2[k]), fma2(cla, neg1, xl2[k]));  // (xh-ch)+(xl-cl)
              const uint64_t db = add2(fma2(chb, neg1, xh2[k]), fma2(clb, neg1, xl2[k]));
              r2a = fma2(da, da, r2a);
              r2b = fma2(db, db, r2b);
            }
            uint64_t kv[2] = {kernel_pair<FAM>(p, r2a), kernel_pair<FAM>(p, r2b)};
            if (fix) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                float v0 = pk_lo(kv[h]), v1 = pk_hi(kv[h]);
                const int64_t c0 = j0 + e + 2 * h;
                v0 = (c0 == grow) ? p.diag : (c0 < p.n ? v0 : 0.f);
                v1 = (c0 + 1 == grow) ? p.diag : (c0 + 1 < p.n ? v1 : 0.f);
                kv[h] = pk(v0, v1);
              }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t u0 = (uint32_t)kv[h], u1 = (uint32_t)(kv[h] >> 32);
              const int ee = e + 2 * h;
              if (MODE == 3) {
                const uint32_t h0 = u0 & 0xFFFFE000u, h1 = u1 & 0xFFFFE000u;
                hi[ee] = h0;
                hi[ee + 1] = h1;
                const uint64_t l2 = fma2((uint64_t)h0 | ((uint64_t)h1 << 32), neg1, kv[h]);   // v - hi (exact)
                lo[ee] = (uint32_t)l2;
                lo[ee + 1] = (uint32_t)(l2 >> 32);
              } else {
                hi[ee] = u0;
                hi[ee + 1] = u1;
              }
            }
          }
        } else {
          ptx::mbar_wait(&full[s], it.ph);
          const uint8_t* rowp = smem + (size_t)s * STAGE + row * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = 4 * hsel + c;   // 16-byte chunk of the 128-byte row
            const float4 v = *reinterpret_cast<const float4*>(rowp + ((cc ^ (row & 7)) << 4));
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
        }
        if (j >= NABUF) ptx::mbar_wait(&aempty[b], (uint32_t)(((j / NABUF) - 1) & 1));
        ptx::tc_fence_after();
        const uint32_t ta = tmem + lane_base + A_COL0 + ASTRIDE * b + e0;
        if (p.debug != 1) {
          ptx::tmem_st_32x32b_x16(ta, hi);
          if (MODE == 3) ptx::tmem_st_32x32b_x16(ta + 32, lo);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[b]);
      }
    } else if (warp >= 12) {
      // ---------------- accumulator drain: warp 12 + q + 4h owns TMEM lanes 32q..32q+31 and
      // result columns [h NT/2, (h+1) NT/2); finished groups are added to fp32 registers
      // (round-to-nearest), a finished segment is stored to the partial buffer
      constexpr int HALF = NT / 2;
      const int q = (warp - 12) & 3, hsel = (warp - 12) >> 2;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      const int c_base = hsel * HALF;
      float acc[HALF];
#pragma unroll
      for (int c = 0; c < HALF; ++c) acc[c] = 0.f;
      int64_t gi = -1;
      int tile = (int)(beg / p.ks);
      int64_t seg_lo = beg;
      while (seg_lo < end) {
        const int64_t seg_hi = std::min<int64_t>(end, (int64_t)(tile + 1) * p.ks);
        for (int64_t gs = seg_lo; gs < seg_hi; gs += GROUP) {
        ++gi;
        const bool seg_end = gs + GROUP >= seg_hi;
        const int buf = (int)(gi & 1);
        ptx::mbar_wait_sleep(&accfull[buf], (uint32_t)((gi >> 1) & 1));
        ptx::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < HALF; c0 += 16) {
          uint32_t v[16];
          ptx::tmem_ld_32x32b_x16(tmem + lane_base + (uint32_t)(buf * DW + c_base + c0), v);
          if (Sh::STACK) {
            uint32_t w[16];
            ptx::tmem_ld_32x32b_x16(tmem + lane_base + (uint32_t)(buf * DW + NT + c_base + c0), w);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]) + __uint_as_float(w[e]);
          } else {
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&accempty[buf]);
        if (seg_end) {
          const int seg = (int)(cta - cta_of_step((int64_t)tile * p.ks, p.total, G));
          float* P = partial + ((size_t)tile * p.segs + seg) * (size_t)NT * TC_BM;
#pragma unroll
          for (int c = 0; c < HALF; ++c) {
            P[(size_t)(c_base + c) * TC_BM + row] = acc[c];
            acc[c] = 0.f;
          }
        }
        }
        seg_lo = seg_hi;
        ++tile;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, Sh::TMEM_COLS);
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

template <int MODE, int NT, bool OTF, int DIM, int FAM>
void launch_tc(const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl, TcParams p, int64_t grid,
               cudaStream_t st) {
  using Sh = TcShape<MODE, NT, OTF>;
  const size_t extra = 1024 + 8 * 64;
  const int smem_cap = max_smem_optin() - 1024;
  p.stages = (int)std::min<size_t>(8, (smem_cap - extra) / Sh::STAGE);
  p.tmem_cols = Sh::TMEM_COLS;
  const size_t smem = p.stages * Sh::STAGE + extra;
  RLD_CUDA(cudaFuncSetAttribute(kv_tc_kernel<MODE, NT, OTF, DIM, FAM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  kv_tc_kernel<MODE, NT, OTF, DIM, FAM><<<(unsigned)grid, TC_THREADS, smem, st>>>(mA, mBh, mBl, p);
  RLD_LAUNCH_CHECK();
}

template <int MODE>
void launch_tc_stored(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                      const TcParams& p, int64_t grid, cudaStream_t st) {
  switch (nt) {
    case 32: launch_tc<MODE, 32, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    case 64: launch_tc<MODE, 64, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    case 96: launch_tc<MODE, 96, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    default: launch_tc<MODE, 128, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
  }
}

template <int DIM, int FAM>
void launch_tc_otf_nt(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                      const TcParams& p, int64_t grid, cudaStream_t st) {
  switch (nt) {
    case 32: launch_tc<3, 32, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
    case 64: launch_tc<3, 64, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
    default: launch_tc<3, 128, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
  }
}

// on-the-fly tiles: 3xTF32 only; d = 1 runs as DIM 2 (zero padding)
void launch_tc_otf(int d, int family, int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                   const TcParams& p, int64_t grid, cudaStream_t st) {
  if (family == RLD_RBF) {
    if (d <= 2) launch_tc_otf_nt<2, RLD_RBF>(nt, mA, mBh, mBl, p, grid, st);
    else if (d == 3) launch_tc_otf_nt<3, RLD_RBF>(nt, mA, mBh, mBl, p, grid, st);
    else launch_tc_otf_nt<4, RLD_RBF>(nt, mA, mBh, mBl, p, grid, st);
  } else {
    if (d <= 2) launch_tc_otf_nt<2, RLD_MATERN52>(nt, mA, mBh, mBl, p, grid, st);
    else if (d == 3) launch_tc_otf_nt<3, RLD_MATERN52>(nt, mA, mBh, mBl, p, grid, st);
    else launch_tc_otf_nt<4, RLD_MATERN52>(nt, mA, mBh, mBl, p, grid, st);
  }
}

// 2-D map over the coordinate-major split points [8][ldp] fp32: box {32, 8} = the
// 32 column points of one k-step
CUtensorMap make_points_map(const float* pts, int64_t n, int64_t ldp) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)n, 8};
  cuuint64_t strides[1] = {(cuuint64_t)ldp * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, 8};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(pts), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled (points) failed (" + std::to_string((int)r) + ")");
  return m;
}

}  // namespace

bool kv_tc_supported(const KvOperand& op) {
  if (op.dtype != RLD_FP32) return false;
  if (op.K == nullptr) return op.pts4 != nullptr && op.kp.d <= 4 && op.tc_mode == 3;   // on the fly
  return (op.ldk % 4) == 0 && (reinterpret_cast<uintptr_t>(op.K) % 16) == 0;
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
  // vectors per pass: <= 128 (two TMEM accumulators + A buffers within 512 columns)
  const int npass = (int)ceil_div(m, 128);
  int width = (int)(ceil_div(ceil_div(m, npass), 32) * 32);
  if (op.K == nullptr && width == 96) width = 128;   // on-the-fly kernels come in NT = 32, 64, 128
  const int64_t Gl = std::min<int64_t>(std::max(1, G / npass), total);
  int segs = 1;
  for (int t = 0; t < tiles; ++t) {
    const int64_t x0 = (int64_t)t * ks;
    segs = (int)std::max<int64_t>(segs, cta_of_step(x0 + ks - 1, total, Gl) - cta_of_step(x0, total, Gl) + 1);
  }
  const bool otf = op.K == nullptr;
  const int64_t ldp = ceil_div(n, 4) * 4;
  const CUtensorMap mA = otf ? make_points_map(op.pts4, n, ldp)
                             : make_map(static_cast<const float*>(op.K), n, rows, op.ldk, TC_BM);
  TcParams p{};
  p.pts = op.pts4;
  p.ldp = ldp;
  p.n = n;
  p.row0 = op.row0;
  p.rows = rows;
  p.family = op.kp.family;
  p.a2 = (float)op.kp.a2;
  p.gscale = (float)(op.kp.inv_2l2 * 1.4426950408889634);
  p.s5 = (float)op.kp.s5_over_l;
  p.diag = (float)op.kp.diag;
  p.la2 = (float)std::log2(op.kp.a2);
  p.total = total;
  p.ks = ks;
  p.tiles = tiles;
  p.npass = npass;
  p.segs = segs;
  {
    static const int dbg = getenv("RLD_TC_DEBUG") ? atoi(getenv("RLD_TC_DEBUG")) : 0;
    p.debug = dbg;
  }
  ws.tc_partial.reserve(sizeof(float) * (size_t)npass * tiles * segs * width * TC_BM);
  p.partial = ws.tc_partial.as<float>();
  const CUtensorMap mBh = make_map(ws.bhi.as<float>(), n, m, ldb, width);
  const CUtensorMap mBl = mode == 3 ? make_map(ws.blo.as<float>(), n, m, ldb, width) : mBh;
  if (otf) {
    launch_tc_otf(op.kp.d, op.kp.family, width, mA, mBh, mBl, p, Gl * npass, st);
  } else {
    if (mode == 3)
      launch_tc_stored<3>(width, mA, mBh, mBl, p, Gl * npass, st);
    else
      launch_tc_stored<1>(width, mA, mBh, mBl, p, Gl * npass, st);
  }
  const int64_t count = m * rows;
  const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 16);
  kv_tc_reduce<<<blocks, 256, 0, st>>>(p.partial, total, Gl, ks, tiles, segs, width, m, rows, Y, ldy);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
