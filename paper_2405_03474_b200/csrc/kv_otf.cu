// On-the-fly K x block products on the tcgen05 kind::f16 tensor cores.
//
// Y[c, i] = sum_j K[i, j] V[c, j] with the K tiles generated from the points
// (BASELINE configs 4-5; reference call sites src/estimators.py:72,
// src/precond.py:186, 189, K entries src/kernels.py:40-46, 72), in float32
// accuracy from three fp16 products:
//
//   K' = 2^sK K and V'_c = 2^eV_c V_c are power-of-two scaled into [2^13, 2^14)
//   (exact), each split into an fp16 head and tail, K' = Kh + Kl, V' = Vh + Vl:
//   Kh = K' with the low 13 fp32 mantissa bits cleared (fp16-exact), Kl = fp16(K' - Kh)
//   (K' - Kh is exact in fp32), so |K' - Kh - Kl| <= 2^-22 |K'| (normal range) or
//   2^-25 absolute (fp16 subnormals, i.e. entries below 2^-27 of the row's scale);
//   D += Kh Vh + Kh Vl + Kl Vh, fp32 accumulation (the dropped Kl Vl is 2^-22).
//   This is the accuracy of the 3xTF32 split of kv_tc.cu (11 + 11 bits) at twice the
//   tensor-core rate per instruction: kind::f16 takes K = 16 per MMA where kind::tf32
//   takes K = 8, so a 64-column k-step costs the instructions a 32-column tf32 step did.
//
// One persistent CTA per SM, 20 warps (the roles of kv_tc.cu):
//   warp 0       TMA producer of the 64 column points of each k-step (2 KB: two
//                [8][32] fp32 blocks of the k-step-blocked point array);
//   warp 2       TMEM owner and TMA producer of the B tiles (NT vectors x 64 fp16,
//                head and tail, 128-byte swizzled, k-step blocked);
//   warps 1, 3   MMA issuers on alternate k-steps, named-barrier baton;
//   converters   thread = one K row: 64 entries per k-step from the points (FFMA2 +
//                MUFU sqrt / ex2), split into fp16 head / tail pairs, tcgen05.st into
//                a TMEM A buffer (2 fp16 per 32-bit column: 32 + 32 columns);
//   drains       add each finished GROUP of k-steps to fp32 registers with
//                round-to-nearest (the tensor core truncates its accumulator).
// The float64 result is 2^-(sK + eV_c) times the fixed-order float64 sum of the
// per-segment partials (kv_otf_reduce).
#include <cuda.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kv_sched.cuh"
#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"

namespace rld {

namespace {

constexpr int OB_M = 128;          // K rows per tile (UMMA M)
constexpr int OB_K = 64;           // k-elements per step (one 128-byte fp16 swizzle row)
constexpr int OTF_THREADS = 640;   // 20 warps
constexpr uint32_t PTS_STAGE_POINTS = 2048;   // 64 column points: [2][8][32] fp32
constexpr int SCALE_TOP = 13;      // scaled magnitudes in [2^13, 2^14)

struct OtfParams {
  Sched sched;
  int mp;               // B rows per k-step block (vectors padded to npass x NT)
  unsigned int* sync;   // phase-1 epoch barrier counters (per pass, or one for all passes)
  int sync_k;
  int sync_all;         // stored K, several passes: one counter, so the passes' CTAs that stream the same
                        // K tiles stay within an L2-sized window and K comes from HBM once
  int ks, tiles, npass, segs;
  int sa, sb;
  float* partial;       // [npass][tiles][segs][NT][128], scaled units
  int wait_mode;
  uint32_t wait_ns;
  const float* pts;     // [ceil(n/64) * 2][8][32] pre-scaled float32 coordinates
  int64_t n, row0, rows;
  const float* rowscale;   // stored K (DIM == 0): per local row 2^s_i with max_j |K_ij| 2^s_i in [2^13, 2^14)
  const uint32_t* skip;    // on the fly: bit k of word [tile][k / 32] set = the tile's k-step k has only
  int skip_wpt;            // exactly-zero fp16 operands (far field in Morton order): no loads, no MMAs
  int ks32;             // stored K: 32-column tiles per row tile of the tiled layout
  float diag;           // 2^sK (a^2 + jitter)
  float la2;            // log2(a^2) + sK
  int family;
  unsigned long long* prof;   // RLD_OTF_PROFILE: per-CTA cycle counters [grid][16], else null
};

// idesc: kind::f16, D f32, A/B f16 K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// two fp32 -> packed fp16x2, `lo` in the low half (the lower k index)
__device__ __forceinline__ uint32_t f16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

template <int FAM>
__device__ __forceinline__ uint64_t kpair(float la2, uint64_t r2) {
  if (FAM == RLD_RBF) {
    const uint64_t t = fma2(r2, pk(-1.f, -1.f), pk(la2, la2));
    return pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t)));
  }
  const uint64_t u = pk(fast_sqrt(pk_lo(r2)), fast_sqrt(pk_hi(r2)));
  const uint64_t poly = fma2(u, fma2(u, pk(1.0f / 3.0f, 1.0f / 3.0f), pk(1.f, 1.f)), pk(1.f, 1.f));
  const uint64_t t = fma2(u, pk(-1.4426950408889634f, -1.4426950408889634f), pk(la2, la2));
  return mul2(poly, pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t))));
}

// 32 K' entries of one converter thread: its row x the 32 column points at `pp`
// ([8][32] fp32), as 16 fp16x2 head words and 16 tail words.  FIX: the block holds a
// diagonal entry of these rows or padding columns >= n (warp-uniform).
template <int DIM, int FAM, bool FIX>
__device__ __forceinline__ void gen32(const OtfParams& p, uint32_t pp, const uint64_t (&xr2)[DIM], int j0, int grow,
                                      int n32, uint32_t (&hw)[16], uint32_t (&lw)[16]) {
  // four entries (two pairs) per iteration; the compiler interleaves consecutive iterations
  // (computing all 16 pairs stage by stage measured slower: register-bound at 96 per thread)
  const uint64_t neg1 = pk(-1.f, -1.f);
#pragma unroll
  for (int e = 0; e < 32; e += 4) {
    uint64_t r2a = 0, r2b = 0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const float4 c = ptx::lds128(pp + 4u * (k * 32 + e));
      const uint64_t da = fma2(pk(c.x, c.y), neg1, xr2[k]);
      const uint64_t db = fma2(pk(c.z, c.w), neg1, xr2[k]);
      r2a = fma2(da, da, r2a);
      r2b = fma2(db, db, r2b);
    }
    uint64_t kv[2] = {kpair<FAM>(p.la2, r2a), kpair<FAM>(p.la2, r2b)};
    if (FIX) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v0 = pk_lo(kv[h]), v1 = pk_hi(kv[h]);
        const int c0 = j0 + e + 2 * h;
        v0 = (c0 == grow) ? p.diag : (c0 < n32 ? v0 : 0.f);
        v1 = (c0 + 1 == grow) ? p.diag : (c0 + 1 < n32 ? v1 : 0.f);
        kv[h] = pk(v0, v1);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t h0 = (uint32_t)kv[h] & 0xFFFFE000u, h1 = (uint32_t)(kv[h] >> 32) & 0xFFFFE000u;
      const uint64_t l2 = fma2((uint64_t)h0 | ((uint64_t)h1 << 32), neg1, kv[h]);   // K' - head (exact)
      const int w = (e >> 1) + h;
      hw[w] = f16x2(__uint_as_float(h0), __uint_as_float(h1));
      lw[w] = f16x2(pk_lo(l2), pk_hi(l2));
    }
  }
}

// 32 stored K entries of one row (one 16 KB tile [128][32] fp32, 128-byte swizzled: chunk c of
// row r at ((c ^ (r & 7)) << 4)) scaled by 2^s (exact) and split into fp16 head / tail words
__device__ __forceinline__ void load32(uint32_t rowp, int row, float rs, uint32_t (&hw)[16], uint32_t (&lw)[16]) {
  const uint64_t neg1 = pk(-1.f, -1.f), sc = pk(rs, rs);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = ptx::lds128(rowp + (uint32_t)((c ^ (row & 7)) << 4));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t kv = mul2(h == 0 ? pk(v.x, v.y) : pk(v.z, v.w), sc);
      const uint32_t h0 = (uint32_t)kv & 0xFFFFE000u, h1 = (uint32_t)(kv >> 32) & 0xFFFFE000u;
      const uint64_t l2 = fma2((uint64_t)h0 | ((uint64_t)h1 << 32), neg1, kv);
      hw[2 * c + h] = f16x2(__uint_as_float(h0), __uint_as_float(h1));
      lw[2 * c + h] = f16x2(pk_lo(l2), pk_hi(l2));
    }
  }
}

// First k-step >= k of row tile t below kend that the skip map keeps (kend if none).
__device__ __forceinline__ int next_kept(const OtfParams& p, int t, int k, int kend) {
  const uint32_t* row = p.skip + (int64_t)t * p.skip_wpt;
  while (k < kend) {
    const uint32_t m = ~__ldg(row + (k >> 5)) & (0xFFFFFFFFu << (k & 31));
    if (m) {
      const int kk = (k & ~31) + __ffs(m) - 1;
      return kk < kend ? kk : kend;
    }
    k = (k & ~31) + 32;
  }
  return kend;
}

// The CTA's (tile, k-step) walk of StepIter (kv_sched.cuh) restricted to the k-steps the skip map
// keeps (all of them without a map): every role walks the same sequence, so the rings, the MMA baton
// and the accumulation groups see only kept steps.  u counts kept steps (ring slot u % S); the
// lookahead (l*) is the next kept step, which decides segment and group ends.
template <bool GRP, bool BR>
struct KeptIter {
  const OtfParams* p;
  int ks, G, R, group;
  int64_t vend;
  int tail_next, tail_k0;
  int v, kstep, tile, round;        // current kept step (raw walk position)
  int lv, lkstep, ltile, lround;    // next kept step
  int u = 0;
  int s = 0, S;
  uint32_t ph = 0;
  int gpos = 0;
  int sb = 0, SB = 1;
  uint32_t phb = 0;
  __device__ __forceinline__ KeptIter(const OtfParams& prm, int64_t cta, int S_, int SB_ = 1)
      : p(&prm), ks(prm.sched.ks), G(prm.sched.G), R(prm.sched.R), group(prm.sched.group), S(S_), SB(SB_) {
    const Sched& sc = prm.sched;
    const int64_t tb = sc.tail_beg(cta), te = sc.tail_end(cta);
    vend = (int64_t)R * ks + (te - tb);
    tail_next = R * G + (int)(tb / ks);
    tail_k0 = (int)(tb - (int64_t)(tb / ks) * ks);
    v = 0;
    round = 0;
    if (R > 0) {
      tile = (int)cta;
      kstep = 0;
    } else {
      tile = tail_next;
      kstep = tail_k0;
    }
    seek(v, kstep, tile, round);
    lv = v; lkstep = kstep; ltile = tile; lround = round;
    if (lv < vend) {
      raw_next(lv, lkstep, ltile, lround);
      seek(lv, lkstep, ltile, lround);
    }
  }
  // one raw step (StepIter::next without the rings)
  __device__ __forceinline__ void raw_next(int& v_, int& k_, int& t_, int& r_) const {
    ++v_;
    if (++k_ == ks) {
      k_ = 0;
      if (r_ < R) {
        if (++r_ < R) {
          t_ += G;
        } else {
          t_ = tail_next;
          k_ = tail_k0;
        }
      } else {
        ++t_;
      }
    }
  }
  // forward to the first kept step at or after the position
  __device__ __forceinline__ void seek(int& v_, int& k_, int& t_, int& r_) const {
    if (!p->skip) return;
    while (v_ < vend) {
      const int kend = (int)min64(ks, (int64_t)k_ + (vend - v_));   // this tile's segment ends here
      const int k2 = next_kept(*p, t_, k_, kend);
      v_ += k2 - k_;
      k_ = k2;
      if (k2 < kend) return;
      // the rest of the segment is skipped: onto the next tile
      --v_;
      k_ = kend - 1;
      raw_next(v_, k_, t_, r_);
    }
  }
  __device__ __forceinline__ bool valid() const { return v < vend; }
  __device__ __forceinline__ bool has_next() const { return lv < vend; }
  __device__ __forceinline__ bool group_start() const { return gpos == 0; }
  __device__ __forceinline__ bool seg_end() const { return !has_next() || ltile != tile; }
  __device__ __forceinline__ bool group_end() const { return seg_end() || gpos + 1 == group; }
  __device__ __forceinline__ void next() {
    if (GRP) gpos = group_end() ? 0 : gpos + 1;
    v = lv; kstep = lkstep; tile = ltile; round = lround;
    if (lv < vend) {
      raw_next(lv, lkstep, ltile, lround);
      seek(lv, lkstep, ltile, lround);
    }
    ++u;
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
    if (BR && ++sb == SB) {
      sb = 0;
      phb ^= 1;
    }
  }
};

// kept k-steps of row tile t in [k0, k0 + len)
__device__ __forceinline__ int kept_count(const OtfParams& p, int t, int k0, int len) {
  if (!p.skip) return len;
  const uint32_t* row = p.skip + (int64_t)t * p.skip_wpt;
  int c = 0;
  for (int k = k0; k < k0 + len;) {
    const int b = k & 31, take = min(32 - b, k0 + len - k);
    const uint32_t mask = (take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1u)) << b;
    c += __popc(~__ldg(row + (k >> 5)) & mask);
    k += take;
  }
  return c;
}

template <int NT>
struct OtfShape {
  static constexpr bool STACK = NT == 32;           // [Bh; Bl] as one N = 64 operand
  static constexpr int DW = STACK ? 2 * NT : NT;    // accumulator columns
  static constexpr uint32_t B_BYTES = (uint32_t)NT * 128;   // NT rows x 64 fp16
  static constexpr uint32_t BST = 2 * B_BYTES;              // head, tail
  static constexpr int NACC = 2;
  static constexpr uint32_t ASTRIDE = 64;           // TMEM columns per A buffer: head 32 | tail 32
  static constexpr uint32_t A_COL0 = NACC * DW;
  static constexpr int DP = NT == 64 ? 1 : 2;       // drain warps per lane quarter
#ifndef RLD_OTF_CP128
#define RLD_OTF_CP128 2
#endif
  // converter warps per lane quarter: 3 at NT = 64 (20 warps); at NT = 128 RLD_OTF_CP128 (2: 20
  // warps, 96 registers; 3: 24 warps, 80 registers)
  static constexpr int CP = NT == 128 ? RLD_OTF_CP128 : 4 - DP;
  static constexpr int THREADS = 32 * (4 + 4 * (CP + DP));
  static constexpr int NABUF = (512 - (int)A_COL0) / (int)ASTRIDE < 8 ? (512 - (int)A_COL0) / (int)ASTRIDE : 8;
  static constexpr int TMEM_NEED = (int)A_COL0 + NABUF * (int)ASTRIDE;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(NABUF > CP, "TMEM A buffers");
  static_assert(NT % 16 == 0 && (NT / DP) % 16 == 0 && NT <= 128, "NT");
};

// DIM > 0: K tiles generated from the points; DIM == 0: stored fp32 K (tiled layout, kgen.cu), two
// 16 KB tiles per 64-column stage, per-row power-of-two scales (the wide products of configs 2-3)
template <int NT, int DIM, int FAM>
__global__ void __launch_bounds__(OtfShape<NT>::THREADS, 1)
kv_otf_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmBh,
              const __grid_constant__ CUtensorMap tmBl, const OtfParams p) {
  using Sh = OtfShape<NT>;
  constexpr uint32_t PTS_STAGE = DIM == 0 ? 32768u : PTS_STAGE_POINTS;
  constexpr int DW = Sh::DW, NACC = Sh::NACC;
  constexpr uint32_t B_BYTES = Sh::B_BYTES, BST = Sh::BST, ASTRIDE = Sh::ASTRIDE, A_COL0 = Sh::A_COL0;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  // B ring first (1024-byte aligned stages for the swizzle atoms), then the points ring
  const int SA = p.sa, SB = p.sb;
  uint8_t* const bring = smem;
  uint8_t* const pring = smem + (size_t)SB * BST;
  uint64_t* kfull = reinterpret_cast<uint64_t*>(pring + (size_t)SA * PTS_STAGE);
  uint64_t* kempty = kfull + SA;
  uint64_t* bfull = kempty + SA;
  uint64_t* bempty = bfull + SB;
  uint64_t* afull = bempty + SB;
  uint64_t* accfull = afull + SB;
  uint64_t* accempty = accfull + NACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accempty + NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bid = blockIdx.x;
  const int pass = (int)(bid % p.npass);
  const int64_t cta = bid / p.npass;
  const int b_row0 = pass * NT;
  float* const partial = p.partial + (size_t)pass * p.tiles * p.segs * NT * OB_M;
  unsigned long long* const prof = p.prof ? p.prof + blockIdx.x * 16 : nullptr;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmP);
    ptx::tma_prefetch_desc(&tmBh);
    ptx::tma_prefetch_desc(&tmBl);
    for (int i = 0; i < SA; ++i) {
      ptx::mbar_init(&kfull[i], 1);
      ptx::mbar_init(&kempty[i], 4);   // one arrive per lane-quarter converter warp of the step
    }
    for (int i = 0; i < SB; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1);
      ptx::mbar_init(&afull[i], 4);
    }
    for (int i = 0; i < NACC; ++i) {
      ptx::mbar_init(&accfull[i], 2);   // one commit per MMA-issuing warp
      ptx::mbar_init(&accempty[i], 4 * Sh::DP);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, Sh::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  const unsigned long long k_start = prof ? clock64() : 0;
  if (StepIter<false, false>(p.sched, cta, 1).valid()) {   // raw schedule: empty segments still get zeros
    if (warp == 0) {
      // ---------------- points producer
      for (KeptIter<false, false> it(p, cta, SA); it.valid(); it.next()) {
        const int s = it.s;
        ptx::mbar_wait_idle(&kempty[s], it.ph ^ 1, p.wait_mode, p.wait_ns);
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(&kfull[s], PTS_STAGE);
          if (DIM == 0)   // tiles 2 kstep, 2 kstep + 1 of row tile `tile`: one 256-row box
            ptx::tma_load_2d(pring + (size_t)s * PTS_STAGE, &tmP, &kfull[s], 0,
                             (it.tile * p.ks32 + 2 * it.kstep) * OB_M);
          else
            ptx::tma_load_2d(pring + (size_t)s * PTS_STAGE, &tmP, &kfull[s], 0, it.kstep * 16);
        }
        __syncwarp();
      }
    } else if (warp == 2) {
      // ---------------- B producer
      int64_t epoch = 0;
      unsigned long long pb[2] = {0, 0};
      for (KeptIter<false, false> it(p, cta, SB); it.valid(); it.next()) {
        const int s = it.s;
        // (no epoch barrier with a skip map: the kept steps differ between CTAs)
        if (p.sync_k > 0 && it.round < p.sched.R && it.v > 0 && (it.kstep & (p.sync_k - 1)) == 0) {
          ++epoch;
          const unsigned long long e0 = prof ? clock64() : 0;
          if (lane == 0) {
            unsigned int* ctr = p.sync + (p.sync_all ? 0 : pass);
            atomicAdd(ctr, 1u);
            const unsigned int target = (unsigned int)(epoch * p.sched.G * (p.sync_all ? p.npass : 1));
            while (*(volatile unsigned int*)ctr < target) __nanosleep(100);
            if (prof) pb[1] += clock64() - e0;
          }
          __syncwarp();
        }
        const unsigned long long b0 = prof ? clock64() : 0;
        ptx::mbar_wait_idle(&bempty[s], it.ph ^ 1, p.wait_mode, p.wait_ns);
        if (prof) pb[0] += clock64() - b0;
        if (ptx::elect_one()) {
          uint8_t* st = bring + (size_t)s * BST;
          const int brow = it.kstep * p.mp + b_row0;
          ptx::mbar_arrive_expect_tx(&bfull[s], BST);
          ptx::tma_load_2d(st, &tmBh, &bfull[s], 0, brow);
          ptx::tma_load_2d(st + B_BYTES, &tmBl, &bfull[s], 0, brow);
        }
        __syncwarp();
      }
      if (prof && lane == 0) {
        prof[11] = pb[0];
        prof[12] = pb[1];
      }
    } else if (warp == 1 || warp == 3) {
      // ---------------- MMA issuers (alternate k-steps, baton through named barriers 1 / 2)
      const int mpar = warp == 3;
      constexpr uint32_t idesc = idesc_f16(128, DW);
      const uint64_t desc0 = ptx::smem_desc_sw128(ptx::smem_u32(bring));
      constexpr uint64_t LO_OFF = (uint64_t)(B_BYTES >> 4);
      int64_t gi = -1;
      unsigned long long pa[5] = {0, 0, 0, 0, 0};
      for (KeptIter<true, false> it(p, cta, SB); it.valid(); it.next()) {
        const bool gstart = it.group_start(), gend = it.group_end();
        if (gstart) ++gi;
        if ((it.u & 1) == mpar) {
          const int s = it.s;
          const unsigned long long t0 = prof ? clock64() : 0;
          if (gstart && gi >= NACC) ptx::mbar_wait(&accempty[gi % NACC], (uint32_t)((gi / NACC - 1) & 1));
          const unsigned long long t1 = prof ? clock64() : 0;
          ptx::mbar_wait(&afull[s], it.ph);
          const unsigned long long t2 = prof ? clock64() : 0;
          ptx::mbar_wait(&bfull[s], it.ph);
          const unsigned long long t3 = prof ? clock64() : 0;
          if (it.u > 0) ptx::named_bar_sync(mpar ? 1 : 2, 64);
          if (prof) {
            pa[0] += t1 - t0;
            pa[1] += t2 - t1;
            pa[2] += t3 - t2;
            pa[3] += clock64() - t3;
            pa[4] += 1;
          }
          ptx::tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(gi % NACC) * DW;
          const uint32_t a0 = tmem + A_COL0 + ASTRIDE * s;
          const uint64_t bdesc = desc0 + (uint64_t)((s * BST) >> 4);
          const bool leader = ptx::elect_one();
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < OB_K / 16; ++kk) {
              const uint64_t bd = bdesc + 2 * kk;   // +32 bytes = 16 fp16 along k
              const uint32_t acc = (gstart && kk == 0) ? 0u : 1u;
              if (Sh::STACK) {
                mma_f16_ts(d, a0 + 8 * kk, bd, idesc, acc);         // D += Kh [Vh; Vl]
                mma_f16_ts(d, a0 + 32 + 8 * kk, bd, idesc, 1u);     // D += Kl [Vh; Vl]
              } else {
                mma_f16_ts(d, a0 + 8 * kk, bd, idesc, acc);             // D += Kh Vh
                mma_f16_ts(d, a0 + 8 * kk, bd + LO_OFF, idesc, 1u);     // D += Kh Vl
                mma_f16_ts(d, a0 + 32 + 8 * kk, bd, idesc, 1u);         // D += Kl Vh
              }
            }
          }
          __syncwarp();
          if (it.has_next()) ptx::named_bar_arrive(mpar ? 2 : 1, 64);
          if (leader) ptx::tc_commit(&bempty[s]);
        }
        if (gend) {
          if (ptx::elect_one()) ptx::tc_commit(&accfull[gi % NACC]);
          __syncwarp();
        }
      }
      if (prof && warp == 1 && lane == 0)
        for (int k = 0; k < 5; ++k) prof[k] = pa[k];
    } else if (warp >= 4 && warp < 4 + 4 * Sh::CP) {
      // ---------------- converters: warp 4 + q + 4 par owns TMEM lanes 32q.. (K rows) and the
      // steps j with j % CP == par; a step's afull arrive is posted after the first half of the
      // warp's next step is generated, so tcgen05.wait::st rarely waits
      const int q = (warp - 4) & 3, par = (warp - 4) >> 2;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      int cur_tile = -1;
      uint64_t xr2[DIM > 0 ? DIM : 1];
#pragma unroll
      for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) xr2[k] = 0;
      float rs = 0.f;   // stored K: this row's scale
      int grow = 0, wrow0 = 0;
      const int n32 = (int)p.n;
      int pend = -1;
      unsigned long long t_post = 0, pc[3] = {0, 0, 0};
      auto post = [&](int buf) {
        const unsigned long long q0 = prof ? clock64() : 0;
        ptx::tmem_wait_st();
        if (prof) t_post += clock64() - q0;
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[buf]);
      };
      KeptIter<false, true> it(p, cta, SA, SB);
      for (int k = 0; k < par; ++k) it.next();
      for (; it.valid(); [&] { for (int k = 0; k < Sh::CP; ++k) it.next(); }()) {
        const int s = it.s, sb = it.sb;
        if (it.tile != cur_tile) {
          cur_tile = it.tile;
          const int lr = cur_tile * OB_M + row;
          wrow0 = (int)p.row0 + cur_tile * OB_M + q * 32;
          grow = wrow0 + lane;
          if (lr < p.rows) {
            if (DIM == 0) {
              rs = p.rowscale[lr];
            } else {
#pragma unroll
              for (int k = 0; k < DIM; ++k) {
                const float x = p.pts[(((int64_t)(grow >> 5) * 8 + k) << 5) + (grow & 31)];
                xr2[k] = pk(x, x);
              }
            }
          }
        }
        const unsigned long long c0 = prof ? clock64() : 0;
        ptx::mbar_wait(&kfull[s], it.ph);
        const unsigned long long c1 = prof ? clock64() : 0;
        if (it.u >= SB) ptx::mbar_wait(&bempty[sb], it.phb ^ 1);   // TMEM A buffer sb free
        if (prof) {
          pc[0] += c1 - c0;
          pc[1] += clock64() - c1;
          pc[2] += 1;
        }
        ptx::tc_fence_after();
        const uint32_t ta = tmem + lane_base + A_COL0 + ASTRIDE * sb;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hw[16], lw[16];
          if constexpr (DIM == 0) {
            load32(ptx::smem_u32(pring + (size_t)s * PTS_STAGE) + 16384u * half + (uint32_t)row * 128u, row, rs, hw,
                   lw);
          } else {
            const uint32_t pp = ptx::smem_u32(pring + (size_t)s * PTS_STAGE) + 1024u * half;
            const int j0 = it.kstep * OB_K + 32 * half;
            const bool fix = (j0 < wrow0 + 32 && j0 + 32 > wrow0) || (j0 + 32 > n32);
            if (!fix) gen32<DIM, FAM, false>(p, pp, xr2, 0, 0, 0, hw, lw);
            else gen32<DIM, FAM, true>(p, pp, xr2, j0, grow, n32, hw, lw);
          }
          if (half == 1) {   // the points stage is read: release it
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&kempty[s]);
          }
          if (half == 0 && pend >= 0) post(pend);
          ptx::tmem_st_32x32b_x16(ta + 16 * half, hw);
          ptx::tmem_st_32x32b_x16(ta + 32 + 16 * half, lw);
        }
        pend = sb;
      }
      if (pend >= 0) post(pend);
      if (prof && warp == 4 && lane == 0) {
        prof[5] = pc[0];
        prof[6] = pc[1];
        prof[7] = pc[2];
        prof[8] = t_post;
      }
    } else {
      // ---------------- accumulator drains: warp 4 + 4 CP + q + 4 h owns TMEM lanes 32q.. and
      // result columns [h NT/DP, (h+1) NT/DP)
      constexpr int HALF = NT / Sh::DP;
      const int dw = warp - (4 + 4 * Sh::CP);
      const int q = dw & 3, hsel = dw >> 2;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      const int c_base = hsel * HALF;
      float acc[HALF];
#pragma unroll
      for (int c = 0; c < HALF; ++c) acc[c] = 0.f;
      int64_t gi = -1;
      unsigned long long pd[2] = {0, 0};
      SegIter si(p.sched, cta);
      int tile = 0, len = 0, seg = 0, k0 = 0;
      while (si.next(tile, len, seg, k0)) {
        const int kept = kept_count(p, tile, k0, len);   // the MMA groups cover the kept k-steps only
        for (int g0 = 0; g0 < kept; g0 += p.sched.group) {
          ++gi;
          const int buf = (int)(gi % NACC);
          const bool any = true;
          const unsigned long long d0 = prof ? clock64() : 0;
          ptx::mbar_wait_idle(&accfull[buf], (uint32_t)((gi / NACC) & 1), p.wait_mode, p.wait_ns);
          if (prof) {
            pd[0] += clock64() - d0;
            pd[1] += 1;
          }
          ptx::tc_fence_after();
          if (any) {
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
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&accempty[buf]);
        }
        float* P = partial + ((size_t)tile * p.segs + seg) * (size_t)NT * OB_M;
#pragma unroll
        for (int c = 0; c < HALF; ++c) {
          if (tile < p.tiles) P[(size_t)(c_base + c) * OB_M + row] = acc[c];
          acc[c] = 0.f;
        }
      }
      if (prof && dw == 0 && lane == 0) {
        prof[9] = pd[0];
        prof[10] = pd[1];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[13] = clock64() - k_start;
  if (warp == 2) ptx::tmem_dealloc(tmem, Sh::TMEM_COLS);
}

// Y[c * ldy + i] = 2^-(sK + eV_c) * (fixed-order float64 sum of the tile's segment partials)
constexpr int RED_COLS = 8;
__global__ void __launch_bounds__(256)
kv_otf_reduce(const float* __restrict__ P, Sched sc, int tiles, int segs, int nt, int64_t m, int64_t rows, int sK,
              const float* __restrict__ rowscale, const unsigned long long* __restrict__ vmax, double* __restrict__ Y,
              int64_t ldy) {
  const int tile = blockIdx.x;
  const int r = threadIdx.x & 127;
  const int64_t i = (int64_t)tile * OB_M + r;
  const int full = sc.R * sc.G;
  int nseg = 1;
  if (tile >= full) {
    const int64_t x0 = (int64_t)(tile - full) * sc.ks;
    nseg = (int)(cta_of_step(x0 + sc.ks - 1, sc.tail_total, sc.G) - cta_of_step(x0, sc.tail_total, sc.G) + 1);
  }
  if (i >= rows) return;
  const int c0 = blockIdx.y * RED_COLS;
#pragma unroll
  for (int q = threadIdx.x >> 7; q < RED_COLS; q += 2) {
    const int c = c0 + q;
    if (c >= m) break;
    const int pass = c / nt, cc = c - pass * nt;
    const float* Pp = P + (size_t)pass * tiles * segs * nt * OB_M + ((size_t)tile * segs * nt + cc) * OB_M + r;
    double s = 0.0;
    for (int k = 0; k < nseg; ++k) s += (double)Pp[(size_t)k * nt * OB_M];
    const double mx = __longlong_as_double((long long)vmax[c]);
    const int ev = mx > 0.0 ? SCALE_TOP - ilogb(mx) : 0;
    if (rowscale)
      Y[(int64_t)c * ldy + i] = ldexp(s, -ev) / (double)rowscale[i];   // exact: powers of two
    else
      Y[(int64_t)c * ldy + i] = ldexp(s, -(sK + ev));
  }
}

// max |V_c| per vector, as the bit pattern of a non-negative double (ordered like the value)
__global__ void kv_otf_vmax(const double* __restrict__ V, int64_t ldv, int64_t n, unsigned long long* __restrict__ vmax) {
  const int64_t c = blockIdx.y;
  double mx = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fabs(V[c * ldv + j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(vmax + c, (unsigned long long)__double_as_longlong(mx));
}

// B operand: V'_c = 2^eV_c V_c split into fp16 head / tail in k-step blocks Bt[ks][mp][64]
// (zero padded for c >= m, j >= n)
__global__ void kv_otf_split(const double* __restrict__ V, int64_t ldv, int64_t m, int64_t n, int64_t mp, int64_t ks,
                             const unsigned long long* __restrict__ vmax, __half* __restrict__ Bh,
                             __half* __restrict__ Bl) {
  const int64_t c = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ks * OB_K) return;
  double v = 0.0;
  if (c < m && j < n) {
    const double mx = __longlong_as_double((long long)vmax[c]);
    v = mx > 0.0 ? ldexp(V[c * ldv + j], SCALE_TOP - ilogb(mx)) : 0.0;
  }
  const int64_t o = ((j >> 6) * mp + c) * OB_K + (j & 63);
  const float f = __uint_as_float(__float_as_uint((float)v) & 0xFFFFE000u);   // fp16-exact head
  const __half h = __float2half_rn(f);
  Bh[o] = h;
  Bl[o] = __double2half(v - (double)__half2float(h));
}

CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* base, int64_t cols, int64_t rows, int64_t ld_bytes,
                        int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled (kv_otf) failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int NT, int DIM, int FAM>
void launch_otf(const CUtensorMap& mP, const CUtensorMap& mBh, const CUtensorMap& mBl, OtfParams p, int64_t grid,
                cudaStream_t st) {
  using Sh = OtfShape<NT>;
  constexpr size_t AST = DIM == 0 ? 32768u : PTS_STAGE_POINTS;   // A-source stage: K tiles or points
  const size_t extra = 1024 + 8 * 64;   // alignment slack + barriers
  const size_t cap = (size_t)max_smem_optin() - extra;
  // stored K: 4 A stages (32 KB each) to cover HBM latency where the B stages are small enough (NT <= 96:
  // config-2 sketch 3.0 -> 2.4 ms); at NT = 128 the fourth TMEM A buffer is worth more (4 B + 2 A
  // stages: config-3 sketch 14 ms, 3 B + 4 A: 18 ms)
  int sb = Sh::NABUF;
  const int min_sb = (DIM == 0 && NT <= 96) ? Sh::CP + 1 : 2;
  const size_t a_need = (DIM == 0 && NT > 96) ? 2 : 4;
  while (sb > min_sb && cap < sb * (size_t)Sh::BST + a_need * AST) --sb;
  p.sb = sb;
  p.sa = (int)std::min<size_t>(12, (cap - sb * (size_t)Sh::BST) / AST);
  // the converter warp of step j (j % CP) reads A-ring slot j % SA: with SA a multiple of CP every
  // slot belongs to one converter warp, so no warp can pass a kfull parity wait a whole ring phase
  // early (SA = 3 with CP = 2 let one warp read a slot still holding the other warp's step)
  p.sa = p.sa / Sh::CP * Sh::CP;
  if (p.sa < Sh::CP) fail(RLD_ERR_NOT_SUPPORTED, "kv_otf: shared memory below one A stage per converter warp");
  const size_t smem = (size_t)p.sa * AST + (size_t)p.sb * Sh::BST + extra;
  auto kern = kv_otf_kernel<NT, DIM, FAM>;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin()));
  });
  kern<<<(unsigned)grid, Sh::THREADS, smem, st>>>(mP, mBh, mBl, p);
  RLD_LAUNCH_CHECK();
}

template <int DIM, int FAM>
void launch_otf_nt(int nt, const CUtensorMap& mP, const CUtensorMap& mBh, const CUtensorMap& mBl, const OtfParams& p,
                   int64_t grid, cudaStream_t st) {
  switch (nt) {
    case 32: launch_otf<32, DIM, FAM>(mP, mBh, mBl, p, grid, st); break;
    case 64: launch_otf<64, DIM, FAM>(mP, mBh, mBl, p, grid, st); break;
    case 96:
      if constexpr (DIM == 0) {   // stored K only: tensor-bound, so less padding pays (config 2: 3 x 96 for 266)
        launch_otf<96, DIM, FAM>(mP, mBh, mBl, p, grid, st);
        break;
      }
      [[fallthrough]];
    default: launch_otf<128, DIM, FAM>(mP, mBh, mBl, p, grid, st); break;
  }
}

}  // namespace

// Per-row scales of a tiled fp32 K: rowscale[i] = 2^s, max_j |K_ij| 2^s in [2^13, 2^14) (1 for a zero
// row).  Thread = row; it reads the row's 32-float segment of every tile.
__global__ void kv_rowscale_tiled(const float* __restrict__ Kt, int64_t rows, int64_t ks32, float* __restrict__ rs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t t = i / OB_M, r = i % OB_M;
  float mx = 0.f;
  for (int64_t k = 0; k < ks32; ++k) {
    const float4* row = reinterpret_cast<const float4*>(Kt + ((t * ks32 + k) * OB_M + r) * 32);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 v = row[c];
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
  rs[i] = mx > 0.f ? ldexpf(1.f, SCALE_TOP - ilogbf(mx)) : 1.f;
}

void kv_rowscales(const float* Kt, int64_t rows, int64_t n, float* rs, cudaStream_t st) {
  if (rows <= 0) return;
  kv_rowscale_tiled<<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(Kt, rows, ceil_div(n, 32), rs);
  RLD_LAUNCH_CHECK();
}

// ---- far-field skip map of the on-the-fly product (points in Morton order).  Box of the points of
// each 128-row tile and of each 64-column k-step, then per (tile, k-step) an upper bound on K from the
// boxes' distance: a k-step whose scaled bound 2^sK K_max is below 2^-27 (4x under the 2^-25 at
// which fp16 head and tail both round to zero) has only exactly-zero operands.
__global__ void otf_boxes(const double* __restrict__ X, int64_t first, int64_t count, int d, int64_t group,
                          int64_t groups, double* __restrict__ box) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  double lo[4], hi[4];
  for (int c = 0; c < 4; ++c) {
    lo[c] = INFINITY;
    hi[c] = -INFINITY;
  }
  const int64_t a = g * group, b = min64(count, a + group);
  for (int64_t i = a; i < b; ++i)
    for (int c = 0; c < d; ++c) {
      const double x = X[(first + i) * d + c];
      lo[c] = fmin(lo[c], x);
      hi[c] = fmax(hi[c], x);
    }
  for (int c = 0; c < 4; ++c) {
    box[g * 8 + c] = lo[c];
    box[g * 8 + 4 + c] = hi[c];
  }
}

__global__ void otf_skip_kernel(const double* __restrict__ tbox, const double* __restrict__ kbox, int64_t tiles,
                                int64_t ks, int wpt, int d, KernelParams kp, double thresh, int64_t row0, int64_t rows,
                                uint32_t* __restrict__ bits) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tiles * wpt) return;
  const int64_t t = e / wpt;
  const int w = (int)(e - t * wpt);
  uint32_t word = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t k = (int64_t)w * 32 + b;
    if (k >= ks) break;
    double r2 = 0.0;
    for (int c = 0; c < d; ++c) {
      const double g = fmax(0.0, fmax(kbox[k * 8 + c] - tbox[t * 8 + 4 + c], tbox[t * 8 + c] - kbox[k * 8 + 4 + c]));
      r2 += g * g;
    }
    // the k-step may hold a diagonal entry of these rows: never skipped (r2 = 0 there anyway)
    const int64_t r_lo = row0 + t * 128, r_hi = row0 + min64(rows, (t + 1) * 128), c_lo = k * 64, c_hi = c_lo + 64;
    if (r_lo < c_hi && c_lo < r_hi) continue;
    if (kernel_value_f64(kp, r2) < thresh) word |= 1u << b;
  }
  bits[e] = word;
}

void otf_skip_map(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, uint32_t* bits,
                  DevBuf& scratch, cudaStream_t st) {
  if (rows <= 0 || kp.d > 4) return;
  const int64_t tiles = ceil_div(rows, OB_M), ks = ceil_div(n, OB_K);
  const int wpt = (int)ceil_div(ks, 32);
  scratch.reserve(sizeof(double) * 8 * (tiles + ks));
  double* tb = scratch.as<double>();
  double* kb = tb + 8 * tiles;
  otf_boxes<<<(unsigned)ceil_div(tiles, 128), 128, 0, st>>>(X, row0, rows, kp.d, OB_M, tiles, tb);
  RLD_LAUNCH_CHECK();
  otf_boxes<<<(unsigned)ceil_div(ks, 128), 128, 0, st>>>(X, 0, n, kp.d, OB_K, ks, kb);
  RLD_LAUNCH_CHECK();
  const int sK = kp.diag > 0.0 ? SCALE_TOP - ilogb(kp.diag) : 0;
  const double thresh = std::ldexp(1.0, -27 - sK);
  otf_skip_kernel<<<(unsigned)ceil_div(tiles * wpt, 256), 256, 0, st>>>(tb, kb, tiles, ks, wpt, kp.d, kp, thresh, row0,
                                                                        rows, bits);
  RLD_LAUNCH_CHECK();
}

int64_t otf_skip_words(int64_t rows, int64_t n) { return ceil_div(rows, OB_M) * ceil_div(ceil_div(n, OB_K), 32); }

__global__ void popc_kernel(const uint32_t* __restrict__ w, int64_t n, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(w[i]);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// fraction of the (tile, k-step) pairs the map skips
double otf_skip_fraction(const uint32_t* bits, int64_t rows, int64_t n, DevBuf& scratch, cudaStream_t st) {
  const int64_t words = otf_skip_words(rows, n);
  if (words <= 0) return 0.0;
  scratch.reserve(sizeof(unsigned long long));
  RLD_CUDA(cudaMemsetAsync(scratch.ptr, 0, sizeof(unsigned long long), st));
  popc_kernel<<<(unsigned)std::min<int64_t>(ceil_div(words, 256), 1024), 256, 0, st>>>(
      bits, words, scratch.as<unsigned long long>());
  RLD_LAUNCH_CHECK();
  unsigned long long c = 0;
  RLD_CUDA(cudaMemcpyAsync(&c, scratch.ptr, sizeof c, cudaMemcpyDeviceToHost, st));
  RLD_CUDA(cudaStreamSynchronize(st));
  return (double)c / (double)(ceil_div(rows, OB_M) * ceil_div(n, OB_K));
}

// The fp16 kernel is the default on-the-fly float32 product; RLD_OTF_KIND=tf32 selects the
// 3xTF32 kernel of kv_tc.cu (read per call, for A/B measurements).
bool kv_otf_f16_enabled() {
  const char* e = getenv("RLD_OTF_KIND");
  return !(e && e[0] == 't');
}

int64_t otf_points_floats(int64_t n) { return 8 * ceil_div(n, OB_K) * OB_K; }

void kv_product_otf16(const KvOperand& op, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                      KvWorkspace& ws, cudaStream_t st) {
  const int64_t n = op.n, rows = op.rows;
  const bool stored = op.K != nullptr;   // tiled fp32 K with per-row scales, else points
  if (stored && (!op.tiled || !op.rowscale)) fail(RLD_ERR_INVALID_ARGUMENT, "kv_otf: stored K must be tiled and scaled");
  if (n >= (int64_t)1 << 31) fail(RLD_ERR_NOT_SUPPORTED, "kv_otf: n >= 2^31");
  const int ks = (int)ceil_div(n, OB_K);
  const int npass = (int)ceil_div(m, 128);
  int width = (int)(ceil_div(ceil_div(m, npass), 32) * 32);
  if (width == 96 && !stored) width = 128;   // on the fly: generation-bound, passes of 96 gain nothing
  const int64_t mp = (int64_t)npass * width;
  // per-vector scales, then the fp16 head / tail operand
  ws.otf_vmax.reserve(sizeof(unsigned long long) * mp);
  unsigned long long* vmax = ws.otf_vmax.as<unsigned long long>();
  RLD_CUDA(cudaMemsetAsync(vmax, 0, sizeof(unsigned long long) * mp, st));
  {
    const dim3 g((unsigned)std::min<int64_t>(64, ceil_div(n, 256 * 8)), (unsigned)m);
    kv_otf_vmax<<<g, 256, 0, st>>>(V, ldv, n, vmax);
    RLD_LAUNCH_CHECK();
  }
  ws.bhi.reserve(sizeof(__half) * mp * ks * OB_K);
  ws.blo.reserve(sizeof(__half) * mp * ks * OB_K);
  {
    const dim3 g((unsigned)ceil_div((int64_t)ks * OB_K, 256), (unsigned)mp);
    kv_otf_split<<<g, 256, 0, st>>>(V, ldv, m, n, mp, ks, vmax, ws.bhi.as<__half>(), ws.blo.as<__half>());
    RLD_LAUNCH_CHECK();
  }
  const int G = sm_count();
  const int tiles = (int)ceil_div(rows, OB_M);
  const int64_t total = (int64_t)tiles * ks;
  const int64_t Gl = std::min<int64_t>(std::max(1, G / npass), total);
  Sched sc{};
  sc.ks = ks;
  sc.G = (int)Gl;
  sc.R = (int)(tiles / Gl);
  sc.tail_total = (int64_t)(tiles - sc.R * Gl) * ks;
  int segs = 1;
  for (int t = sc.R * (int)Gl; t < tiles; ++t) {
    const int64_t x0 = (int64_t)(t - sc.R * Gl) * ks;
    segs = (int)std::max<int64_t>(segs, cta_of_step(x0 + ks - 1, sc.tail_total, Gl) - cta_of_step(x0, sc.tail_total, Gl) + 1);
  }
  OtfParams p{};
  p.sched = sc;
  p.mp = (int)mp;
  p.ks = ks;
  p.tiles = tiles;
  p.npass = npass;
  p.segs = segs;
  p.wait_mode = getenv("RLD_TC_WAIT") ? atoi(getenv("RLD_TC_WAIT")) : 1;
  p.wait_ns = 256;
  p.pts = op.pts4;
  p.rowscale = op.rowscale;
  p.ks32 = (int)ceil_div(n, 32);
  p.skip = stored ? nullptr : op.otf_skip;
  p.skip_wpt = (int)ceil_div(ks, 32);
  // Morton order puts a row's near field (most of |Y_i|) into a few consecutive k-steps, so a TMEM
  // group would carry nearly the whole sum through its truncating (round-toward-zero) adds: flush
  // every k-step there (config 3 on the fly, log det P vs the float64 oracle: groups of 4: 2.6e-5,
  // of 1: see DESIGN.md §3.4)
  static const int grp_sorted = getenv("RLD_OTF_GROUP") ? atoi(getenv("RLD_OTF_GROUP")) : 1;
  if (p.skip) p.sched.group = std::max(1, grp_sorted);
  p.n = n;
  p.row0 = op.row0;
  p.rows = rows;
  p.family = op.kp.family;
  const int sK = (!stored && op.kp.diag > 0.0) ? SCALE_TOP - ilogb(op.kp.diag) : 0;
  p.diag = (float)std::ldexp(op.kp.diag, sK);
  p.la2 = (float)(std::log2(op.kp.a2) + sK);
  {
    static const int sync_k = [] {
      int v = getenv("RLD_TC_SYNC_K") ? atoi(getenv("RLD_TC_SYNC_K")) : 1024;
      int pw = 0;
      while (v > 1 && (1 << (pw + 1)) <= v) ++pw;
      return v > 0 ? (1 << pw) : 0;
    }();
    // (none with a skip map: the kept steps differ between CTAs, so they share no epochs)
    p.sync_k = (sc.R > 1 || (sc.R == 1 && sc.tail_total > 0)) && g_live_handles.load() <= 1 && !p.skip ? sync_k : 0;
    // stored K in several passes: every pass streams all of K; keep the passes together (64 k-steps
    // = 2 MB of K per CTA per epoch, ~60 MB across the wave: inside L2)
    static const int sync_multi = getenv("RLD_OTF_SYNC_MULTI") ? atoi(getenv("RLD_OTF_SYNC_MULTI")) : 64;
    p.sync_all = (stored && npass > 1 && p.sync_k > 0 && sync_multi > 0) ? 1 : 0;
    if (p.sync_all) p.sync_k = sync_multi;
    ws.tc_sync.reserve(sizeof(unsigned int) * npass);
    p.sync = ws.tc_sync.as<unsigned int>();
    if (p.sync_k > 0) RLD_CUDA(cudaMemsetAsync(p.sync, 0, sizeof(unsigned int) * npass, st));
  }
  ws.tc_partial.reserve(sizeof(float) * (size_t)npass * tiles * segs * width * OB_M);
  p.partial = ws.tc_partial.as<float>();
  // points: [ceil(n/64) * 2 * 8][32] fp32, one 2 KB box {32, 16} per k-step
  // points: [ceil(n/64) * 2 * 8][32] fp32, one 2 KB box {32, 16} per k-step; stored K: the tiled
  // layout as [tiles * ks32 * 128][32] fp32, one 32 KB box {32, 256} (two tiles) per k-step
  const CUtensorMap mP = stored ? make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, op.K, 32,
                                              (int64_t)tiles * p.ks32 * OB_M, 128, 32, 256, CU_TENSOR_MAP_SWIZZLE_128B)
                                : make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, op.pts4, 32, (int64_t)ks * 16, 128, 32, 16,
                                              CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap mBh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, ws.bhi.ptr, OB_K, mp * ks, OB_K * 2, OB_K,
                                      width, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap mBl = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, ws.blo.ptr, OB_K, mp * ks, OB_K * 2, OB_K,
                                      width, CU_TENSOR_MAP_SWIZZLE_128B);
  const int64_t grid = Gl * npass;
  const bool prof_on = getenv("RLD_OTF_PROFILE") != nullptr;
  static DevBuf prof_buf;
  if (prof_on) {
    prof_buf.reserve(sizeof(unsigned long long) * 16 * (size_t)grid);
    RLD_CUDA(cudaMemsetAsync(prof_buf.ptr, 0, sizeof(unsigned long long) * 16 * (size_t)grid, st));
    p.prof = prof_buf.as<unsigned long long>();
  }
  const int d = op.kp.d;
  if (stored) {
    launch_otf_nt<0, 0>(width, mP, mBh, mBl, p, grid, st);
  } else if (op.kp.family == RLD_RBF) {
    if (d <= 2) launch_otf_nt<2, RLD_RBF>(width, mP, mBh, mBl, p, grid, st);
    else if (d == 3) launch_otf_nt<3, RLD_RBF>(width, mP, mBh, mBl, p, grid, st);
    else launch_otf_nt<4, RLD_RBF>(width, mP, mBh, mBl, p, grid, st);
  } else {
    if (d <= 2) launch_otf_nt<2, RLD_MATERN52>(width, mP, mBh, mBl, p, grid, st);
    else if (d == 3) launch_otf_nt<3, RLD_MATERN52>(width, mP, mBh, mBl, p, grid, st);
    else launch_otf_nt<4, RLD_MATERN52>(width, mP, mBh, mBl, p, grid, st);
  }
  if (prof_on) {
    std::vector<unsigned long long> h(16 * (size_t)grid);
    RLD_CUDA(cudaMemcpyAsync(h.data(), prof_buf.ptr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    double a[16] = {0};
    double tmax = 0.0, tmin = 1e300;
    for (int64_t c = 0; c < grid; ++c) {
      for (int k = 0; k < 16; ++k) a[k] += (double)h[c * 16 + k];
      tmax = std::max(tmax, (double)h[c * 16 + 13]);
      tmin = std::min(tmin, (double)h[c * 16 + 13]);
    }
    fprintf(stderr, "[kv_otf prof] CTA cycles: min %.3g avg %.3g max %.3g\n", tmin, a[13] / grid, tmax);
    const double ms = a[4] > 0 ? a[4] : 1, cs = a[7] > 0 ? a[7] : 1, ds = a[10] > 0 ? a[10] : 1;
    const double steps = (double)total * npass / grid;   // k-steps per CTA
    fprintf(stderr,
            "[kv_otf prof] m=%ld n=%ld nt=%d: kernel %.0f cycles/k-step | mma(w1) per own step: accempty %.0f afull %.0f "
            "bfull %.0f baton %.0f | conv(w4) per own step: kfull %.0f bempty %.0f post %.0f | drain wait per group %.0f "
            "| B producer bempty %.0f epoch %.0f per k-step\n",
            (long)m, (long)n, width, a[13] / grid / steps, a[0] / ms, a[1] / ms, a[2] / ms, a[3] / ms, a[5] / cs,
            a[6] / cs, a[8] / cs, a[9] / ds, a[11] / grid / steps, a[12] / grid / steps);
  }
  const dim3 rgrid((unsigned)tiles, (unsigned)ceil_div(m, RED_COLS));
  kv_otf_reduce<<<rgrid, 256, 0, st>>>(p.partial, sc, tiles, segs, width, m, rows, sK, stored ? op.rowscale : nullptr,
                                       vmax, Y, ldy);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
