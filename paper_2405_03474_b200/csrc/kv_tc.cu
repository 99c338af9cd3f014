// K x block products on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Y[c, i] = sum_j K[i, j] V[c, j] for a stored float32 K (the HBM-streaming
// path of BASELINE configs 2-3) or for K tiles generated on the fly from the
// points (configs 4-5); reference call sites src/estimators.py:72 and
// src/precond.py:186, 189.
//
// One persistent CTA per SM, 20 warps:
//   warp 0       TMA producer: per k-step, the K tile (128 rows x 32 fp32,
//                128B-swizzled) or the 32 column points (on the fly), plus the B
//                tiles (NT vectors x 32 fp32: tf32-hi, and lo for 3xTF32, stored in
//                k-step blocks so each box is contiguous) into an S-stage ring.
//   warps 1, 3   MMA issuers, alternate k-steps, handing a named-barrier baton so
//                the tensor core sees one fixed instruction order while each warp's
//                mbarrier wait and commit overlap the other's MMAs.  3xTF32 per
//                8-wide k chunk:
//                  NT == 32: D[2NT] += Ahi [Bhi; Blo] + Alo [Bhi; Blo] (two N = 64
//                            instructions: small N costs the same as N = 64);
//                  NT >= 64: D[NT] += Ahi Bhi + Ahi Blo + Alo Bhi.
//                1xTF32 (optional sketch mode): D[NT] += A Bhi.
//   warp 2       TMEM allocation owner.
//   4 CP warps   converters (CP per TMEM lane quarter, alternate k-steps): thread = one
//                K row; it reads its 32 values from the swizzled tile or generates
//                them from the points (FFMA2 + MUFU sqrt/ex2), splits them into tf32
//                hi + lo (lo exact in fp32) and tcgen05.st's them into a TMEM
//                A-operand buffer, so the tensor core never re-reads A from SMEM.
//   4 DP warps   accumulator drains (CP + DP = 4 per quarter).
//
// Accuracy: the tensor core rounds its fp32 accumulator toward zero, so a long
// accumulation drifts (measured -2e-4 relative at n = 16384, -9e-4 at 65536).
// The MMAs therefore accumulate only GROUP k-steps into one of two TMEM
// accumulators; the drain warps add each finished group into fp32 registers
// with round-to-nearest while the tensor core fills the other accumulator.
//
// Work split (Sched): full rounds of G row tiles, all CTAs sweeping k in step
// (kept within an epoch of each other by a producer barrier) so L2 serves the B
// operand to every CTA; the tail tiles are cut into equal stream-K ranges whose
// per-CTA partial sums kv_tc_reduce adds in fixed order, in float64
// (deterministic).  Column passes (more vectors than one TMEM accumulator holds)
// run as concurrent CTA groups of the same launch so K streams from HBM once.
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cstdio>

#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"
#include "kv_sched.cuh"

namespace rld {

namespace {

constexpr int TC_BM = 128;          // K rows per tile (UMMA M)
constexpr int TC_BK = 32;           // fp32 k-elements per step (one 128-byte swizzle row)
constexpr int TC_THREADS = 640;   // 20 warps: TMA, 2 MMA, TMEM owner, 4 CP converters, 4 DP drains (CP + DP = 4)
constexpr int NABUF_MAX = 8;        // pipeline stages = TMEM A-operand buffers: as many as the 512 columns leave (<= 8)
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;  // 16 KB

// CTA b works on column pass b % npass over stream-K range b / npass.
struct TcParams {
  Sched sched;      // work schedule (per column pass)
  int mp;           // B rows per k-step block (vectors padded to npass x NT)
  int a_tiled;      // stored K in 16 KB tiles (box row (tile ks + kstep) 128) instead of row-major
  int bcol_step, brow_step;   // TMA coordinates of B per k-step: blocked (0, mp) or row-major (32, 0)
  unsigned int* sync;   // per-pass arrival counters of the phase-1 epoch barrier (zeroed per launch)
  int sync_k;           // k-steps per epoch (0: no barrier)
  int sync_all;         // 1: the epoch barrier spans all passes (one counter)
  int arrive_sem;       // CTA pairs: semantics of the remote mbarrier arrives (RLD_TC_ARRIVE)
  int ks;           // k-steps per tile
  int tiles;
  int npass;        // column passes in this launch
  int segs;         // partial slots per tile
  int sa, sb;       // A-source ring and B ring (= TMEM A buffers) depths
  uint32_t tmem_cols;
  float* partial;   // [npass][tiles][segs][NT][128]
  int wait_mode;    // producer / drain wait strategy (RLD_TC_WAIT, see ptx::mbar_wait_idle)
  uint32_t wait_ns;  // back-off of wait_mode 1 (RLD_TC_WAIT_NS)
  unsigned long long* prof;   // RLD_TC_PROFILE: per-CTA cycle counters [grid][16], else null
  int debug;        // profiling bitmask (RLD_TC_DEBUG): 1 skip A stores, 2 skip MMAs, 4 skip K-tile loads,
                    // 8 skip tile generation math, 16 converters only arrive, 32 drains skip TMEM loads
  // on-the-fly kernel tiles (src/kernels.py:40-46, 72)
  const float* pts;  // [ceil(n/32)][8][32] float32 k-step blocks: scaled x,y,z,w rows, rows 4-7 zero
  int64_t n, row0, rows;
  int family;
  float diag;                  // a^2 + jitter
  float la2;                   // log2(amplitude^2), folded into the exponent
};

// Two K entries from packed scaled squared distances (src/kernels.py:40-46), float32:
// RBF a^2 2^(-r2') with r2' = r^2 log2(e) / (2 l^2); Matern-5/2 a^2 (1 + u + u^2/3) e^-u
// with u = sqrt(r2') = sqrt(5) r / l.  a^2 is folded into the exponent (la2 = log2 a^2).
template <int FAM>
__device__ __forceinline__ uint64_t kernel_pair(const TcParams& p, uint64_t r2) {
  if (FAM == RLD_RBF) {
    const uint64_t t = fma2(r2, pk(-1.f, -1.f), pk(p.la2, p.la2));
    return pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t)));
  }
  const uint64_t u = pk(fast_sqrt(pk_lo(r2)), fast_sqrt(pk_hi(r2)));
  const uint64_t poly = fma2(u, fma2(u, pk(1.0f / 3.0f, 1.0f / 3.0f), pk(1.f, 1.f)), pk(1.f, 1.f));
  const uint64_t t = fma2(u, pk(-1.4426950408889634f, -1.4426950408889634f), pk(p.la2, p.la2));
  return mul2(poly, pk(fast_exp2(pk_lo(t)), fast_exp2(pk_hi(t))));
}

// 16 on-the-fly K entries of one converter thread: its row x 16 column points of
// the stage (columns [e0, e0 + 16) of the k-step), split into tf32 hi + lo.
// Coordinates arrive pre-scaled in float32 (x sqrt(5)/l for Matern-5/2, x
// sqrt(log2(e)/(2 l^2)) for RBF), so r2 is the kernel's argument directly.  FIX:
// the half step holds a diagonal entry (a^2 + jitter, src/kernels.py:72) or
// padding columns >= n (zero) -- warp-uniform, so the common path has no selects.
template <int DIM, int FAM, bool FIX>
__device__ __forceinline__ void gen16(const TcParams& p, uint32_t pp, const uint64_t (&xr2)[DIM], int j0,
                                      int grow, int n32, uint32_t (&hi)[16], uint32_t (&lo)[16]) {
  const uint64_t neg1 = pk(-1.f, -1.f);
#pragma unroll
  for (int e = 0; e < 16; e += 4) {
    uint64_t r2a = 0, r2b = 0;   // entries (e, e+1) and (e+2, e+3)
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const float4 c = ptx::lds128(pp + 4u * (k * 32 + e));
      const uint64_t da = fma2(pk(c.x, c.y), neg1, xr2[k]);
      const uint64_t db = fma2(pk(c.z, c.w), neg1, xr2[k]);
      r2a = fma2(da, da, r2a);
      r2b = fma2(db, db, r2b);
    }
    uint64_t kv[2] = {kernel_pair<FAM>(p, r2a), kernel_pair<FAM>(p, r2b)};
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
      const uint32_t u0 = (uint32_t)kv[h], u1 = (uint32_t)(kv[h] >> 32);
      const int ee = e + 2 * h;
      const uint32_t h0 = u0 & 0xFFFFE000u, h1 = u1 & 0xFFFFE000u;
      hi[ee] = h0;
      hi[ee + 1] = h1;
      const uint64_t l2 = fma2((uint64_t)h0 | ((uint64_t)h1 << 32), neg1, kv[h]);   // v - hi (exact)
      lo[ee] = (uint32_t)l2;
      lo[ee + 1] = (uint32_t)(l2 >> 32);
    }
  }
}

// 16 stored K entries of one converter thread (its row, columns [16 half, +16) of
// the 128-byte-swizzled tile), split into tf32 hi + lo (3xTF32) or passed (1xTF32).
template <int MODE>
__device__ __forceinline__ void load16(const uint8_t* rowp, int row, int half, uint32_t (&hi)[16],
                                       uint32_t (&lo)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int cc = 4 * half + c;   // 16-byte chunk of the 128-byte row
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

// On-the-fly K: the stage carries the 32 column points of the k-step (TMA box of
// the coordinate-major point array [8][ldp]: rows x,y,z,w of the pre-scaled
// float32 coordinates, rows 4-7 zero padding so the B tiles stay 1024-byte
// aligned) instead of a K tile; the converter warps generate the tile with packed
// FP32x2 arithmetic (FFMA2/FMUL2) and MUFU sqrt/ex2.  Rounding the coordinates to
// float32 moved reduced config-4/5 estimates by 4e-10 / 1e-8 relative in float64
// (scripts/otf_points_fp32.py), far inside the 1e-4 fp32 budget.
constexpr uint32_t PTS_BYTES = 1024;

template <int MODE, int NT, bool OTF = false, bool CG2 = false>
struct TcShape {
  static constexpr bool STACK = MODE == 3 && NT == 32;  // [Bhi; Blo] as one N = 2 NT operand
  static constexpr int DW = STACK ? 2 * NT : NT;       // accumulator columns
  // CTA pairs (CG2, cta_group::2): each CTA holds half of the B operand's N rows -- NT / 2 rows of
  // Bhi and of Blo, or, stacked, all NT rows of Bhi (leader) / Blo (peer)
  static constexpr int BROWS = (CG2 && !STACK) ? NT / 2 : NT;   // B rows per operand in this CTA
  static constexpr int BOPS = (CG2 && STACK) ? 1 : (MODE == 3 ? 2 : 1);   // B operands in this CTA's stage
  static constexpr uint32_t B_BYTES = (uint32_t)BROWS * 128;
  static constexpr int MM = CG2 ? 256 : 128;                    // MMA M (over the pair)
  static constexpr uint32_t A_REGION = OTF ? PTS_BYTES : A_BYTES;
  static constexpr uint32_t STAGE = A_REGION + B_BYTES * BOPS;
  static constexpr uint32_t ASTRIDE = MODE == 3 ? 64 : 32;  // TMEM columns per A buffer (hi | lo)
  // TMEM accumulator buffers: two, or (CTA pairs) three / four -- the pair's drain handshake
  // (multicast commit, remote arrive) is longer than one group of MMAs
  static constexpr int NACC = (CG2 && DW <= 64) ? 3 : 2;
  static constexpr uint32_t A_COL0 = NACC * DW;
  // warps per TMEM lane quarter: drains (DP; each holds NT / DP fp32 running sums in
  // registers) and converters (CP = 4 - DP), within the 20-warp CTA.  A third
  // converter warp per quarter measured +6 % at NT = 64 (config 4 on the fly) and
  // -10 % at NT = 32, where the extra polling warps cost more than they hide
  static constexpr int DP = NT == 64 ? 1 : 2;
  static constexpr int CP = 4 - DP;
  static constexpr int NABUF =
      (512 - NACC * DW) / (int)ASTRIDE < NABUF_MAX ? (512 - NACC * DW) / (int)ASTRIDE : NABUF_MAX;
  static constexpr int TMEM_NEED = NACC * DW + NABUF * (int)ASTRIDE;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  // a converter posts step j's afull only after starting step j + CP, whose TMEM buffer must not
  // be the one step j's MMAs still hold: more buffers than converter warps per quarter
  static_assert(NABUF > CP, "TMEM A buffers");
  static_assert(NT % 16 == 0 && (NT / DP) % 8 == 0 && NT <= 144, "NT");
  static_assert(!CG2 || (!OTF && (STACK || (NT / 2) % 16 == 0)), "pair variant: stored K, half of N a multiple of 16");
};

template <int MODE, int NT, bool OTF, int DIM, int FAM, bool CG2 = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
kv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
             const __grid_constant__ CUtensorMap tmBlo, const TcParams p) {
  using Sh = TcShape<MODE, NT, OTF, CG2>;
  constexpr int DW = Sh::DW;
  constexpr uint32_t B_BYTES = Sh::B_BYTES, ASTRIDE = Sh::ASTRIDE, A_COL0 = Sh::A_COL0;
  constexpr uint32_t AR = Sh::A_REGION;   // K tile (stored) or column points (on the fly)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw so the compiler keeps the shared
  // address space (plain C++ loads compile to LDS and are ordered by the mbarrier asm)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  // Two rings.  Step j reads its A source (K tile, or the 32 column points on the
  // fly) from A-ring stage j % SA and its B tiles from B-ring stage j % SB; TMEM A
  // buffer j % SB goes with the B stage (NA == SB):
  //   kfull/kempty[SA]   K tile landed / read by the 4 converter warps of the step --
  //                      released right after conversion, so the HBM stream of K can
  //                      run up to SA steps ahead of the tensor core;
  //   bfull/bempty[SB]   B tiles landed (producer warp 2) / MMAs of the step done
  //                      (tcgen05.commit); bempty also frees TMEM A buffer j % SB;
  //   afull[SB]          A tile converted into TMEM (4 converter warps -> MMA).
  // One wait on afull + one on bfull and one commit per step keep the serial
  // MMA-issue loops short.
  const int SA = p.sa, SB = p.sb;
  constexpr uint32_t BST = B_BYTES * Sh::BOPS;
  uint8_t* const bring = smem + (size_t)SA * AR;
  uint64_t* kfull = reinterpret_cast<uint64_t*>(bring + (size_t)SB * BST);
  uint64_t* kempty = kfull + SA;
  uint64_t* bfull = kempty + SA;
  uint64_t* bempty = bfull + SB;
  uint64_t* afull = bempty + SB;
  constexpr int NACC = Sh::NACC;
  uint64_t* accfull = afull + SB;       // [NACC]
  uint64_t* accempty = accfull + NACC;  // [NACC]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accempty + NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CG2: blockIdx.x = 2 (pair * npass + pass) + rank; the schedule walks pair tiles of 256 rows,
  // rank r takes row tile 2 t + r
  const int rank = CG2 ? (int)(blockIdx.x & 1) : 0;
  const int64_t bid = CG2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int pass = (int)(bid % p.npass);
  const int64_t cta = bid / p.npass;
  auto row_tile = [&](int t) { return CG2 ? 2 * t + rank : t; };
  const int b_row0 = pass * NT;
  float* const partial = p.partial + (size_t)pass * p.tiles * p.segs * NT * TC_BM;
  unsigned long long* const prof = p.prof ? p.prof + blockIdx.x * 16 : nullptr;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmBhi);
    if (MODE == 3) ptx::tma_prefetch_desc(&tmBlo);
    for (int i = 0; i < SA; ++i) {
      ptx::mbar_init(&kfull[i], 1);
      ptx::mbar_init(&kempty[i], 4);   // one arrive per lane-quarter converter warp
    }
    for (int i = 0; i < SB; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1);
      ptx::mbar_init(&afull[i], CG2 ? 8 : 4);   // CG2: the leader's barrier counts both CTAs' converters
    }
    for (int i = 0; i < NACC; ++i) {
      ptx::mbar_init(&accfull[i], 2);   // one commit per MMA-issuing warp
      ptx::mbar_init(&accempty[i], (CG2 ? 8 : 4) * Sh::DP);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) {
    if constexpr (CG2) ptx::tmem_alloc_pair(tmem_holder, Sh::TMEM_COLS);
    else ptx::tmem_alloc(tmem_holder, Sh::TMEM_COLS);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG2) ptx::cluster_sync();   // both CTAs' barriers initialised before any remote arrive
  ptx::tc_fence_after();
  // barriers of the pair leader, as shared::cluster addresses (remote arrives / 2-SM TMA)
  const uint32_t afull_l = CG2 ? ptx::mapa(afull, 0) : 0, accempty_l = CG2 ? ptx::mapa(accempty, 0) : 0;
  const uint32_t bfull_l = CG2 ? ptx::mapa(bfull, 0) : 0;
  const uint32_t tmem = *tmem_holder;

  if (StepIter<false, false>(p.sched, cta, 1).valid()) {
    if (warp == 0) {
      // ---------------- A-source producer: K tiles from HBM (or the column points)
      unsigned long long t_wait = 0;
      const unsigned long long t_start = prof ? clock64() : 0;
      for (StepIter<false, false> it(p.sched, cta, SA); it.valid(); it.next()) {
        const int s = it.s;
        const unsigned long long t0 = prof ? clock64() : 0;
        ptx::mbar_wait_idle(&kempty[s], it.ph ^ 1, p.wait_mode, p.wait_ns);
        if (prof) t_wait += clock64() - t0;
        if (ptx::elect_one()) {
          uint8_t* st = smem + (size_t)s * AR;
          if (OTF) {
            ptx::mbar_arrive_expect_tx(&kfull[s], AR);
            ptx::tma_load_2d(st, &tmA, &kfull[s], 0, it.kstep * 8);   // 32 column points, 8 coordinate rows
          } else if (p.debug & 4) {
            ptx::mbar_arrive(&kfull[s]);
          } else {
            ptx::mbar_arrive_expect_tx(&kfull[s], AR);
            if (p.a_tiled)
              ptx::tma_load_2d(st, &tmA, &kfull[s], 0, (row_tile(it.tile) * p.ks + it.kstep) * TC_BM);
            else
              ptx::tma_load_2d(st, &tmA, &kfull[s], it.kstep * TC_BK, row_tile(it.tile) * TC_BM);
          }
        }
        __syncwarp();
      }
      if (prof && lane == 0) {
        prof[0] = t_wait;
        prof[1] = clock64() - t_start;
      }
    } else if (warp == 2) {
      // ---------------- B producer (after the TMEM allocation)
      int64_t epoch = 0;
      for (StepIter<false, false> it(p.sched, cta, SB); it.valid(); it.next()) {
        const int s = it.s;
        // phase-1 epoch barrier: the CTAs' B producers meet every sync_k k-steps, so all
        // CTAs stream the same window of B and L2 serves it (their drift otherwise
        // accumulates tile after tile until B comes from HBM once per tile)
        if (p.sync_k > 0 && !it.in_tail() && it.v > 0 && (it.kstep & (p.sync_k - 1)) == 0) {
          ++epoch;
          if (lane == 0) {
            // one counter for all passes (p.sync_all): CTA c of every pass streams the same
            // row tiles of K, so aligned passes read each K tile from HBM once, not npass times
            unsigned int* ctr = p.sync + (p.sync_all ? 0 : pass);
            atomicAdd(ctr, 1u);
            const unsigned int target =
                (unsigned int)(epoch * p.sched.G * (p.sync_all ? p.npass : 1) * (CG2 ? 2 : 1));
            while (*(volatile unsigned int*)ctr < target) __nanosleep(100);
          }
          __syncwarp();
        }
        ptx::mbar_wait_idle(&bempty[s], it.ph ^ 1, p.wait_mode, p.wait_ns);
        if (ptx::elect_one()) {
          uint8_t* st = bring + (size_t)s * BST;
          const int bcol = it.kstep * p.bcol_step, brow = it.kstep * p.brow_step + b_row0;
          if constexpr (CG2) {
            // each CTA loads its half of N; both count on the leader's barrier
            if (rank == 0) ptx::mbar_arrive_expect_tx(&bfull[s], 2 * BST);
            const uint32_t bar = bfull_l + 8u * (uint32_t)s;
            if (Sh::STACK) {
              ptx::tma_load_2d_pair(st, rank ? &tmBlo : &tmBhi, bar, bcol, brow);
            } else {
              ptx::tma_load_2d_pair(st, &tmBhi, bar, bcol, brow + rank * Sh::BROWS);
              if (MODE == 3) ptx::tma_load_2d_pair(st + B_BYTES, &tmBlo, bar, bcol, brow + rank * Sh::BROWS);
            }
          } else {
            ptx::mbar_arrive_expect_tx(&bfull[s], BST);
            // B in k-step blocks [ks][mp][32]: one contiguous NT x 128-byte box per step
            ptx::tma_load_2d(st, &tmBhi, &bfull[s], bcol, brow);
            if (MODE == 3) ptx::tma_load_2d(st + B_BYTES, &tmBlo, &bfull[s], bcol, brow);
          }
        }
        __syncwarp();
      }
    } else if ((warp == 1 || warp == 3) && rank == 0) {
      // ---------------- MMA issuers: warps 1 and 3 take alternate steps (whole warp walks
      // the pipeline so every descriptor is warp-uniform; one elected lane issues).  A
      // named-barrier baton hands the issue slot from step j's warp to step j+1's, so the
      // tensor core sees one deterministic instruction order, while each warp's
      // per-step mbarrier waits and commit overlap the other warp's MMAs.  Each warp
      // commits accfull at every group end (count 2): together the two commits cover
      // all MMAs of the group.
      const int mpar = warp == 3;
      constexpr uint32_t idesc = ptx::idesc_tf32(Sh::MM, DW);
      const uint64_t desc0 = ptx::smem_desc_sw128(ptx::smem_u32(bring));
      constexpr uint64_t LO_OFF = (uint64_t)(B_BYTES >> 4);   // Blo rows, in descriptor units
      int64_t gi = -1;  // group index
      unsigned long long t_acc = 0, t_afull = 0, t_iss = 0, nsteps = 0;
      const unsigned long long t_start = prof ? clock64() : 0;
      for (StepIter<true, false> it(p.sched, cta, SB); it.valid(); it.next()) {
        const bool gstart = it.group_start(), gend = it.group_end();
        if (gstart) ++gi;
        if ((it.v & 1) == mpar) {
          const int s = it.s;
          const unsigned long long t0 = prof ? clock64() : 0;
          if (gstart && gi >= NACC) ptx::mbar_wait(&accempty[gi % NACC], (uint32_t)((gi / NACC - 1) & 1));
          ptx::mbar_wait(&afull[s], it.ph);
          ptx::mbar_wait(&bfull[s], it.ph);
          const unsigned long long t1 = prof ? clock64() : 0;
          if (it.v > 0) ptx::named_bar_sync(mpar ? 1 : 2, 64);   // baton from step j - 1
          const unsigned long long t2 = prof ? clock64() : 0;
          ptx::tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(gi % NACC) * DW;
          const uint32_t a0 = tmem + A_COL0 + ASTRIDE * s;
          const uint64_t bdesc = desc0 + (uint64_t)((s * BST) >> 4);
          const bool leader = ptx::elect_one();
          if (leader && !(p.debug & 2)) {
#pragma unroll
            for (int kk = 0; kk < TC_BK / 8; ++kk) {
              const uint64_t bd = bdesc + 2 * kk;  // +32 bytes along k
              const uint32_t acc = (gstart && kk == 0) ? 0u : 1u;
              auto mma = [&](uint32_t dd, uint32_t aa, uint64_t bb, uint32_t ac) {
                if constexpr (CG2) ptx::mma_tf32_ts_pair(dd, aa, bb, idesc, ac);
                else ptx::mma_tf32_ts(dd, aa, bb, idesc, ac);
              };
              if (MODE == 1) {
                mma(d, a0 + 8 * kk, bd, acc);
              } else if (Sh::STACK) {
                mma(d, a0 + 8 * kk, bd, acc);        // D += Ahi [Bhi; Blo]
                mma(d, a0 + 32 + 8 * kk, bd, 1u);    // D += Alo [Bhi; Blo]
              } else {
                mma(d, a0 + 8 * kk, bd, acc);            // D += Ahi Bhi
                mma(d, a0 + 8 * kk, bd + LO_OFF, 1u);    // D += Ahi Blo
                mma(d, a0 + 32 + 8 * kk, bd, 1u);        // D += Alo Bhi
              }
            }
          }
          __syncwarp();
          if (it.v + 1 < it.vend) ptx::named_bar_arrive(mpar ? 2 : 1, 64);   // baton to step j + 1
          if (leader) {
            if constexpr (CG2) ptx::tc_commit_pair(&bempty[s]);
            else ptx::tc_commit(&bempty[s]);
          }
          if (prof) {
            t_acc += t1 - t0;
            t_afull += t2 - t1;
            t_iss += clock64() - t2;
            ++nsteps;
          }
        }
        if (gend) {
          if (ptx::elect_one()) {
            if constexpr (CG2) ptx::tc_commit_pair(&accfull[gi % NACC]);
            else ptx::tc_commit(&accfull[gi % NACC]);
          }
          __syncwarp();
        }
      }
      if (prof && lane == 0 && warp == 1) {
        prof[2] = t_acc; prof[4] = t_afull; prof[5] = t_iss; prof[6] = clock64() - t_start; prof[13] = 2 * nsteps;
      }
    } else if (warp >= 4 && warp < 4 + 4 * Sh::CP) {
      // ---------------- converters: warp 4 + q + 4 par owns TMEM lanes 32q..32q+31 (K rows)
      // and the steps j with j % CP == par (all 32 k-columns of each), so the warps of a
      // sub-partition work on different steps and one's generation overlaps another's
      // TMEM stores; each warp posts the afull arrive of a step only after generating
      // the first half of its next step, so tcgen05.wait::st rarely waits.
      const int q = (warp - 4) & 3, par = (warp - 4) >> 2;
      const int row = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      int cur_tile = -1;
      uint64_t xr2[DIM > 0 ? DIM : 1];   // this row's scaled point, packed twice (on the fly)
#pragma unroll
      for (int k = 0; k < (DIM > 0 ? DIM : 1); ++k) xr2[k] = 0;
      int grow = 0, wrow0 = 0;   // global row of this lane / of lane 0 (n < 2^31)
      const int n32 = (int)p.n;
      int pend = -1;             // A buffer whose TMEM stores are in flight
      auto arrive_afull = [&](int buf) {   // CG2: on the leader's barrier
        if constexpr (CG2) ptx::mbar_arrive_cluster(afull_l + 8u * (uint32_t)buf, p.arrive_sem);
        else ptx::mbar_arrive(&afull[buf]);
      };
      auto post = [&](int buf) {
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_afull(buf);
      };
      unsigned long long cv_full = 0;
      const unsigned long long cv_start = prof ? clock64() : 0;
      StepIter<false, true> it(p.sched, cta, SA, SB);
      for (int k = 0; k < par; ++k) it.next();
      for (; it.valid(); [&] { for (int k = 0; k < Sh::CP; ++k) it.next(); }()) {
        const int s = it.s, sb = it.sb;
        if constexpr (OTF) if (it.tile != cur_tile) {
          cur_tile = it.tile;
          const int lr = cur_tile * TC_BM + row;
          wrow0 = (int)p.row0 + cur_tile * TC_BM + q * 32;
          grow = wrow0 + lane;
          if (lr < p.rows) {
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
              const float x = p.pts[(((int64_t)(grow >> 5) * 8 + k) << 5) + (grow & 31)];
              xr2[k] = pk(x, x);
            }
          }
        }
        const unsigned long long c0 = prof ? clock64() : 0;
        ptx::mbar_wait(&kfull[s], it.ph);
        // TMEM A buffer sb is free once the MMAs of step j - SB completed
        if (it.v >= SB) ptx::mbar_wait(&bempty[sb], it.phb ^ 1);
        if (prof) cv_full += clock64() - c0;
        ptx::tc_fence_after();
        const uint32_t ta = tmem + lane_base + A_COL0 + ASTRIDE * sb;
        if (p.debug & 16) {   // profiling: no converter work at all
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&kempty[s]);
            arrive_afull(sb);
          }
          continue;
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hi[16], lo[16];
          if constexpr (OTF) {
            const uint32_t pp = ptx::smem_u32(smem + (size_t)s * AR) + 64u * half;   // [8][32] fp32
            const int j0 = it.kstep * TC_BK + 16 * half;
            // warp-uniform: a diagonal entry of these rows, or columns >= n?
            const bool fix = (j0 < wrow0 + 32 && j0 + 16 > wrow0) || (j0 + 16 > n32);
            if (p.debug & 8) {   // profiling: raw stage words, no generation math
#pragma unroll
              for (int c = 0; c < 16; c += 4) {
                const float4 v = ptx::lds128(pp + 4u * c);
                hi[c] = lo[c] = __float_as_uint(v.x); hi[c + 1] = lo[c + 1] = __float_as_uint(v.y);
                hi[c + 2] = lo[c + 2] = __float_as_uint(v.z); hi[c + 3] = lo[c + 3] = __float_as_uint(v.w);
              }
            } else if (!fix) {
              gen16<DIM, FAM, false>(p, pp, xr2, 0, 0, 0, hi, lo);
            } else {
              gen16<DIM, FAM, true>(p, pp, xr2, j0, grow, n32, hi, lo);
            }
          } else {
            load16<MODE>(smem + (size_t)s * AR + row * 128, row, half, hi, lo);
          }
          if (half == 1) {   // the stage is read: release it to the producer
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&kempty[s]);
          }
          if (half == 0 && pend >= 0) post(pend);
          if (!(p.debug & 1)) {
            ptx::tmem_st_32x32b_x16(ta + 16 * half, hi);
            if (MODE == 3) ptx::tmem_st_32x32b_x16(ta + 32 + 16 * half, lo);
          }
        }
        pend = sb;
      }
      if (pend >= 0) post(pend);
      if (prof && warp == 4 && lane == 0) {
        prof[7] = cv_full; prof[10] = clock64() - cv_start;
      }
    } else if (warp >= 4 + 4 * Sh::CP) {
      // ---------------- accumulator drain: warp 12 + q + 4h owns TMEM lanes 32q..32q+31 and
      // result columns [h NT/2, (h+1) NT/2); finished groups are added to fp32 registers
      // (round-to-nearest), a finished segment is stored to the partial buffer
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
      unsigned long long dr_wait = 0;
      const unsigned long long dr_start = prof ? clock64() : 0;
      SegIter si(p.sched, cta);
      int tile = 0, len = 0, seg = 0;
      while (si.next(tile, len, seg)) {
        for (int g0 = 0; g0 < len; g0 += GROUP) {
          ++gi;
          const int buf = (int)(gi % NACC);
          const unsigned long long d0 = prof ? clock64() : 0;
          ptx::mbar_wait_idle(&accfull[buf], (uint32_t)((gi / NACC) & 1), p.wait_mode, p.wait_ns);
          if (prof) dr_wait += clock64() - d0;
          ptx::tc_fence_after();
          if (!(p.debug & 32)) {
#pragma unroll
            for (int c0 = 0; c0 + 16 <= HALF; c0 += 16) {
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
            if constexpr (HALF % 16 == 8) {   // NT = 144: a last 8-column chunk (never stacked)
              constexpr int c0 = HALF - 8;
              uint32_t v[8];
              ptx::tmem_ld_32x32b_x8(tmem + lane_base + (uint32_t)(buf * DW + c_base + c0), v);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[c0 + e] += __uint_as_float(v[e]);
            }
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG2) ptx::mbar_arrive_cluster(accempty_l + 8u * (uint32_t)buf, p.arrive_sem);
            else ptx::mbar_arrive(&accempty[buf]);
          }
        }
        const int rt = row_tile(tile);
        float* P = partial + ((size_t)rt * p.segs + seg) * (size_t)NT * TC_BM;
#pragma unroll
        for (int c = 0; c < HALF; ++c) {
          if (rt < p.tiles) P[(size_t)(c_base + c) * TC_BM + row] = acc[c];
          acc[c] = 0.f;
        }
      }
      if (prof && dw == 0 && lane == 0) {
        prof[11] = dr_wait; prof[12] = clock64() - dr_start;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG2) {
    ptx::cluster_sync();   // the peer's last remote arrives have landed; no MMA reads TMEM any more
    if (warp == 2) ptx::tmem_dealloc_pair(tmem, Sh::TMEM_COLS);
  } else {
    if (warp == 2) ptx::tmem_dealloc(tmem, Sh::TMEM_COLS);
  }
}

// Y[c * ldy + i] = sum over the tile's segments of the partials (float64 accumulation, fixed order).
// One block per (row tile, 8 columns): the segment count is computed once per block.
constexpr int RED_COLS = 8;
__global__ void __launch_bounds__(256)
kv_tc_reduce(const float* __restrict__ P, Sched sc, int tiles, int segs, int nt, int64_t m, int64_t rows,
             double* __restrict__ Y, int64_t ldy, int pair) {
  const int tile = blockIdx.x;
  const int r = threadIdx.x & 127;
  const int64_t i = (int64_t)tile * TC_BM + r;
  const int unit = pair ? tile >> 1 : tile;   // schedule unit (a pair tile for CTA pairs)
  const int full = sc.R * sc.G;
  int nseg = 1;
  if (unit >= full) {
    const int64_t x0 = (int64_t)(unit - full) * sc.ks;
    nseg = (int)(cta_of_step(x0 + sc.ks - 1, sc.tail_total, sc.G) - cta_of_step(x0, sc.tail_total, sc.G) + 1);
  }
  if (i >= rows) return;
  const int c0 = blockIdx.y * RED_COLS;
#pragma unroll
  for (int q = threadIdx.x >> 7; q < RED_COLS; q += 2) {
    const int c = c0 + q;
    if (c >= m) break;
    const int pass = c / nt, cc = c - pass * nt;
    const float* Pp = P + (size_t)pass * tiles * segs * nt * TC_BM + ((size_t)tile * segs * nt + cc) * TC_BM + r;
    double s = 0.0;
    for (int k = 0; k < nseg; ++k) s += (double)Pp[(size_t)k * nt * TC_BM];
    Y[(int64_t)c * ldy + i] = s;
  }
}

// B operand from float64 V (m rows of length n) in k-step blocks Bt[ks][mp][32]
// (contiguous 128-byte rows per vector and k-step, zero padded for c >= m, j >= n):
// hi = tf32(v) (3xTF32) or fp32(v) (1xTF32), lo = fp32(v - hi).  The blocked layout
// makes every pipeline step's TMA box one contiguous NT x 128-byte range, instead of
// NT rows n*4 bytes apart (256 distinct 2 MB pages per box at n = 2^20).
__global__ void kv_tc_split(const double* __restrict__ V, int64_t ldv, int64_t m, int64_t n, int64_t mp, int64_t ks,
                            int mode, int blocked, float* __restrict__ Bhi, float* __restrict__ Blo) {
  // grid (ceil(ks * 32 / 256), mp): one vector per block row, contiguous columns per warp
  const int64_t c = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ks * 32) return;
  const double v = (c < m && j < n) ? V[c * ldv + j] : 0.0;
  const int64_t o = blocked ? ((j >> 5) * mp + c) * 32 + (j & 31) : c * (ks * 32) + j;
  float h = (float)v;
  if (mode == 3) {
    h = __uint_as_float(__float_as_uint(h) & 0xFFFFE000u);
    Blo[o] = (float)(v - (double)h);
  }
  Bhi[o] = h;
}

// ---------------------------------------------------------------- host side

}  // namespace

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

namespace {

template <int MODE, int NT, bool OTF, int DIM, int FAM, bool CG2 = false>
void launch_tc(const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl, TcParams p, int64_t grid,
               cudaStream_t st) {
  using Sh = TcShape<MODE, NT, OTF, CG2>;
  const size_t extra = 1024 + 8 * 96;   // alignment slack + barriers
  const size_t smem_cap = (size_t)max_smem_optin() - 1024 - extra;
  constexpr size_t BST = (size_t)Sh::B_BYTES * Sh::BOPS;
  static const int max_sa = getenv("RLD_TC_STAGES") ? atoi(getenv("RLD_TC_STAGES")) : 12;
  // B ring = TMEM A buffers (as many as TMEM leaves, <= 8); the A-source ring (K tiles
  // from HBM) takes the rest of shared memory, at least 3 stages
  int sb = Sh::NABUF;
  while (sb > 2 && smem_cap < sb * BST + 3 * (size_t)Sh::A_REGION) --sb;
  p.sb = sb;
  p.sa = (int)std::min<size_t>(max_sa, (smem_cap - sb * BST) / Sh::A_REGION);
  // one A-ring slot per converter warp parity (SA a multiple of CP): a slot shared by two converter
  // warps lets the one a whole ring phase ahead pass its kfull parity wait on the other's step
  p.sa = p.sa / Sh::CP * Sh::CP;
  if (p.sa < Sh::CP) fail(RLD_ERR_NOT_SUPPORTED, "kv_tc: shared memory below one A stage per converter warp");
  p.tmem_cols = Sh::TMEM_COLS;
  const size_t smem = (size_t)p.sa * Sh::A_REGION + (size_t)p.sb * BST + extra;
  auto kern = kv_tc_kernel<MODE, NT, OTF, DIM, FAM, CG2>;
  // the opt-in maximum once per device (not the launch's own size: another host thread could lower
  // the attribute between this thread's set and launch)
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    int dev = 0, optin = 0;
    RLD_CUDA(cudaGetDevice(&dev));
    RLD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    RLD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  });
  if (smem > 232448) fail(RLD_ERR_NOT_SUPPORTED, "kv_tc: shared memory request above the sm_100 limit");
  if constexpr (CG2) {   // CTA pairs: clusters of two on one TPC
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RLD_CUDA(cudaLaunchKernelEx(&cfg, kern, mA, mBh, mBl, p));
  } else {
    kern<<<(unsigned)grid, TC_THREADS, smem, st>>>(mA, mBh, mBl, p);
  }
  RLD_LAUNCH_CHECK();
}

template <int MODE>
void launch_tc_stored(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                      const TcParams& p, int64_t grid, cudaStream_t st, bool cg2 = false) {
  if (cg2) {
    switch (nt) {
      case 32: launch_tc<MODE, 32, false, 0, 0, true>(mA, mBh, mBl, p, grid, st); break;
      case 64: launch_tc<MODE, 64, false, 0, 0, true>(mA, mBh, mBl, p, grid, st); break;
      case 96: launch_tc<MODE, 96, false, 0, 0, true>(mA, mBh, mBl, p, grid, st); break;
      default: launch_tc<MODE, 128, false, 0, 0, true>(mA, mBh, mBl, p, grid, st); break;
    }
    return;
  }
  switch (nt) {
    case 32: launch_tc<MODE, 32, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    case 64: launch_tc<MODE, 64, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    case 96: launch_tc<MODE, 96, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    case 144: launch_tc<MODE, 144, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
    default: launch_tc<MODE, 128, false, 0, 0>(mA, mBh, mBl, p, grid, st); break;
  }
}

template <int DIM, int FAM>
void launch_tc_otf_nt(int nt, const CUtensorMap& mA, const CUtensorMap& mBh, const CUtensorMap& mBl,
                      const TcParams& p, int64_t grid, cudaStream_t st) {
  switch (nt) {
    case 32: launch_tc<3, 32, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
    case 64: launch_tc<3, 64, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
    case 144: launch_tc<3, 144, true, DIM, FAM>(mA, mBh, mBl, p, grid, st); break;
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

// 2-D map over the blocked points [ceil(n/32) * 8][32] fp32: box {32, 8} = the 32
// column points of one k-step (1 KB contiguous)
CUtensorMap make_points_map(const float* pts, int64_t n) {
  CUtensorMap m;
  const int64_t ks = ceil_div(n, TC_BK);
  cuuint64_t dims[2] = {(cuuint64_t)TC_BK, (cuuint64_t)(ks * 8)};
  cuuint64_t strides[1] = {(cuuint64_t)TC_BK * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, 8};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(pts), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RLD_ERR_CUDA, "cuTensorMapEncodeTiled (points) failed (" + std::to_string((int)r) + ")");
  return m;
}

// B operand layout: k-step blocks (default; contiguous TMA boxes) or row-major
// vectors (RLD_TC_BLAYOUT=0), for A/B measurements.
bool blocked_b() {
  static const bool b = !(getenv("RLD_TC_BLAYOUT") && getenv("RLD_TC_BLAYOUT")[0] == '0');
  return b;
}

}  // namespace

bool kv_tc_supported(const KvOperand& op) {
  if (op.dtype != RLD_FP32) return false;
  if (op.K == nullptr) return op.pts4 != nullptr && op.kp.d <= 4 && op.tc_mode == 3;   // on the fly
  if (op.tiled) return true;
  return (op.ldk % 4) == 0 && (reinterpret_cast<uintptr_t>(op.K) % 16) == 0;
}

// Y (m x rows, float64, row stride ldy) = V (m x n float64 rows) K^T on the tensor cores.
namespace {
// vectors per pass (two TMEM accumulators + A buffers within 512 columns): NT = 32..128 in
// steps of 32, or 144 when that saves a pass of a stored-K product with 129..144 vectors
// (0.43 vs 0.47 ms at n = 16384, m = 140).  For more vectors NT = 144 measured slower than
// passes of 96 / 128 (config 2 sketch, m = 266: 0.82 vs 0.72 ms; RLD_TC_NT144=1 forces it).
void tc_passes(const KvOperand& op, int64_t m, int& npass, int& width) {
  static const int wide_env = getenv("RLD_TC_NT144") ? atoi(getenv("RLD_TC_NT144")) : -1;
  const bool otf = op.K == nullptr;
  // on the fly every pass regenerates its K tiles; passes of 144 would save one at configs 4/5
  // (8 instead of 9, 15 instead of 17) but measured slower per pass (3 TMEM A buffers): 988 vs
  // 754 ms (config 4 sketch), 2091 vs 1639 ms (config 5, n = 262144).  Opt-in RLD_TC_OTF144=1.
  static const bool otf_wide = getenv("RLD_TC_OTF144") && getenv("RLD_TC_OTF144")[0] == '1';
  if (m > 128 && otf && otf_wide && ceil_div(m, 144) < ceil_div(m, 128)) {
    npass = (int)ceil_div(m, 144);
    width = 144;
    return;
  }
  const bool wide = wide_env == 1 || (wide_env < 0 && m > 128 && m <= 144);
  if (m > 128 && !otf && wide) {
    npass = (int)ceil_div(m, 144);
    width = (int)(ceil_div(ceil_div(m, npass), 16) * 16);
    width = width > 128 ? 144 : (int)(ceil_div(width, 32) * 32);
  } else {
    npass = (int)ceil_div(m, 128);
    width = (int)(ceil_div(ceil_div(m, npass), 32) * 32);
    if (otf && width == 96) width = 128;   // on-the-fly kernels come in NT = 32, 64, 128
  }
}
}  // namespace

bool kv_tc_b_layout(const KvOperand& op, int64_t m, KvWorkspace& ws, TcBLayout& out) {
  if (!kv_tc_supported(op) || (!op.tiled && getenv("RLD_NO_TC"))) return false;
  int npass = 0, width = 0;
  tc_passes(op, m, npass, width);
  const int64_t ks = ceil_div(op.n, TC_BK);
  out.mp = (int64_t)npass * width;
  out.ks = ks;
  out.blocked = blocked_b() ? 1 : 0;
  out.mode = op.tc_mode;
  ws.bhi.reserve(sizeof(float) * out.mp * ks * 32);
  if (op.tc_mode == 3) ws.blo.reserve(sizeof(float) * out.mp * ks * 32);
  out.bhi = ws.bhi.as<float>();
  out.blo = op.tc_mode == 3 ? ws.blo.as<float>() : nullptr;
  return true;
}

void kv_product_tc(const KvOperand& op, int mode, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                   KvWorkspace& ws, cudaStream_t st, bool presplit) {
  if (op.K == nullptr && !presplit && kv_otf_f16_enabled()) {
    kv_product_otf16(op, m, V, ldv, Y, ldy, ws, st);
    return;
  }
  // wide products of a stored (tiled) fp32 K: tensor-bound, so the fp16 head / tail kernel at twice
  // the tf32 rate; the HBM-bound Lanczos block (m <= 64) stays on 3xTF32
  if (op.K && op.tiled && op.rowscale && m > 64 && mode == 3 && !presplit && kv_otf_f16_enabled()) {
    kv_product_otf16(op, m, V, ldv, Y, ldy, ws, st);
    return;
  }
  const int64_t n = op.n, rows = op.rows;
  const int ks = (int)ceil_div(n, TC_BK);
  int npass = 0, width = 0;
  tc_passes(op, m, npass, width);
  const bool otf = op.K == nullptr;
  const int64_t mp = (int64_t)npass * width;
  ws.bhi.reserve(sizeof(float) * mp * ks * 32);
  if (mode == 3) ws.blo.reserve(sizeof(float) * mp * ks * 32);
  if (!presplit) {
    const dim3 sgrid((unsigned)ceil_div((int64_t)ks * 32, 256), (unsigned)mp);
    kv_tc_split<<<sgrid, 256, 0, st>>>(V, ldv, m, n, mp, ks, mode, blocked_b(), ws.bhi.as<float>(),
                                        mode == 3 ? ws.blo.as<float>() : nullptr);
    RLD_LAUNCH_CHECK();
  }
  const int G = sm_count();
  const int tiles = (int)ceil_div(rows, TC_BM);
  // CTA pairs (stored K, NT >= 64; RLD_TC_CG2=0/1 forces off/on): 2-SM MMAs (cta_group::2,
  // M = 256), each SM loads half of the B operand, the schedule runs over pair tiles of 256 rows.
  // Config 2 sketch (m = 266) 0.69 vs 0.74 ms, config 3 Lanczos (m = 64) 3.57 vs 3.70 ms; the
  // HBM-bound m = 32 product is unchanged (0.215 vs 0.212 ms), so it keeps single CTAs.
  static const int cg2_env = getenv("RLD_TC_CG2") ? atoi(getenv("RLD_TC_CG2")) : -1;
  const bool cg2_ok = !otf && (width == 32 ? mode == 3 : (width / 2) % 16 == 0) && width <= 128;
  const bool cg2 = cg2_ok && (cg2_env == 1 || (cg2_env < 0 && width >= 64));
  const int units = cg2 ? (tiles + 1) / 2 : tiles;
  const int per = cg2 ? 2 : 1;
  const int64_t total = (int64_t)units * ks;
  const int64_t Gl = std::min<int64_t>(std::max(1, G / (npass * per)), total);
  Sched sc{};
  sc.ks = ks;
  sc.G = (int)Gl;
  {
    static const bool streamk_only = getenv("RLD_TC_STREAMK") && getenv("RLD_TC_STREAMK")[0] == '1';
    sc.R = streamk_only ? 0 : (int)(units / Gl);
  }
  sc.tail_total = (int64_t)(units - sc.R * Gl) * ks;
  int segs = 1;
  for (int t = sc.R * (int)Gl; t < units; ++t) {
    const int64_t x0 = (int64_t)(t - sc.R * Gl) * ks;
    segs = (int)std::max<int64_t>(
        segs, cta_of_step(x0 + ks - 1, sc.tail_total, Gl) - cta_of_step(x0, sc.tail_total, Gl) + 1);
  }
  const int64_t nblocks = Gl * npass * per;
  // tiled K: one 16 KB box = 128 contiguous rows of 128 bytes of the [tiles * ks * 128][32] view
  const CUtensorMap mA = otf ? make_points_map(op.pts4, n)
                             : op.tiled ? make_map(static_cast<const float*>(op.K), TC_BK,
                                                   (int64_t)ceil_div(rows, TC_BM) * ks * TC_BM, TC_BK, TC_BM)
                                        : make_map(static_cast<const float*>(op.K), n, rows, op.ldk, TC_BM);
  TcParams p{};
  p.pts = op.pts4;
  p.mp = (int)mp;
  p.a_tiled = op.tiled ? 1 : 0;
  p.n = n;
  p.row0 = op.row0;
  p.rows = rows;
  p.family = op.kp.family;
  p.diag = (float)op.kp.diag;
  p.la2 = (float)std::log2(op.kp.a2);
  p.sched = sc;
  p.ks = ks;
  p.tiles = tiles;
  p.npass = npass;
  p.segs = segs;
  {
    static const int dbg = getenv("RLD_TC_DEBUG") ? atoi(getenv("RLD_TC_DEBUG")) : 0;
    p.debug = dbg;
    static const int wm = getenv("RLD_TC_WAIT") ? atoi(getenv("RLD_TC_WAIT")) : 1;
    static const int wns = getenv("RLD_TC_WAIT_NS") ? atoi(getenv("RLD_TC_WAIT_NS")) : 256;
    p.wait_mode = wm;
    p.wait_ns = (uint32_t)wns;
    static const int asem = getenv("RLD_TC_ARRIVE") ? atoi(getenv("RLD_TC_ARRIVE")) : 2;
    p.arrive_sem = asem;
  }
  static const bool prof_on = getenv("RLD_TC_PROFILE") != nullptr;
  static DevBuf prof_buf;
  if (prof_on) {
    prof_buf.reserve(sizeof(unsigned long long) * 16 * (size_t)nblocks);
    RLD_CUDA(cudaMemsetAsync(prof_buf.ptr, 0, sizeof(unsigned long long) * 16 * (size_t)nblocks, st));
    p.prof = prof_buf.as<unsigned long long>();
  }
  {
    static const int sync_k = [] {   // power of two (the producer tests kstep & (sync_k - 1))
      int v = getenv("RLD_TC_SYNC_K") ? atoi(getenv("RLD_TC_SYNC_K")) : 2048;
      int pw = 0;
      while (v > 1 && (1 << (pw + 1)) <= v) ++pw;
      return v > 0 ? (1 << pw) : 0;
    }();
    p.sync_k = (sc.R > 1 || (sc.R == 1 && sc.tail_total > 0)) && g_live_handles.load() <= 1 ? sync_k : 0;
    static const int sync_all = getenv("RLD_TC_SYNC_ALL") ? atoi(getenv("RLD_TC_SYNC_ALL")) : 0;
    static const int sync_k_multi = getenv("RLD_TC_SYNC_K_MULTI") ? atoi(getenv("RLD_TC_SYNC_K_MULTI")) : 0;
    p.sync_all = (npass > 1 && sync_all) ? 1 : 0;
    if (p.sync_all && sync_k_multi > 0 && p.sync_k > 0) p.sync_k = sync_k_multi;
    ws.tc_sync.reserve(sizeof(unsigned int) * npass);
    p.sync = ws.tc_sync.as<unsigned int>();
    if (p.sync_k > 0) RLD_CUDA(cudaMemsetAsync(p.sync, 0, sizeof(unsigned int) * npass, st));
  }
  ws.tc_partial.reserve(sizeof(float) * (size_t)npass * tiles * segs * width * TC_BM);
  p.partial = ws.tc_partial.as<float>();
  const bool blk = blocked_b();
  const int64_t bcols = blk ? TC_BK : (int64_t)ks * TC_BK, brows = blk ? mp * ks : mp;
  const int bbox = (cg2 && !(mode == 3 && width == 32)) ? width / 2 : width;   // B rows per TMA box
  const CUtensorMap mBh = make_map(ws.bhi.as<float>(), bcols, brows, bcols, bbox);
  const CUtensorMap mBl = mode == 3 ? make_map(ws.blo.as<float>(), bcols, brows, bcols, bbox) : mBh;
  p.bcol_step = blk ? 0 : TC_BK;
  p.brow_step = blk ? (int)mp : 0;
  if (otf) {
    launch_tc_otf(op.kp.d, op.kp.family, width, mA, mBh, mBl, p, Gl * npass, st);
  } else {
    if (mode == 3)
      launch_tc_stored<3>(width, mA, mBh, mBl, p, nblocks, st, cg2);
    else
      launch_tc_stored<1>(width, mA, mBh, mBl, p, nblocks, st, cg2);
  }
  if (prof_on) {
    std::vector<unsigned long long> h(16 * (size_t)nblocks);
    RLD_CUDA(cudaMemcpyAsync(h.data(), prof_buf.ptr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    double a[16] = {0};
    for (int64_t c = 0; c < nblocks; ++c)
      for (int k = 0; k < 16; ++k) a[k] += (double)h[c * 16 + k];
    const double steps = a[13] > 0 ? a[13] : 1;
    if (cg2) {   // per rank: leaders (even blocks) and peers (odd blocks)
      for (int rk = 0; rk < 2; ++rk) {
        double b[16] = {0};
        for (int64_t c = rk; c < nblocks; c += 2)
          for (int k = 0; k < 16; ++k) b[k] += (double)h[c * 16 + k];
        fprintf(stderr, "[kv_tc prof rank %d] per k-step: producer wait %.0f / loop %.0f | conv wait %.0f loop %.0f | drain wait %.0f loop %.0f\n",
                rk, 2 * b[0] / steps, 2 * b[1] / steps, 2 * b[7] / steps, 2 * b[10] / steps, 2 * b[11] / steps,
                2 * b[12] / steps);
      }
    }
    fprintf(stderr,
            "[kv_tc prof] m=%ld n=%ld nt=%d otf=%d per k-step cycles: producer wait %.0f / loop %.0f | mma wait acc %.0f "
            "afull %.0f issue %.0f loop %.0f | conv(w4) wait full %.0f loop %.0f | drain wait %.0f loop %.0f\n",
            (long)m, (long)n, width, (int)otf, a[0] / steps, a[1] / steps, a[2] / steps, a[4] / steps,
            a[5] / steps, a[6] / steps, a[7] / steps, a[10] / steps, a[11] / steps, a[12] / steps);
  }
  const dim3 rgrid((unsigned)tiles, (unsigned)ceil_div(m, RED_COLS));
  kv_tc_reduce<<<rgrid, 256, 0, st>>>(p.partial, sc, tiles, segs, width, m, rows, Y, ldy, cg2 ? 1 : 0);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
