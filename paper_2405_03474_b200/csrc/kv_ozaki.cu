// Float64-accurate K x V on the INT8 tensor cores (tcgen05 kind::i8): exact integer slicing
// ("Ozaki scheme").  The stored-K product of the float64 estimate (src/estimators.py:72,
// src/precond.py:186, 189) at 3-4x the FP64 (DMMA) peak.
//
// Slicing (exact, deterministic):
//   each row i of K gets sigma_i = 2^e with 2.016 max_j |K_ij| < sigma_i <= 4.032 max_j |K_ij|, each
//   vector c of V gets tau_c likewise; x = K_ij / sigma_i, |x| < 127 / 256, is cut into S = 7 signed
//   digits of the integer rint(x 2^56) (digits7: balanced base 256, d_6..d_1 in [-128, 127], the top
//   d_0 in [-127, 127] by the bound on |x|) -- the whole int8 range, 56 bits in 7 bytes:
//       K_ij = sigma_i (sum_s d_s 2^{-8 (s+1)} + rho 2^{-56}),   |rho| <= 1/2
//   (a round-to-nearest integer leaves an unbiased remainder, so the dropped terms do not add up
//   coherently over the n-term sums).
//   Then (K V^T)_ic = sigma_i tau_c sum_{s+t <= 6} 2^{-8 (s+t+2)} sum_j d_s[i,j] e_t[c,j] + err,
//   28 int8 x int8 products accumulated EXACTLY in int32, combined in float64.  The dropped digits
//   and slice pairs (s + t >= 7: <= 6 x 2^14 x 2^-72 per term) bound |err| <= ~2^-52 sigma_i tau_c per
//   term of the j-sum: the float64 GEMM's own rounding level, scaled by the row / column maxima
//   instead of the entries.  (Round 2 first used 8 digits of 7 bits, |d| <= 64: the same 56 bits
//   and the same dropped-term level with 36 pairs and 8 bytes per entry.)
//
// Kernel (one CTA per SM, 256 threads; grid = column passes x row tiles x k splits):
//   warp 0  producer: per 32-column k-step ONE bulk copy (TMA engine) of all 7 K slices' tile
//           (7 x 128 rows x 32 B = 28 KB) and one of all 7 V slices' (7 x 64 vectors x 32 B), both
//           stored pre-swizzled in the k-step-tiled global image (a 3-D TMA box with 32-byte rows
//           moved 1536 32-byte rows per step and bound the product), 5-stage ring;
//   warp 1  MMA issuer (one thread): the 28 slice pairs of a k-step as 10 tcgen05.mma kind::i8
//           M = 128, K = 32, N = 64..256 from shared-memory descriptors -- A slice s against the
//           stacked V slices 0..6-s, pair (s, t) landing in the int32 TMEM accumulator of its
//           diagonal d = s + t (7 x 64 columns) -- and a commit frees the stage;
//   warp 2  TMEM owner;
//   warps 4-7 drain: after the CTA's k range (<= 16384 columns: the int32 bound, 7 pairs x 128^2 x
//           16384 = 7 2^28 < 2^31) they read the 7 accumulators (thread = row), form
//           sum_d 2^{-8(d+2)} I_d in float64, scale by sigma_i tau_c and store.
// k splits (at least n / 16384 of them) write float64 partials that a fixed-order reduce adds
// (deterministic).
#include <cuda.h>

#include <thrust/execution_policy.h>
#include <thrust/scan.h>

#include <algorithm>
#include <mutex>

#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"
#include "crt_common.cuh"

namespace rld {

namespace {

constexpr int OZ_S = OZ_NSLICES;    // float64: 7 digits (bytes) per operand, diagonals d = s + t <= 6 (28 pairs)
constexpr int OZ_S32 = 3;           // float32 K: 3 digits (24 bits relative to the row scale) ...
constexpr int OZ_V32 = 4;           // ... against 4 digits of V, diagonals d <= 3 (9 pairs)
constexpr int OZ_DBITS = 8;         // bits per digit
constexpr int OZ_BM = 128;          // K rows per tile (UMMA M)
constexpr int OZ_BN = 64;           // vectors per column pass (UMMA N)
constexpr int OZ_BK = 32;           // int8 columns per k-step (UMMA K for kind::i8, one 32-byte row)
constexpr int64_t OZ_KMAX = 16384;  // columns per CTA: <= 7 pairs x 128^2 x 16384 = 7 2^28 < 2^31 (exact int32)
constexpr int OZ_THREADS = 256;
constexpr uint32_t OZ_A_SLICE = OZ_BM * OZ_BK;            // 4 KB
constexpr uint32_t OZ_B_SLICE = OZ_BN * OZ_BK;            // 2 KB
// SA digits of K against SB >= SA digits of V, pairs s + t <= SB - 1 (one TMEM accumulator per diagonal)
// BN vectors per column pass: 64, or 128 for the wide products of the float32 variant (4 x 128 = all
// 512 TMEM columns: half as many (CTA, k-step) handshakes per product)
template <int SA, int SB, int BN = OZ_BN>
struct OzCfg {
  static constexpr uint32_t A_BYTES = SA * OZ_A_SLICE;          // 28 KB (float64) / 12 KB (float32)
  static constexpr uint32_t B_SLICE = BN * OZ_BK;               // 2 KB / 4 KB (BN = 128)
  static constexpr uint32_t B_BYTES = SB * B_SLICE;             // 14 KB / 8 KB / 16 KB
  static constexpr int PC = 256 / BN;                           // V slices per MMA piece (N <= 256)
  // kept k-steps per pipeline stage (one mbarrier handshake and one commit per stage): the float32
  // variant's steps carry one to three small MMAs and are bound by that handshake, so it groups 2
  static constexpr int GROUP = SA == OZ_S ? 1 : (BN == OZ_BN ? 3 : 2);
  static constexpr uint32_t STEP = A_BYTES + B_BYTES;           // 42 KB / 20 KB
  static constexpr uint32_t STAGE = GROUP * STEP;
  static constexpr int STAGES = SA == OZ_S ? 5 : 3;
  // columns per CTA, exact in int32: <= min(SA, SB) pairs per diagonal x 128^2 x KMAX < 2^31
  static constexpr int64_t KMAX = SA == OZ_S ? OZ_KMAX : 2 * OZ_KMAX;
  static constexpr int SMEM = STAGES * (int)STAGE + 1024 + 256;
  static constexpr uint32_t ACC_COLS = SB * BN;                 // 448 / 256 / 512 accumulator columns
  static constexpr uint32_t TMEM_COLS = ACC_COLS <= 256 ? 256 : 512;   // allocation (a power of two)
};

// UMMA shared-memory descriptor: K-major operand, 32-byte swizzle atoms (8 rows x 32 B), 8-row
// groups 256 B apart -- the layout TMA writes for a box with a 32-byte inner dimension and
// CU_TENSOR_MAP_SWIZZLE_32B.
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);   // start address
  d |= (uint64_t)1 << 16;                    // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;           // stride byte offset: 8 rows x 32 B
  d |= (uint64_t)1 << 46;                    // descriptor version (sm100)
  d |= (uint64_t)6 << 61;                    // layout: SWIZZLE_32B
  return d;
}

// kind::i8 instruction descriptor: D s32, A and B s8, K-major, M = 128, N
constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                       // c_format S32
         | (1u << 7)                     // a_format S8 (signed)
         | (1u << 10)                    // b_format S8
         | ((uint32_t)(N >> 3) << 17)    // n_dim
         | ((uint32_t)(M >> 4) << 24);   // m_dim
}

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------------------------------------
// Slicing.  Global layout = the shared-memory image of one k-step: for tile t (TR rows) and k-step
// ks (32 columns) the 7 slices' [TR][32]-byte tiles are contiguous, ((t KS + ks) 7 + s) TR 32 bytes,
// each already in the 32-byte-swizzle order (Swizzle<1,4,3>: the two 16-byte halves of a row swap
// in rows 4..7 of every 8-row atom) the UMMA descriptor expects -- so a stage is ONE bulk copy.
// Rows >= rows and columns >= n are zero.

// The 7 signed base-256 digits of x (|x| <= 127 / 256 - 2^-10, guaranteed by scale_exponent):
// K = rint(x 2^56) (x 2^56 is exact in float64 or rounds once), then balanced digits from the bottom,
// d_s in [-128, 127] for s = 6..1 and the top d_0 = what remains: |K| 2^-48 <= 127 - 2^-2 and the
// carry adds at most 1/2, so |d_0| <= 127 and every digit is an int8:
// x = sum_s d_s 2^{-8(s+1)} + rho 2^-56, |rho| <= 1/2.  Integer work on the ALU pipe (one F2I per
// entry).  Also returns K' = sum_{s<6} d_s 256^{5-s} (the CRT integer, kv_crt.cu) and 7 - the number
// of leading zero digits.
// 32-bit arithmetic: the 64-bit integer is never formed for the digits.  hi = rint(x 2^24) and
// lo = rint((x 2^24 - hi) 2^32) (the difference is exact in float64) give the same integer
// hi 2^32 + lo = rint(x 2^56); the low three digits come from lo, the other four from
// hi 256 + (what is left of lo) -- about half the ALU work of the 64-bit shifts and masks it replaces
// (the slicing of K from the points is bound by this integer work, not by its float64 exp).
template <int NB>
__device__ __forceinline__ void low_digits(int& v, int* d_top_down_end) {   // NB digits from the bottom of v
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int dd = ((v + 128) & 255) - 128;
    *(d_top_down_end - i) = dd;
    v = (v - dd) >> 8;   // exact (arithmetic shift)
  }
}
template <int S>
__device__ __forceinline__ void digits8(double x, int (&d)[S], long long& kprime, int& nz) {
  nz = 0;        // (the callers that need it derive it from the packed slices)
  kprime = 0;
  if constexpr (S <= 4) {   // |x 2^(8 S)| <= 63/128 2^32 < 2^31
    int v = __double2int_rn(x * (double)(1ull << (OZ_DBITS * S)));
    low_digits<S - 1>(v, &d[S - 1]);
    d[0] = v;
  } else {
    static_assert(S == 7, "7 digits: 3 + 4 bytes");
    const int hi = __double2int_rn(x * 16777216.0);                       // rint(x 2^24), |hi| < 2^23
    const double r = fma(x, 16777216.0, -(double)hi);                     // exact, |r| <= 1/2
    const long long lo = __double2ll_rn(r * 4294967296.0);                // |lo| <= 2^31
    const int d6 = (((int)lo + 128) & 255) - 128;
    const long long l1 = (lo - d6) >> 8;                                  // |l1| <= 2^23
    int v = (int)l1;
    d[6] = d6;
    low_digits<2>(v, &d[5]);                                              // d5, d4; |v| <= 128 left
    kprime = ((long long)hi << 24) + l1;                                  // (K - d6) / 256: the CRT integer
    int u = hi * 256 + v;                                                 // |u| < 2^31
    low_digits<3>(u, &d[3]);                                              // d3, d2, d1
    d[0] = u;
  }
}

// Exponent e of the scale sigma = 2^(e+1) for a row (vector) of maximum mx = f 2^e', f in [0.5, 1):
// e = e', or e' + 1 when f > 63/64, so that |x| = |a| / sigma <= 63/128 and the top base-256 digit of
// rint(x 2^56) stays within int8 (digits8: |d_0| <= 126.5)
__host__ __device__ inline int oz_scale_exp(double mx) {
  int e = 0;
  const double f = frexp(mx, &e);
  return f > 0.984375 ? e + 1 : e;
}

// scale[row] = sigma = 2^e with 2 max_j |A_row,j| < sigma <= 4.07 max (1 for an all-zero row)
__global__ void ozaki_scale_kernel(const double* __restrict__ A, int64_t lda, int64_t n, double* __restrict__ scale) {
  const int64_t row = blockIdx.x;
  const double* a = A + row * lda;
  double mx = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, fabs(a[j]));
  __shared__ double red[32];
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    scale[row] = mx > 0.0 ? ldexp(1.0, oz_scale_exp(mx) + 1) : 1.0;   // |a| / sigma <= 63/128
  }
}

// The same scales with the row split over many CTAs (the one-CTA-per-row version left most SMs idle
// for the m = 64 Lanczos block): per-chunk maxima of |A| merged with atomicMax on their bit patterns
// (non-negative doubles order like unsigned integers) into `bits` (zeroed), then converted in place.
constexpr int OZ_MAX_CHUNK = 4096;
__global__ void ozaki_rowmax_kernel(const double* __restrict__ A, int64_t lda, int64_t n,
                                    unsigned long long* __restrict__ bits) {
  const int64_t row = blockIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * OZ_MAX_CHUNK, j1 = min64(n, j0 + OZ_MAX_CHUNK);
  const double* a = A + row * lda;
  double mx = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) mx = fmax(mx, fabs(a[j]));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(bits + row, (unsigned long long)__double_as_longlong(mx));
}
__global__ void ozaki_scale_finish_kernel(int64_t rows, double* __restrict__ scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double mx = __longlong_as_double((long long)reinterpret_cast<unsigned long long*>(scale)[i]);
  scale[i] = mx > 0.0 ? ldexp(1.0, oz_scale_exp(mx) + 1) : 1.0;
}

// one thread per (padded row, 16-column half of a k-step): 7 exact digits of 16 entries of A / sigma,
// written as one 16-byte store per slice (the half lands at byte 16 h ^ 16 in rows 4..7 of an atom)
template <int TR, int S>
__global__ void ozaki_digits_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t n,
                                    const double* __restrict__ scale, int64_t KS, int8_t* __restrict__ q) {
  const int64_t total = ceil_div(rows, TR) * TR * KS * 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    // h fastest, then the tile row: a warp writes 512 contiguous bytes of one slice image per store
    const int h = (int)(e & 1);
    const int i = (int)((e >> 1) % TR);
    const int64_t rest = (e >> 1) / TR;
    const int64_t ks = rest % KS;
    const int64_t t = rest / KS;
    const int64_t row = t * TR + i;
    const int64_t j0 = ks * OZ_BK + 16 * h;
    int ee = 0;
    if (row < rows) frexp(scale[row], &ee);   // sigma = 2^(ee-1): x = a 2^(1-ee), exact
    // one multiply by the exact power of two when it is a normal double, ldexp otherwise (no
    // overflow / underflow of the multiplier for extreme scales)
    const bool mul = ee > -1000 && ee < 1000;
    const double f = mul ? __longlong_as_double((long long)(1023 + 1 - ee) << 52) : 1.0;
    uint32_t w[S][4];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t j = j0 + k;
      const double a = (row < rows && j < n) ? A[row * lda + j] : 0.0;
      const double r = mul ? a * f : ldexp(a, 1 - ee);
      int dg[S];
      long long kp;
      int nzk;
      digits8<S>(r, dg, kp, nzk);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const uint32_t b = (uint32_t)(uint8_t)(int8_t)dg[s];
        if ((k & 3) == 0) w[s][k >> 2] = b;
        else w[s][k >> 2] |= b << (8 * (k & 3));
      }
    }
    const uint32_t o = (uint32_t)(i * OZ_BK + 16 * h);
    const uint32_t phys = o ^ (((o >> 7) & 1u) << 4);
    int8_t* base = q + (t * KS + ks) * (int64_t)S * TR * OZ_BK + phys;
#pragma unroll
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint4*>(base + (int64_t)s * TR * OZ_BK) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
  }
}

// The same sliced image straight from the points (stored float64 path, no float64 K in HBM): the
// entries are kgen.cu's float64 values (direct differences, kernel_value_f64, exact diagonal) and
// every row's maximum is the diagonal a^2 + jitter (a stationary kernel: |K_ij| <= a^2), so sigma is
// known up front.  Bitwise the slices of the stored float64 K.
// Kr != null: also the CRT residue image (kv_crt.cu) of K' = sum_{s<7} d_s 128^{6-s}, same
// swizzled position, ((t L + l) KS + ks) 4096 + phys -- in the same pass (no second read of the
// 34 GB slice image).  Thread = EL consecutive columns of one row (EL = 8: 80 registers, 3 CTAs per
// SM; 16 columns per thread held 128 registers and ran at 25 % occupancy, latency-bound).
template <bool CRT, int EL, int DMAX, int S>
__global__ void __launch_bounds__(256)
ozaki_points_kernel(const double* __restrict__ X, int64_t n, KernelParams kp, int64_t row0,
                    int64_t rows, int64_t KS, int8_t* __restrict__ q, int8_t* __restrict__ Kr, int* __restrict__ knz,
                    const uint32_t* __restrict__ koff) {
  constexpr int TR = OZ_BM;
  constexpr int PARTS = OZ_BK / EL;          // threads per (row, k-step)
  constexpr int W = EL / 4;                  // 32-bit words per slice
  const int d = kp.d;
  const int ee = oz_scale_exp(kp.diag > 0.0 ? kp.diag : 1.0);   // sigma = 2^(ee+1), x = v 2^-(ee+1)
  const double scl = ldexp(1.0, -(ee + 1));    // exact power of two
  const int64_t total = ceil_div(rows, TR) * TR * KS * PARTS;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int h = (int)(e % PARTS);
    const int i = (int)((e / PARTS) % TR);
    const int64_t rest = (e / PARTS) / TR;
    const int64_t ks = rest % KS;
    const int64_t t = rest / KS;
    const int64_t row = t * TR + i;
    const int64_t gi = row0 + row;
    const int64_t j0 = ks * OZ_BK + EL * h;
    // sparse image (koff): knz is an INPUT, the slices kept of this block (a bound from the point
    // boxes, ozaki_sparse_plan); a block keeping none is neither evaluated nor stored.  Uniform over
    // the 512 consecutive threads of a block, so whole warps leave together.
    int keep = S;
    if (koff) {
      keep = knz[t * KS + ks];
      if (keep == 0) continue;
    }
    double xi[DMAX];   // DMAX = 4: registers (d <= 4), else local memory
#pragma unroll
    for (int k = 0; k < DMAX; ++k) xi[k] = (k < d && row < rows) ? X[gi * d + k] : 0.0;
    uint32_t w[S][W];
    long long kq[EL];   // CRT: K' of the EL entries
    int nz = 0;         // slices from the first nonzero digit of any of the EL entries: 7 - leading zero slices
#pragma unroll
    for (int k = 0; k < EL; ++k) {
      const int64_t j = j0 + k;
      double v = 0.0;
      if (row < rows && j < n) {
        if (j == gi) {
          v = kp.diag;
        } else {
          double r2 = 0.0;
#pragma unroll
          for (int c = 0; c < DMAX; ++c) {
            if (c < d) {
              const double df = xi[c] - X[j * d + c];
              r2 = fma(df, df, r2);
            }
          }
          v = kernel_value_f64(kp, r2);
        }
      }
      int dg[S];
      long long kp;
      int nzk;
      digits8<S>(v * scl, dg, kp, nzk);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const uint32_t b = (uint32_t)(uint8_t)(int8_t)dg[s];
        if ((k & 3) == 0) w[s][k >> 2] = b;
        else w[s][k >> 2] |= b << (8 * (k & 3));
      }
      if (CRT) kq[k] = kp;
    }
    // slices from the first one with a nonzero digit in any of this thread's EL entries
#pragma unroll
    for (int sl = S - 1; sl >= 0; --sl) {
      uint32_t any = 0;
#pragma unroll
      for (int q4 = 0; q4 < W; ++q4) any |= w[sl][q4];
      if (any) nz = S - sl;
    }
    // a warp holds 8 rows x 4 column parts of one (tile, k-step) block: reduce, one atomic per warp
    if (knz && !koff) {
      const int wnz = (int)__reduce_max_sync(0xffffffffu, (unsigned)nz);
      if ((threadIdx.x & 31) == 0 && wnz > 0) atomicMax(knz + t * KS + ks, wnz);
    }
    const uint32_t o = (uint32_t)(i * OZ_BK + EL * h);
    const uint32_t phys = o ^ (((o >> 7) & 1u) << 4);
    // dense: all S slices of the block; sparse: its last `keep` slices at slice offset koff[block]
    int8_t* base = koff ? q + ((int64_t)koff[t * KS + ks] - (S - keep)) * (int64_t)(TR * OZ_BK) + phys
                        : q + (t * KS + ks) * (int64_t)S * TR * OZ_BK + phys;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (s < S - keep) continue;
      if (W == 4)
        *reinterpret_cast<uint4*>(base + (int64_t)s * TR * OZ_BK) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
      else
        *reinterpret_cast<uint2*>(base + (int64_t)s * TR * OZ_BK) = make_uint2(w[s][0], w[s][1]);
    }
    if (CRT) {
      // residues on the FP32 pipe: K' = a 2^36 + b 2^24 + c 2^12 + d (|a| < 2^12.02, 0 <= b, c, d < 2^12);
      // acc = a (2^36 mod p) + b (2^24 mod p) + c (2^12 mod p) + d with symmetric constants (|.| <= 128)
      // is an exact fp32 integer (|acc| < 2^21); r = acc - p rint(acc / p) (rint by the 1.5 2^23
      // magic add: exact for odd p, whose residues never tie) and its int8 byte is the low byte of
      // r + 1.5 2^23 (for p = 256 a tie gives +-128, the same class mod 256)
      float fa[EL], fb[EL], fc[EL], fd[EL];
#pragma unroll
      for (int k = 0; k < EL; ++k) {
        const long long kk = kq[k];
        fa[k] = (float)(int)(kk >> 36);
        fb[k] = (float)(int)((kk >> 24) & 0xFFF);
        fc[k] = (float)(int)((kk >> 12) & 0xFFF);
        fd[k] = (float)(int)(kk & 0xFFF);
      }
      constexpr float MAGIC = 12582912.0f;
#pragma unroll
      for (int l = 0; l < CRT_L; ++l) {
        const int p = crt_mod(l);
        const float A = (float)crt_pow2_sym(36, p), B = (float)crt_pow2_sym(24, p), C = (float)crt_pow2_sym(12, p);
        const float pf = (float)p, inv = 1.0f / (float)p;
        uint32_t wv[W];
#pragma unroll
        for (int k = 0; k < EL; ++k) {
          const float acc = fmaf(fa[k], A, fmaf(fb[k], B, fmaf(fc[k], C, fd[k])));
          const float qq = fmaf(acc, inv, MAGIC) - MAGIC;
          const float rr = fmaf(-qq, pf, acc);
          const uint32_t b8 = __float_as_uint(rr + MAGIC) & 0xFFu;
          if ((k & 3) == 0) wv[k >> 2] = b8;
          else wv[k >> 2] |= b8 << (8 * (k & 3));
        }
        int8_t* dst = Kr + ((t * CRT_L + l) * KS + ks) * (int64_t)TR * OZ_BK + phys;
        if (W == 4)
          *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        else
          *reinterpret_cast<uint2*>(dst) = make_uint2(wv[0], wv[1]);
      }
    }
  }
}

// ---- plan of a SPARSE slice image (float32 K, points in Morton order): boxes of the points of each
// 128-row tile and each 32-column k-step, then per (tile, k-step) block an upper bound on |K| from
// the boxes' distance and from it how many of the S = 3 slices can be nonzero (the balanced digits
// of k = rint(x 2^24): none when |k| < 1/2, only the last when |k| <= 127, the last two when
// |k| <= 32639).  A block keeps that many trailing slices; an exclusive scan gives their offsets.
__global__ void oz_boxes_kernel(const double* __restrict__ X, int64_t first, int64_t count, int d, int64_t group,
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

__global__ void oz_keep_kernel(const double* __restrict__ tbox, const double* __restrict__ kbox, int64_t tiles,
                               int64_t KS, int d, KernelParams kp, double scl, int64_t row0, int64_t rows,
                               int* __restrict__ keep) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tiles * KS) return;
  const int64_t t = e / KS, k = e - t * KS;
  double r2 = 0.0;
  for (int c = 0; c < d; ++c) {
    const double g = fmax(0.0, fmax(kbox[k * 8 + c] - tbox[t * 8 + 4 + c], tbox[t * 8 + c] - kbox[k * 8 + 4 + c]));
    r2 += g * g;
  }
  // a block holding a diagonal entry of its rows: bounded by the diagonal a^2 + jitter
  const int64_t r_lo = row0 + t * OZ_BM, r_hi = row0 + min64(rows, (t + 1) * OZ_BM), c_lo = k * OZ_BK, c_hi = c_lo + OZ_BK;
  const double kmax = (r_lo < c_hi && c_lo < r_hi) ? kp.diag : kernel_value_f64(kp, r2 * (1.0 - 1e-12));
  const double km = kmax * scl * (1.0 + 1e-9);   // >= |rint(x 2^24)| of every entry of the block
  keep[e] = km < 0.49 ? 0 : (km < 126.5 ? 1 : (km < 32638.0 ? 2 : 3));
}

__global__ void oz_fill_kernel(int64_t rows, double v, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) out[i] = v;
}

// row c = blockIdx.y (grid-stride over m), columns grid-stride over x; pairs of doubles when the
// rows and the output pitch allow 16-byte accesses
__global__ void oz_split_reduce_kernel(const double* __restrict__ part, int splits, int64_t stride, int64_t m,
                                       int64_t rows, double* __restrict__ out, int64_t ldo) {
  const bool v2 = (rows % 2 == 0) && (ldo % 2 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) &&
                  ((reinterpret_cast<uintptr_t>(part) & 15) == 0) && (stride % 2 == 0);
  for (int64_t c = blockIdx.y; c < m; c += gridDim.y) {
    const double* pc = part + c * rows;
    double* oc = out + c * ldo;
    if (v2) {
      for (int64_t r = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); r < rows;
           r += 2 * (int64_t)gridDim.x * blockDim.x) {
        double2 s = make_double2(0.0, 0.0);
        for (int k = 0; k < splits; ++k) {
          const double2 v = *reinterpret_cast<const double2*>(pc + k * stride + r);
          s.x += v.x;
          s.y += v.y;
        }
        *reinterpret_cast<double2*>(oc + r) = s;
      }
    } else {
      for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < splits; ++k) s += pc[k * stride + r];
        oc[r] = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// SA K digits against SB V digits (float64: 7 x 7; float32 K: 3 x 4), pairs s + t <= nd - 1 <= SB - 1.
// k-steps whose kept K slices are all zero (lz >= min(SA, nd)) are left out by the producer and the
// MMA thread alike (same metadata, same sequence of kept steps): no load, no handshake.
template <int SA, int SB, int BN>
__global__ void __launch_bounds__(OZ_THREADS, 1)
ozaki_kv_kernel(const int8_t* __restrict__ Aq, const int8_t* __restrict__ Bq, int64_t KS,
                const double* __restrict__ sigma, const double* __restrict__ tau, int64_t rows, int64_t m, int64_t n,
                int64_t kchunk, double* __restrict__ out, int64_t ldo, int64_t split_stride, int nd,
                const int* __restrict__ knz, int probe, const uint32_t* __restrict__ koff) {
  using C = OzCfg<SA, SB, BN>;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accfull = empty + C::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col0 = (int64_t)blockIdx.x * BN;
  const int64_t row0 = (int64_t)blockIdx.y * OZ_BM;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min64(n, kbeg + kchunk);
  const int steps = (int)ceil_div(max64(kend - kbeg, 0), OZ_BK);
  const int na = nd < SA ? nd : SA;   // K slices that take part

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accfull, 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  {
    // blocks skip their leading all-zero K slices, so a diagonal's first MMA can come at any k-step
    // (and the MMAs of a step are issued smallest first): the accumulators start from zero and every
    // MMA accumulates
    if (warp >= 4) {
      const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
      uint32_t z[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) z[e] = 0u;
#pragma unroll 1
      for (int c = 0; c < (int)C::ACC_COLS; c += 32) ptx::tmem_st_32x32b_x32(tmem + lb + (uint32_t)c, z);
      ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  }
  // leading all-zero K slices of the k-th block of this CTA's range (0 without the metadata), staged
  // in shared memory: the producer and the MMA thread walk it step by step (a global read per step
  // would put an L2 latency on each of their iterations)
  // The k-steps with a kept K slice are compacted into a list (warp 3) that both walk: fully skipped
  // steps cost nothing.  Sparse image (koff, float32 K): the slice offset of every block as well.
  __shared__ uint8_t s_lead[C::KMAX / OZ_BK];
  __shared__ uint16_t s_kept[C::KMAX / OZ_BK];
  __shared__ uint32_t s_off[SA == OZ_S ? 1 : C::KMAX / OZ_BK];
  __shared__ int s_cnt;
  const int* kb_nz = knz ? knz + (int64_t)blockIdx.y * KS + kbeg / OZ_BK : nullptr;
  for (int i = threadIdx.x; i < steps; i += OZ_THREADS) {
    s_lead[i] = kb_nz ? (uint8_t)(SA - kb_nz[i]) : (uint8_t)0;
    if (SA != OZ_S && koff) s_off[i] = koff[(int64_t)blockIdx.y * KS + kbeg / OZ_BK + i];
  }
  __syncthreads();
  if (warp == 3) {
    int cnt = 0;
    for (int b0 = 0; b0 < steps; b0 += 32) {
      const int i = b0 + lane;
      const bool kp_ = i < steps && (int)s_lead[i] < na;
      const unsigned mk = __ballot_sync(0xffffffffu, kp_);
      if (kp_) s_kept[cnt + __popc(mk & ((1u << lane) - 1u))] = (uint16_t)i;
      cnt += __popc(mk);
    }
    if (lane == 0) s_cnt = cnt;
  }
  __syncthreads();
  const int kept = s_cnt;

  if (warp == 0) {   // ---- producer: one bulk copy of the A image and one of the B image per kept k-step
    if (ptx::elect_one()) {
      const int8_t* ga = Aq + ((int64_t)blockIdx.y * KS + kbeg / OZ_BK) * C::A_BYTES;
      const int8_t* gb = Bq + ((int64_t)blockIdx.x * KS + kbeg / OZ_BK) * C::B_BYTES;
      // K slices lz .. na-1 (lz leading all-zero slices skipped) and V slices 0 .. nd-1-lz take part:
      // contiguous ranges of the k-step image
      const int groups = (kept + C::GROUP - 1) / C::GROUP;
      for (int g = 0; g < groups; ++g) {
        const int st = g % C::STAGES;
        if (g >= C::STAGES) ptx::mbar_wait(&empty[st], ((g / C::STAGES) - 1) & 1);
        if (probe == 2) {   // RLD_OZ_PROBE=2 (measurement only): no loads, the MMAs read stale stages
          ptx::mbar_arrive(&full[st]);
          continue;
        }
        uint32_t bytes = 0;
#pragma unroll
        for (int j = 0; j < C::GROUP; ++j) {
          const int it = g * C::GROUP + j;
          if (it >= kept) break;
          const int lz = s_lead[s_kept[it]];
          const int nbv = (nd - lz) < SB ? (nd - lz) : SB;
          bytes += (uint32_t)(na - lz) * OZ_A_SLICE + (uint32_t)nbv * C::B_SLICE;
        }
        ptx::mbar_arrive_expect_tx(&full[st], bytes);
#pragma unroll
        for (int j = 0; j < C::GROUP; ++j) {
          const int it = g * C::GROUP + j;
          if (it >= kept) break;
          const int s = s_kept[it];
          const int lz = s_lead[s];
          unsigned char* dst = smem + st * C::STAGE + j * C::STEP;
          const int nbv = (nd - lz) < SB ? (nd - lz) : SB;
          const uint32_t abytes = (uint32_t)(na - lz) * OZ_A_SLICE, bbytes = (uint32_t)nbv * C::B_SLICE;
          const int8_t* asrc = (SA != OZ_S && koff) ? Aq + (int64_t)s_off[s] * OZ_A_SLICE   // the kept suffix
                                                    : ga + (int64_t)s * C::A_BYTES + lz * OZ_A_SLICE;
          bulk_load(dst + lz * OZ_A_SLICE, asrc, abytes, &full[st]);
          bulk_load(dst + C::A_BYTES, gb + (int64_t)s * C::B_BYTES, bbytes, &full[st]);
        }
      }
    }
  } else if (warp == 1) {   // ---- MMA issuer
    if (ptx::elect_one()) {
      const uint32_t sbase = ptx::smem_u32(smem);
      const int groups = (kept + C::GROUP - 1) / C::GROUP;
      for (int g = 0; g < groups; ++g) {
        const int st = g % C::STAGES;
        ptx::mbar_wait(&full[st], (uint32_t)((g / C::STAGES) & 1));
#pragma unroll
        for (int j = 0; j < C::GROUP; ++j) {
        const int it = g * C::GROUP + j;
        if (it >= kept) break;
        const int lz = s_lead[s_kept[it]];
        const uint32_t a0 = sbase + st * C::STAGE + j * C::STEP;
        const uint32_t b0 = a0 + C::A_BYTES;
        // A slice sa against the stacked B slices 0 .. nd-1-sa at once: the accumulators of the
        // diagonals d = sa + t are adjacent TMEM column blocks, so one N = 64 (nd - sa) product
        // (in N <= 256 pieces; 5 slices as 3 + 2, not 4 + 1: an N = 64 MMA is bound by its A read)
        // covers the whole row of pairs -- 10 MMAs per k-step instead of 28 N = 64 ones (float64).
        // Last slice first: the widest MMAs (sa = lz: N up to 448) go out last, so the tensor pipe
        // still has ~250 cycles queued while this thread commits and waits for the next stage (the
        // pipe accepts only a couple of MMAs ahead: with the narrow ones last it ran dry every step).
#pragma unroll
        for (int sa = SA - 1; sa >= 0; --sa) {
          if (sa >= na || sa < lz || probe == 1) continue;   // RLD_OZ_PROBE=1 (measurement only): loads, no MMAs
          const uint64_t adesc = desc_sw32(a0 + sa * OZ_A_SLICE);
          constexpr uint32_t acc = 1u;
          const int cnt = (nd - sa) < SB ? (nd - sa) : SB;   // B slices 0 .. cnt-1, in at most two pieces
          const int first = (C::PC == 4 && cnt == 5) ? 3 : (cnt < C::PC ? cnt : C::PC);
          mma_i8_ss(tmem + (uint32_t)(sa * BN), adesc, desc_sw32(b0), idesc_i8(OZ_BM, first * BN), acc);
          if (cnt > first)
            mma_i8_ss(tmem + (uint32_t)((sa + first) * BN), adesc, desc_sw32(b0 + first * C::B_SLICE),
                      idesc_i8(OZ_BM, (cnt - first) * BN), acc);
        }
        }
        ptx::tc_commit(&empty[st]);   // the stage is free once these MMAs have read it
      }
      ptx::tc_commit(accfull);        // (no MMA pending: arrives at once)
    }
  } else if (warp >= 4) {   // ---- drains: thread = row (TMEM lane); one drain (k range <= OZ_KMAX)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int64_t r = row0 + row;
    double* o = out + (int64_t)blockIdx.z * split_stride;
    ptx::mbar_wait_sleep(accfull, 0);
    ptx::tc_fence_after();
    const double sg = (r < rows) ? sigma[r] : 0.0;
    const bool have = true;   // the accumulators are zeroed up front
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      double part[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) part[e] = 0.0;
      if (have) {
#pragma unroll 1
        for (int d = nd - 1; d >= 0; --d) {   // small terms first
          const double w = __longlong_as_double((long long)(1023 - OZ_DBITS * (d + 2)) << 52);   // 2^{-8(d+2)}
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(d * BN + c0), v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) part[e] = fma(w, (double)(int32_t)v[e], part[e]);
        }
      }
      if (r < rows) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int64_t cc = col0 + c0 + e;
          if (cc < m) o[cc * ldo + r] = part[e] * sg * tau[cc];
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
}

int oz_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    RLD_CUDA(cudaGetDevice(&dev));
    RLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

}  // namespace

int64_t ozaki_bytes(int64_t rows, int64_t n, int tile_rows, int slices) {
  return ceil_div(rows, tile_rows) * tile_rows * ceil_div(n, OZ_BK) * OZ_BK * slices;
}

// float32 stored K from Morton-ordered points as 3 int8 slices (RLD_FP32_PRODUCT=tf32 keeps the fp32
// tiles and the 3xTF32 / fp16 kernels); read at every prepare
bool fp32_product_slices() {
  const char* e = getenv("RLD_FP32_PRODUCT");
  return !(e && std::string(e) == "tf32");
}

// Read at every prepare, so a process can compare both products.  Default: the int8 slices.
bool fp64_product_ozaki() {
  const char* e = getenv("RLD_FP64_PRODUCT");
  return !(e && std::string(e) == "dmma");
}

void ozaki_slice(const double* A, int64_t lda, int64_t rows, int64_t n, int tile_rows, int8_t* q, double* scale,
                 cudaStream_t st, int slices) {
  if (rows <= 0) return;
  if (rows > 2147483647LL) fail(RLD_ERR_NOT_SUPPORTED, "ozaki_slice: too many rows");
  if (rows <= 65535) {
    RLD_CUDA(cudaMemsetAsync(scale, 0, sizeof(double) * rows, st));
    ozaki_rowmax_kernel<<<dim3((unsigned)rows, (unsigned)ceil_div(std::max<int64_t>(n, 1), OZ_MAX_CHUNK)), 256, 0, st>>>(
        A, lda, n, reinterpret_cast<unsigned long long*>(scale));
    RLD_LAUNCH_CHECK();
    ozaki_scale_finish_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, scale);
  } else {
    ozaki_scale_kernel<<<(unsigned)rows, 256, 0, st>>>(A, lda, n, scale);
  }
  RLD_LAUNCH_CHECK();
  const int64_t KS = ceil_div(n, OZ_BK);
  const int64_t total = ceil_div(rows, tile_rows) * tile_rows * KS * 2;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)oz_sms() * 16);
  if (tile_rows == OZ_BM && slices == OZ_S)
    ozaki_digits_kernel<OZ_BM, OZ_S><<<blocks, 256, 0, st>>>(A, lda, rows, n, scale, KS, q);
  else if (tile_rows == OZ_BN && slices == OZ_S)
    ozaki_digits_kernel<OZ_BN, OZ_S><<<blocks, 256, 0, st>>>(A, lda, rows, n, scale, KS, q);
  else if (tile_rows == OZ_BN && slices == OZ_V32)
    ozaki_digits_kernel<OZ_BN, OZ_V32><<<blocks, 256, 0, st>>>(A, lda, rows, n, scale, KS, q);
  else if (tile_rows == 128 && slices == OZ_V32)
    ozaki_digits_kernel<128, OZ_V32><<<blocks, 256, 0, st>>>(A, lda, rows, n, scale, KS, q);
  else
    fail(RLD_ERR_INVALID_ARGUMENT, "ozaki_slice: tile rows must be 128 (K) or 64 (V), 7 (or, V: 4) slices");
  RLD_LAUNCH_CHECK();
}

// Plan of the sparse 3-slice image of the local rows' float32 K (points X in Morton order, d <= 4):
// keep[block] = slices kept (0..3, a bound from the point boxes), koff[block] = their slice offset
// (exclusive scan).  Returns the number of slices kept in all (bytes = 4096 x that).
int64_t ozaki_sparse_plan(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, int* keep,
                          uint32_t* koff, DevBuf& scratch, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (kp.d > 4) fail(RLD_ERR_NOT_SUPPORTED, "ozaki_sparse_plan: d > 4");
  const int64_t tiles = ceil_div(rows, OZ_BM), KS = ceil_div(n, OZ_BK), nb = tiles * KS;
  scratch.reserve(sizeof(double) * 8 * (tiles + KS));
  double* tb = scratch.as<double>();
  double* kb = tb + 8 * tiles;
  oz_boxes_kernel<<<(unsigned)ceil_div(tiles, 128), 128, 0, st>>>(X, row0, rows, kp.d, OZ_BM, tiles, tb);
  RLD_LAUNCH_CHECK();
  oz_boxes_kernel<<<(unsigned)ceil_div(KS, 128), 128, 0, st>>>(X, 0, n, kp.d, OZ_BK, KS, kb);
  RLD_LAUNCH_CHECK();
  const int ee = oz_scale_exp(kp.diag > 0.0 ? kp.diag : 1.0);   // sigma = 2^(ee+1), as ozaki_slice_points
  const double scl = ldexp(1.0, OZ_DBITS * OZ_S32 - (ee + 1));
  oz_keep_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, st>>>(tb, kb, tiles, KS, kp.d, kp, scl, row0, rows, keep);
  RLD_LAUNCH_CHECK();
  thrust::exclusive_scan(thrust::cuda::par.on(st), keep, keep + nb, koff, 0u);
  uint32_t last_off = 0;
  int last_keep = 0;
  RLD_CUDA(cudaMemcpyAsync(&last_off, koff + nb - 1, sizeof last_off, cudaMemcpyDeviceToHost, st));
  RLD_CUDA(cudaMemcpyAsync(&last_keep, keep + nb - 1, sizeof last_keep, cudaMemcpyDeviceToHost, st));
  RLD_CUDA(cudaStreamSynchronize(st));
  return (int64_t)last_off + last_keep;
}

void ozaki_slice_points(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, int8_t* q,
                        double* scale, cudaStream_t st, int8_t* Kr, int* knz, int slices, const uint32_t* koff) {
  if (rows <= 0) return;
  if (kp.d > RLD_MAX_DIM) fail(RLD_ERR_NOT_SUPPORTED, "ozaki_slice_points: d > 32");
  const int ee = oz_scale_exp(kp.diag > 0.0 ? kp.diag : 1.0);
  oz_fill_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, ldexp(1.0, ee + 1), scale);
  RLD_LAUNCH_CHECK();
  const int64_t KS = ceil_div(n, OZ_BK);
  const int64_t total = ceil_div(rows, OZ_BM) * OZ_BM * KS * 4;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)oz_sms() * 16);
  if (koff && (slices != OZ_S32 || !knz)) fail(RLD_ERR_INVALID_ARGUMENT, "ozaki_slice_points: sparse image needs 3 slices and its plan");
  if (knz && !koff) RLD_CUDA(cudaMemsetAsync(knz, 0, sizeof(int) * ceil_div(rows, OZ_BM) * KS, st));
  if (slices == OZ_S32) {   // float32 K: 24 bits of the float64 kernel value relative to the row scale
    if (Kr || kp.d > 4) fail(RLD_ERR_INVALID_ARGUMENT, "ozaki_slice_points: 3 slices need d <= 4 and no CRT image");
    ozaki_points_kernel<false, 8, 4, OZ_S32><<<blocks, 256, 0, st>>>(X, n, kp, row0, rows, KS, q, nullptr, knz, koff);
  } else if (slices != OZ_S)
    fail(RLD_ERR_INVALID_ARGUMENT, "ozaki_slice_points: 7 or 3 slices");
  else if (Kr && kp.d <= 4)
    ozaki_points_kernel<true, 8, 4, OZ_S><<<blocks, 256, 0, st>>>(X, n, kp, row0, rows, KS, q, Kr, knz, nullptr);
  else if (Kr)
    ozaki_points_kernel<true, 8, RLD_MAX_DIM, OZ_S><<<blocks, 256, 0, st>>>(X, n, kp, row0, rows, KS, q, Kr, knz, nullptr);
  else if (kp.d <= 4)
    ozaki_points_kernel<false, 8, 4, OZ_S><<<blocks, 256, 0, st>>>(X, n, kp, row0, rows, KS, q, nullptr, knz, nullptr);
  else
    ozaki_points_kernel<false, 8, RLD_MAX_DIM, OZ_S><<<blocks, 256, 0, st>>>(X, n, kp, row0, rows, KS, q, nullptr, knz,
                                                                             nullptr);
  RLD_LAUNCH_CHECK();
}

namespace {

template <int SA, int SB, int BN>
void launch_product(const int8_t* Kq, const double* ksigma, int64_t rows, int64_t n, const double* V, int64_t ldv,
                    int64_t m, double* Y, int64_t ldy, KvWorkspace& ws, cudaStream_t st, int diags, const int* knz,
                    const uint32_t* koff) {
  using C = OzCfg<SA, SB, BN>;
  if (diags < 1 || diags > SB) fail(RLD_ERR_INVALID_ARGUMENT, "kv_product_ozaki: diagonals out of range");
  const int64_t KS = ceil_div(n, OZ_BK);
  const int64_t passes = ceil_div(m, BN), tiles = ceil_div(rows, OZ_BM);
  {
    // the float64 partials of the k splits (>= n / KMAX of them) take splits x m x rows x 8 bytes:
    // beyond 20 GB (wide products at n >= 2^19) the vectors go through in groups of whole passes
    const int64_t s0 = ceil_div(n, C::KMAX);
    const int64_t per_pass = s0 > 1 ? s0 * BN * rows * (int64_t)sizeof(double) : 0;
    const char* ce = getenv("RLD_OZ_PARTIAL_MB");   // (tests: a small cap exercises the grouping)
    const int64_t cap = ce ? (int64_t)atol(ce) << 20 : (int64_t)20 << 30;
    const int64_t fit = per_pass > 0 ? std::max<int64_t>(1, cap / per_pass) : passes;
    if (passes > fit) {
      for (int64_t p0 = 0; p0 < passes; p0 += fit) {
        const int64_t c0 = p0 * BN, mc = std::min<int64_t>(m - c0, fit * BN);
        launch_product<SA, SB, BN>(Kq, ksigma, rows, n, V + c0 * ldv, ldv, mc, Y + c0 * ldy, ldy, ws, st, diags, knz, koff);
      }
      return;
    }
  }
  ws.oz_vq.reserve((size_t)ozaki_bytes(m, n, BN, SB));
  ws.oz_tau.reserve(sizeof(double) * m);
  ozaki_slice(V, ldv, m, n, BN, ws.oz_vq.as<int8_t>(), ws.oz_tau.as<double>(), st, SB);
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(ozaki_kv_kernel<SA, SB, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  const int64_t units0 = passes * tiles;
  const int64_t slots = oz_sms();
  // k splits: every CTA <= OZ_KMAX columns (exact int32), >= 64 k-steps; the fewest splits whose
  // CTA count fills >= 95 % of whole waves
  const int64_t min_s = ceil_div(n, C::KMAX);
  // (more splits than the range needs only while their partials stay under 8 GB)
  const int64_t mem_s = std::max<int64_t>(min_s, ((int64_t)8 << 30) / std::max<int64_t>(1, m * rows * (int64_t)sizeof(double)));
  const int64_t max_s = std::min(mem_s, std::max<int64_t>(min_s, n / (OZ_BK * 64)));
  int64_t splits = min_s;
  double best = 0.0;
  for (int64_t s = min_s; s <= std::min<int64_t>(max_s, min_s + 64); ++s) {
    const int64_t u = units0 * s, waves = ceil_div(u, slots);
    const double eff = (double)u / (double)(waves * slots);
    if (eff > best + 1e-9) {
      best = eff;
      splits = s;
    }
    if (eff >= 0.95 && waves >= 2) break;
  }
  const int64_t kchunk = ceil_div(ceil_div(n, splits), OZ_BK) * OZ_BK;
  splits = ceil_div(n, kchunk);
  dim3 grid((unsigned)passes, (unsigned)tiles, (unsigned)splits);
  if (grid.y > 65535u || grid.z > 65535u) fail(RLD_ERR_NOT_SUPPORTED, "kv_product_ozaki: grid too large");
  const int8_t* Bq = ws.oz_vq.as<int8_t>();
  const char* pe = getenv("RLD_OZ_PROBE");   // kernel-phase probe for measurement, never set in production
  const int probe = pe ? atoi(pe) : 0;
  if (splits == 1) {
    ozaki_kv_kernel<SA, SB, BN><<<grid, OZ_THREADS, C::SMEM, st>>>(Kq, Bq, KS, ksigma, ws.oz_tau.as<double>(), rows, m, n,
                                                              kchunk, Y, ldy, 0, diags, knz, probe, koff);
    RLD_LAUNCH_CHECK();
    return;
  }
  const int64_t stride = m * rows;
  ws.partial.reserve(sizeof(double) * stride * splits);
  ozaki_kv_kernel<SA, SB, BN><<<grid, OZ_THREADS, C::SMEM, st>>>(Kq, Bq, KS, ksigma, ws.oz_tau.as<double>(), rows, m, n,
                                                            kchunk, ws.partial.as<double>(), rows, stride, diags, knz,
                                                            probe, koff);
  RLD_LAUNCH_CHECK();
  const unsigned gy = (unsigned)std::min<int64_t>(m, 65535);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 512), slots * 8 / gy + 1));
  oz_split_reduce_kernel<<<dim3(gx, gy), 256, 0, st>>>(ws.partial.as<double>(), (int)splits, stride, m, rows, Y, ldy);
  RLD_LAUNCH_CHECK();
}

}  // namespace

// Y (m x rows, ld ldy) = V K^T with K given by its sliced image Kq (ozaki_slice, 128-row tiles, kslices =
// 7: float64, 3: float32 K) and row scales; V (m x n float64 rows, ld ldv) is sliced here (64-vector
// tiles, 7 or 4 slices) into ws.oz_vq.  diags <= 0: all of them.
void kv_product_ozaki(const int8_t* Kq, const double* ksigma, int64_t rows, int64_t n, const double* V, int64_t ldv,
                      int64_t m, double* Y, int64_t ldy, KvWorkspace& ws, cudaStream_t st, int diags,
                      const int* knz, int kslices, const uint32_t* koff) {
  if (m <= 0 || rows <= 0) return;
  if (koff && (kslices != OZ_S32 || !knz)) fail(RLD_ERR_INVALID_ARGUMENT, "kv_product_ozaki: sparse image needs 3 slices");
  if (kslices == OZ_S)
    launch_product<OZ_S, OZ_S, OZ_BN>(Kq, ksigma, rows, n, V, ldv, m, Y, ldy, ws, st, diags <= 0 ? OZ_S : diags, knz, nullptr);
  else if (kslices == OZ_S32 && m <= 96)
    launch_product<OZ_S32, OZ_V32, OZ_BN>(Kq, ksigma, rows, n, V, ldv, m, Y, ldy, ws, st, OZ_V32, knz, koff);
  else if (kslices == OZ_S32)   // wide products: 128 vectors per pass
    launch_product<OZ_S32, OZ_V32, 128>(Kq, ksigma, rows, n, V, ldv, m, Y, ldy, ws, st, OZ_V32, knz, koff);
  else
    fail(RLD_ERR_INVALID_ARGUMENT, "kv_product_ozaki: 7 or 3 K slices");
}

}  // namespace rld
