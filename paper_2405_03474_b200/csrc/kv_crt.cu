// Float64-accurate wide K x V (the sketch products, src/precond.py:186, 189) as L exact int8
// MODULAR products on the INT8 tensor cores and a Chinese-remainder reconstruction ("Ozaki scheme
// II").  For the sketch's m = l + 10 vectors this needs 15 int8 GEMMs where the slice product of
// kv_ozaki.cu needs 36 slice pairs, at the same float64 accuracy.
//
// Integers (exact):
//   K'_ij = sum_{s<6} d_s[i,j] 256^{5-s}  from the first 6 of K's exact int8 slices (kv_ozaki.cu),
//           K_ij = sigma_i 2^-48 (K'_ij + rho_ij), |rho| <= 1/2, |K'| < 2^47;
//   V'_cj = rint(2^{e_c} V_cj), e_c = bV - 1 - ilogb(max_j |V_cj|), |V'| < 2^bV;
//   C'_ic = sum_j K'_ij V'_cj, |C'| < n 2^{48.02 + bV} < P / 2 (bV chosen so; 52 at n = 65536),
//   P = prod of the L = 15 pairwise coprime moduli p_l <= 256 (2^117.8).
// Modular products: residues r_l(K') and r_l(V') in [-128, 127] (int8), C_l = r_l(K') r_l(V')^T
//   accumulated exactly in int32 (n 2^14 < 2^31 for n < 2^17), reduced mod p_l.
// Reconstruction (per output, float64 double-double): y_l = C_l u_l mod p_l with
//   u_l = (P / p_l)^-1 mod p_l, S = sum_l y_l / p_l, C' = P (S - round(S)) (the representative of
//   C' mod P in (-P/2, P/2]), Y_ic = C' sigma_i 2^-48 2^-e_c.  S is formed with 1 / p_l and P as
//   double-double (~2^-100), so C' carries < 2^21 absolute error against |C'| up to 2^116.
// Error against the exact product: the dropped remainders rho (2^-50 sigma_i per entry) and V's
//   rounding (2^-bV max |V_c|): the float64 level of kv_ozaki.cu.
//
// Residue images (k-step-tiled, pre-swizzled like the slice image so a stage is one bulk copy):
//   K: [tile][l][ks][128][32] bytes, built once per prepare from the slice image (15 bytes per
//   entry); V: [l][pass][ks][NT][32] per product.
// GEMM kernel: grid (pass, row tile, modulus), modulus slowest so the wave shares one modulus's V
//   residues in L2 and the passes of a tile share its K residues; one CTA per SM, warp 0 bulk-copies
//   KB = 4 k-steps of A (4 KB each) and B (NT x 32 B each) per stage into a 5-stage ring, warp 1
//   issues one tcgen05.mma.kind::i8 (M = 128, N = NT, K = 32) per k-step into one int32 TMEM
//   accumulator, warps 4-7 reduce it mod p_l and store uint8 residues.
#include <cuda.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <string>

#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "tc_ptx.cuh"
#include "crt_common.cuh"

namespace rld {

namespace {

constexpr int CRT_BM = 128, CRT_BK = 32;
constexpr int CRT_KB = 4;           // k-steps per stage
constexpr int CRT_THREADS = 256;
constexpr int CRT_KBITS_X100 = 4700;   // log2 max|K'| * 100 (|x| <= 63/128: |K'| <= 2^46.98 + 1/2)
struct CrtConst {
  int coef[CRT_SLICES][CRT_L];   // 256^{5-s} mod p_l
  int u[CRT_L];                  // (P / p_l)^-1 mod p_l
  double inv_hi[CRT_L], inv_lo[CRT_L];   // 1 / p_l as double-double
  double P_hi, P_lo;             // P as double-double
  double log2P;
};

CrtConst make_consts() {
  CrtConst c{};
  for (int l = 0; l < CRT_L; ++l) {
    const long long p = crt_mod(l);
    long long w = 1;
    for (int s = CRT_SLICES - 1; s >= 0; --s) {   // coef[s] = 256^{5-s} mod p
      c.coef[s][l] = (int)w;
      w = (w * 256) % p;
    }
    long long Ml = 1;   // prod_{k != l} p_k mod p_l
    for (int k = 0; k < CRT_L; ++k)
      if (k != l) Ml = (Ml * crt_mod(k)) % p;
    long long t0 = 0, t1 = 1, r0 = p, r1 = Ml;   // extended Euclid: inverse of Ml mod p
    while (r1 != 0) {
      const long long q = r0 / r1;
      long long tmp = t0 - q * t1; t0 = t1; t1 = tmp;
      tmp = r0 - q * r1; r0 = r1; r1 = tmp;
    }
    if (r0 != 1) fail(RLD_ERR_CUDA, "kv_crt: moduli not coprime");
    c.u[l] = (int)((t0 % p + p) % p);
    c.inv_hi[l] = 1.0 / (double)p;
    c.inv_lo[l] = std::fma(-c.inv_hi[l], (double)p, 1.0) / (double)p;
  }
  unsigned __int128 P = 1;
  double lg = 0.0;
  for (int l = 0; l < CRT_L; ++l) {
    P *= (unsigned)crt_mod(l);
    lg += std::log2((double)crt_mod(l));
  }
  c.P_hi = (double)P;
  const unsigned __int128 ph = (unsigned __int128)c.P_hi;
  c.P_lo = P >= ph ? (double)(P - ph) : -(double)(ph - P);
  c.log2P = lg;
  return c;
}

const CrtConst& consts() {
  static const CrtConst c = make_consts();
  return c;
}

__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;   // SWIZZLE_32B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// physical byte of element (row, col) in a [R][32]-byte tile with the 32-byte swizzle
__host__ __device__ __forceinline__ uint32_t swz32(uint32_t row, uint32_t col) {
  const uint32_t o = row * 32u + col;
  return o ^ (((o >> 7) & 1u) << 4);
}

// ---------------------------------------------------------------- K residues from the slice image
// Slice image: ((t KS + ks) 7 + s) 4096 + phys; residue image: ((t L + l) KS + ks) 4096 + phys (the
// same swizzled position).  Thread = 16 bytes of one (tile, k-step).
__global__ void crt_k_residues(const int8_t* __restrict__ Kq, int64_t tiles, int64_t KS, CrtConst c,
                               int8_t* __restrict__ Kr) {
  const int64_t total = tiles * KS * 256;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t chunk = e & 255;
    const int64_t tk = e >> 8;   // t KS + ks
    const int64_t t = tk / KS, ks = tk - t * KS;
    alignas(16) int8_t d[CRT_SLICES][16];
#pragma unroll
    for (int s = 0; s < CRT_SLICES; ++s)
      *reinterpret_cast<uint4*>(d[s]) = *reinterpret_cast<const uint4*>(Kq + (tk * OZ_NSLICES + s) * 4096 + chunk * 16);
#pragma unroll
    for (int l = 0; l < CRT_L; ++l) {
      const int p = crt_mod(l);
      alignas(16) int8_t o[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        int acc = 0;
#pragma unroll
        for (int s = 0; s < CRT_SLICES; ++s) acc += (int)d[s][b] * c.coef[s][l];
        o[b] = (int8_t)sym_mod(acc, p);
      }
      *reinterpret_cast<uint4*>(Kr + ((t * CRT_L + l) * KS + ks) * 4096 + chunk * 16) = *reinterpret_cast<uint4*>(o);
    }
  }
}

// max |V_c| per vector (bit pattern of a non-negative double, ordered like the value)
__global__ void crt_vmax(const double* __restrict__ V, int64_t ldv, int64_t n, unsigned long long* __restrict__ vmax) {
  const int64_t c = blockIdx.y;
  double mx = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fabs(V[c * ldv + j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(vmax + c, (unsigned long long)__double_as_longlong(mx));
}

__device__ __forceinline__ int v_exponent(unsigned long long bits, int bV) {
  const double mx = __longlong_as_double((long long)bits);
  return mx > 0.0 ? bV - 1 - ilogb(mx) : 0;
}

// V residues: thread = (padded vector c, 16 consecutive columns j0..j0+15), one 16-byte store per
// modulus (a 16-byte half-row stays contiguous under the 32-byte swizzle); image
// [l][pass][ks][NT][32]
__global__ void crt_v_residues(const double* __restrict__ V, int64_t ldv, int64_t m, int64_t n, int64_t KS, int NT,
                               int passes, int bV, const unsigned long long* __restrict__ vmax,
                               int8_t* __restrict__ Vr) {
  const int64_t c = blockIdx.y;
  const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
  if (j0 >= KS * CRT_BK) return;
  double v[16];
  const int ev = c < m ? v_exponent(vmax[c], bV) : 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int64_t j = j0 + k;
    v[k] = (c < m && j < n) ? rint(ldexp(V[c * ldv + j], ev)) : 0.0;   // exact integer, |v| < 2^bV
  }
  const int pass = (int)(c / NT), row = (int)(c - (int64_t)pass * NT);
  const int64_t ks = j0 >> 5;
  const uint32_t phys = swz32((uint32_t)row, (uint32_t)(j0 & 31));
  const int64_t tile_bytes = (int64_t)NT * CRT_BK;
#pragma unroll
  for (int l = 0; l < CRT_L; ++l) {
    const int p = crt_mod(l);
    const double pinv = 1.0 / (double)p;
    alignas(16) int8_t o[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double q = floor(v[k] * pinv);
      double r = fma(-q, (double)p, v[k]);   // exact; |r| < 2p
      if (r < 0.0) r += p;
      if (r >= p) r -= p;
      int ri = (int)r;
      if (ri > (p - 1) / 2) ri -= p;
      o[k] = (int8_t)ri;
    }
    *reinterpret_cast<uint4*>(Vr + (((int64_t)l * passes + pass) * KS + ks) * tile_bytes + phys) =
        *reinterpret_cast<uint4*>(o);
  }
}

// ---------------------------------------------------------------- modular GEMM
// ring depth: 5 stages, fewer where KB k-steps of A and B would not fit in 227 KB
__host__ __device__ constexpr int crt_stages(int NT) {
  return (232448 - 1280) / (CRT_KB * (CRT_BM * CRT_BK + NT * CRT_BK)) < 5
             ? (232448 - 1280) / (CRT_KB * (CRT_BM * CRT_BK + NT * CRT_BK)) : 5;
}

template <int NT>
__global__ void __launch_bounds__(CRT_THREADS, 1)
crt_gemm_kernel(const int8_t* __restrict__ Kr, const int8_t* __restrict__ Vr, int KS, int passes,
                uint8_t* __restrict__ out, int64_t m_pad, int64_t rows) {
  constexpr uint32_t A_STEP = CRT_BM * CRT_BK, B_STEP = NT * CRT_BK;
  constexpr uint32_t STAGE = CRT_KB * (A_STEP + B_STEP);
  constexpr uint32_t COLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  constexpr int CRT_STAGES = crt_stages(NT);
  extern __shared__ __align__(1024) unsigned char crt_smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(crt_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CRT_STAGES * STAGE);
  uint64_t* empty = full + CRT_STAGES;
  uint64_t* accfull = empty + CRT_STAGES;
  uint32_t* holder = reinterpret_cast<uint32_t*>(accfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pass = blockIdx.x, tile = blockIdx.y, l = blockIdx.z;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CRT_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accfull, 1);
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(holder, COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  const int nst = (int)ceil_div(KS, CRT_KB);
  if (warp == 0) {   // producer: KB k-steps of A and of B per stage (the last stage may be short)
    if (ptx::elect_one()) {
      const int8_t* ga = Kr + ((int64_t)tile * CRT_L + l) * (int64_t)KS * A_STEP;
      const int8_t* gb = Vr + ((int64_t)l * passes + pass) * (int64_t)KS * B_STEP;
      for (int s = 0; s < nst; ++s) {
        const int st = s % CRT_STAGES;
        const int kb = (int)min64(CRT_KB, KS - (int64_t)s * CRT_KB);
        if (s >= CRT_STAGES) ptx::mbar_wait(&empty[st], ((s / CRT_STAGES) - 1) & 1);
        unsigned char* dst = smem + st * STAGE;
        ptx::mbar_arrive_expect_tx(&full[st], (uint32_t)kb * (A_STEP + B_STEP));
        bulk_load(dst, ga + (int64_t)s * CRT_KB * A_STEP, (uint32_t)kb * A_STEP, &full[st]);
        bulk_load(dst + CRT_KB * A_STEP, gb + (int64_t)s * CRT_KB * B_STEP, (uint32_t)kb * B_STEP, &full[st]);
      }
    }
  } else if (warp == 1) {   // MMA issuer
    if (ptx::elect_one()) {
      const uint32_t sbase = ptx::smem_u32(smem);
      for (int s = 0; s < nst; ++s) {
        const int st = s % CRT_STAGES;
        const int kb = (int)min64(CRT_KB, KS - (int64_t)s * CRT_KB);
        ptx::mbar_wait(&full[st], (uint32_t)((s / CRT_STAGES) & 1));
        ptx::tc_fence_after();
        const uint32_t a0 = sbase + st * STAGE, b0 = a0 + CRT_KB * A_STEP;
#pragma unroll
        for (int k = 0; k < CRT_KB; ++k)
          if (k < kb)
            mma_i8_ss(tmem, desc_sw32(a0 + k * A_STEP), desc_sw32(b0 + k * B_STEP), idesc_i8(CRT_BM, NT),
                      (s > 0 || k > 0) ? 1u : 0u);
        ptx::tc_commit(&empty[st]);
      }
      ptx::tc_commit(accfull);
    }
  } else if (warp >= 4) {   // drain: int32 accumulator mod p_l -> uint8 residue in [0, p)
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    ptx::mbar_wait_sleep(accfull, 0);
    ptx::tc_fence_after();
    const int p = crt_mod(l);
    const int64_t r = (int64_t)tile * CRT_BM + row;
    uint8_t* o = out + ((int64_t)l * m_pad + (int64_t)pass * NT) * rows + r;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 16) {
      uint32_t v[16];
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + (uint32_t)c0, v);
      ptx::tmem_wait_ld();
      if (r < rows) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int x = (int)v[e] % p;
          if (x < 0) x += p;
          o[(int64_t)(c0 + e) * rows] = (uint8_t)x;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, COLS);
}

// ---------------------------------------------------------------- reconstruction
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// Y[c ldy + i] = C'_ic sigma_i 2^-48 2^-e_c from the L residues of C'_ic
__global__ void crt_reconstruct(const uint8_t* __restrict__ res, int64_t m, int64_t m_pad, int64_t rows, CrtConst c,
                                int bV, const unsigned long long* __restrict__ vmax, const double* __restrict__ sigma,
                                double* __restrict__ Y, int64_t ldy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t col = blockIdx.y;
  if (i >= rows || col >= m) return;
  double sh = 0.0, sl = 0.0;   // S = sum_l y_l / p_l, double-double
#pragma unroll
  for (int l = 0; l < CRT_L; ++l) {
    const int p = crt_mod(l);
    const int r = res[((int64_t)l * m_pad + col) * rows + i];
    const double y = (double)((r * c.u[l]) % p);   // exact small integer
    const double ph = y * c.inv_hi[l];
    const double pe = fma(y, c.inv_hi[l], -ph) + y * c.inv_lo[l];
    double s, e;
    two_sum(sh, ph, s, e);
    sh = s;
    sl += e + pe;
  }
  double s, e;
  two_sum(sh, sl, s, e);   // renormalise
  const double k = rint(s);
  double fh = s - k, fl = e;   // S - round(S), |.| <= 1/2 (+ rounding)
  two_sum(fh, fl, fh, fl);
  // C' = F P with F and P double-double
  const double ch = fh * c.P_hi;
  const double ce = fma(fh, c.P_hi, -ch) + fh * c.P_lo + fl * c.P_hi;
  const double Cp = ch + ce;
  const double mx = __longlong_as_double((long long)vmax[col]);
  const int ev = mx > 0.0 ? bV - 1 - ilogb(mx) : 0;
  Y[col * ldy + i] = ldexp(Cp * sigma[i], -48 - ev);
}

template <int NT>
void launch_gemm(const int8_t* Kr, const int8_t* Vr, int KS, int passes, int tiles, uint8_t* out, int64_t m_pad,
                 int64_t rows, cudaStream_t st) {
  const size_t smem = (size_t)crt_stages(NT) * CRT_KB * (CRT_BM * CRT_BK + NT * CRT_BK) + 1024 + 256;
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(crt_gemm_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  const dim3 grid((unsigned)passes, (unsigned)tiles, (unsigned)CRT_L);
  crt_gemm_kernel<NT><<<grid, CRT_THREADS, smem, st>>>(Kr, Vr, KS, passes, out, m_pad, rows);
  RLD_LAUNCH_CHECK();
}

void launch_gemm_nt(int NT, const int8_t* Kr, const int8_t* Vr, int KS, int passes, int tiles, uint8_t* out,
                    int64_t m_pad, int64_t rows, cudaStream_t st) {
  switch (NT) {
#define RLD_CRT_NT(X) \
  case X: launch_gemm<X>(Kr, Vr, KS, passes, tiles, out, m_pad, rows, st); break;
    RLD_CRT_NT(96) RLD_CRT_NT(112) RLD_CRT_NT(128) RLD_CRT_NT(144) RLD_CRT_NT(160) RLD_CRT_NT(176) RLD_CRT_NT(192)
    RLD_CRT_NT(208) RLD_CRT_NT(224) RLD_CRT_NT(240) RLD_CRT_NT(256)
#undef RLD_CRT_NT
    default: fail(RLD_ERR_INVALID_ARGUMENT, "kv_crt: unsupported pass width");
  }
}

// bits of V' so that n 2^{47 + bV} < P / 2 (float64-grade needs >= 48), capped at 53
int v_bits(int64_t n) {
  const double b = consts().log2P - 1.0 - CRT_KBITS_X100 / 100.0 - std::log2((double)n);
  return (int)std::min(53.0, std::floor(b - 1e-9));
}

}  // namespace

// CRT products on by default for wide products of a float64 stored K (RLD_FP64_SKETCH=slices: the
// slice product for every width); the residue image needs n < 2^17 (exact int32 sums) and n small
// enough that V' keeps >= 48 bits.
bool crt_supported(int64_t n) {
  const char* e = getenv("RLD_FP64_SKETCH");
  if (e && std::string(e) == "slices") return false;
  return n > 0 && n < (1 << 17) && v_bits(n) >= 48;
}

int64_t crt_bytes(int64_t rows, int64_t n) { return ceil_div(rows, CRT_BM) * (int64_t)CRT_L * ceil_div(n, CRT_BK) * 4096; }

void crt_residues(const int8_t* Kq, int64_t rows, int64_t n, int8_t* Kr, cudaStream_t st) {
  if (rows <= 0) return;
  const int64_t tiles = ceil_div(rows, CRT_BM), KS = ceil_div(n, CRT_BK);
  int dev = 0, sms = 0;
  RLD_CUDA(cudaGetDevice(&dev));
  RLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = (int)std::min<int64_t>(ceil_div(tiles * KS * 256, 256), (int64_t)sms * 16);
  crt_k_residues<<<blocks, 256, 0, st>>>(Kq, tiles, KS, consts(), Kr);
  RLD_LAUNCH_CHECK();
}

void kv_product_crt(const int8_t* Kr, const double* ksigma, int64_t rows, int64_t n, const double* V, int64_t ldv,
                    int64_t m, double* Y, int64_t ldy, KvWorkspace& ws, cudaStream_t st) {
  if (m <= 0 || rows <= 0) return;
  const int bV = v_bits(n);
  if (bV < 48 || n >= (1 << 17)) fail(RLD_ERR_NOT_SUPPORTED, "kv_product_crt: n out of range");
  const int KS = (int)ceil_div(n, CRT_BK);
  const int passes = (int)ceil_div(m, 256);
  const int NT = std::max<int>(96, (int)(ceil_div(ceil_div(m, passes), 16) * 16));
  const int64_t m_pad = (int64_t)passes * NT;
  const int tiles = (int)ceil_div(rows, CRT_BM);
  if (tiles > 65535) fail(RLD_ERR_NOT_SUPPORTED, "kv_product_crt: too many row tiles");
  ws.crt_vmax.reserve(sizeof(unsigned long long) * m_pad);
  unsigned long long* vmax = ws.crt_vmax.as<unsigned long long>();
  RLD_CUDA(cudaMemsetAsync(vmax, 0, sizeof(unsigned long long) * m_pad, st));
  {
    const dim3 g((unsigned)std::min<int64_t>(64, ceil_div(n, 256 * 8)), (unsigned)m);
    crt_vmax<<<g, 256, 0, st>>>(V, ldv, n, vmax);
    RLD_LAUNCH_CHECK();
  }
  ws.crt_vr.reserve((size_t)CRT_L * m_pad * KS * CRT_BK);
  {
    const dim3 g((unsigned)ceil_div((int64_t)KS * CRT_BK / 16, 128), (unsigned)m_pad);
    crt_v_residues<<<g, 128, 0, st>>>(V, ldv, m, n, KS, NT, passes, bV, vmax, ws.crt_vr.as<int8_t>());
    RLD_LAUNCH_CHECK();
  }
  ws.crt_out.reserve((size_t)CRT_L * m_pad * rows);
  launch_gemm_nt(NT, Kr, ws.crt_vr.as<int8_t>(), KS, passes, tiles, ws.crt_out.as<uint8_t>(), m_pad, rows, st);
  const dim3 g((unsigned)ceil_div(rows, 256), (unsigned)m);
  crt_reconstruct<<<g, 256, 0, st>>>(ws.crt_out.as<uint8_t>(), m, m_pad, rows, consts(), bV, vmax, ksigma, Y, ldy);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
