// Device-side helpers shared by the rld kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rld_internal.cuh"

#define RLD_MAX_DIM 32

namespace rld {

// Kernel value from a squared distance (src/kernels.py:40-46), float64.
__device__ __forceinline__ double kernel_value_f64(const KernelParams& kp, double r2) {
  if (kp.family == RLD_RBF) return kp.a2 * exp(-r2 * kp.inv_2l2);
  const double u = sqrt(r2) * kp.s5_over_l;
  return kp.a2 * (1.0 + u + u * u * (1.0 / 3.0)) * exp(-u);
}

// float32 variant for on-the-fly tiles (MUFU ex2/rsqrt on the FP32 pipe).
__device__ __forceinline__ float kernel_value_f32(int family, float a2, float inv_2l2_log2e,
                                                  float s5_over_l, float r2) {
  if (family == RLD_RBF) return a2 * exp2f(-r2 * inv_2l2_log2e);
  const float u = sqrtf(r2) * s5_over_l;
  return a2 * fmaf(u, fmaf(u, 1.0f / 3.0f, 1.0f), 1.0f) * exp2f(-u * 1.4426950408889634f);
}

// ---------------------------------------------------------------------------
// Philox4x64-10 (Salmon et al. 2011) as numpy's bit generator uses it.
struct U64x4 { uint64_t v[4]; };

__device__ __forceinline__ U64x4 philox4x64_10(U64x4 c, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += W0; k1 += W1; }
    const uint64_t lo0 = M0 * c.v[0], hi0 = __umul64hi(M0, c.v[0]);
    const uint64_t lo1 = M1 * c.v[2], hi1 = __umul64hi(M1, c.v[2]);
    U64x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// 64-bit word `q` of a fresh numpy Philox stream: numpy pre-increments the
// 256-bit counter before each block of four words, so block b uses counter b+1.
__device__ __forceinline__ uint64_t philox_word(uint64_t q, uint64_t k0, uint64_t k1) {
  const uint64_t blk = (q >> 2) + 1;
  U64x4 c;
  c.v[0] = blk;
  c.v[1] = (blk == 0) ? 1 : 0;  // carry (only for q >= 2^66, never in practice)
  c.v[2] = 0;
  c.v[3] = 0;
  U64x4 o = philox4x64_10(c, k0, k1);
  return o.v[q & 3];
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum (result valid in thread 0).  `red` has blockDim.x/32 slots.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 0; w < nw; ++w) s += red[w];
  }
  return s;
}

}  // namespace rld
