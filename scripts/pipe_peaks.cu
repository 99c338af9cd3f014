// Whole-GPU pipe peaks on this box ("re-measure FP32, FP64, TF32 and MUFU"):
// FFMA, packed FFMA2 (fma.rn.f32x2), DFMA, MUFU ex2.approx / sqrt.approx, and tcgen05.mma
// kind::tf32 (M = 128, K = 8, N = 64/128/256; A from SMEM "ss" and from TMEM "ts").
// Each test runs on every SM, timed with CUDA events (best of 5 after a warm-up), and prints
// one JSON object.  The SM clock during the run is sampled by the caller (nvidia-smi).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2405_03474_b200/csrc pipe_peaks.cu -o pipe_peaks
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace rld;

constexpr int CHAINS = 8;

__global__ void ffma_kernel(int iters, float seed, float* out) {
  float a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) a[c] = seed + c * 1e-3f + threadIdx.x * 1e-6f;
  const float m = 0.999999f, k = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) a[c] = fmaf(a[c], m, k);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  if (s == 12345.f) out[0] = s;
}

__global__ void ffma2_kernel(int iters, float seed, float* out) {
  uint64_t a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 f = make_float2(seed + c * 1e-3f, seed - threadIdx.x * 1e-6f);
    a[c] = *reinterpret_cast<uint64_t*>(&f);
  }
  float2 mf = make_float2(0.999999f, 0.999998f), kf = make_float2(1e-7f, 2e-7f);
  const uint64_t m = *reinterpret_cast<uint64_t*>(&mf), k = *reinterpret_cast<uint64_t*>(&kf);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[c]) : "l"(m), "l"(k));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 f = *reinterpret_cast<float2*>(&a[c]);
    s += f.x + f.y;
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void dfma_kernel(int iters, double seed, double* out) {
  double a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) a[c] = seed + c * 1e-3 + threadIdx.x * 1e-6;
  const double m = 0.9999999, k = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], m, k);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  if (s == 12345.0) out[0] = s;
}

// FP64 tensor cores: independent chains of mma.sync m8n8k4 f64 (256 FMA each)
__global__ void dmma_kernel(int iters, double seed, double* out) {
  double c[CHAINS][2];
  const double a = seed + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = 1e-3 * k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < CHAINS; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[k][0]), "+d"(c[k][1])
                     : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

template <int OP>   // 0 ex2.approx.ftz, 1 sqrt.approx.ftz
__global__ void mufu_kernel(int iters, float seed, float* out) {
  float a[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) a[c] = seed + c * 1e-3f + threadIdx.x * 1e-6f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (OP == 0)
          asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
        else
          asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
      }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += a[c];
  if (s == 12345.f) out[0] = s;
}

// One issuing thread per CTA, one CTA per SM, back-to-back MMAs into one accumulator.
template <int N, bool TS, bool F16 = false>
__global__ void __launch_bounds__(128) mma_kernel(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t bsm[256 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<float*>(bsm)[i] = 1.0f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbarrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    // kind::f16 (fp16 in, f32 accumulate, K = 16): a_format = b_format = 0
    const uint32_t idesc = F16 ? ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24))
                               : ptx::idesc_tf32(128, N);
    const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(bsm));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS && F16) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256 + 8 * k), "l"(bd + 2 * k), "r"(idesc), "r"(1u)
              : "memory");
        } else if (TS) {
          ptx::mma_tf32_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, 1u);
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(bd + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"(1u)
              : "memory");
        }
      }
    }
    ptx::tc_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

// tcgen05 kind::i8 (s8 x s8 -> s32), M = 128, K = 32, A and B from shared memory (32-byte swizzle
// descriptors as kv_ozaki.cu), N = 64 / 128 / 256
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)6 << 61);
}

// RAND: operands random bytes (the data a real int8-slice / residue product multiplies; constant
// operands draw far less power and never meet the 1 kW cap)
template <int N, bool RAND = false>
__global__ void __launch_bounds__(128) mma_i8_kernel(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t sm[128 * 32 + 256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < (int)sizeof(sm) / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)(i + 1) * 2654435761u ^ (uint32_t)blockIdx.x * 0x9E3779B9u;
    x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12;
    reinterpret_cast<uint32_t*>(sm)[i] = RAND ? x : 0x01010101u;
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbarrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = desc_sw32(ptx::smem_u32(sm)), bd = desc_sw32(ptx::smem_u32(sm + 128 * 32));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)(k & 1) * 256u),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
            : "memory");
    }
    ptx::tc_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

template <typename F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* fo;
  double* dd;
  long long* lo;
  cudaMalloc(&fo, 16);
  cudaMalloc(&dd, 16);
  cudaMalloc(&lo, 16);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double ops = (double)blocks * threads * iters * 16 * CHAINS;   // instructions (per lane)
  printf("{\n \"sms\": %d, \"clock_attr_mhz\": %.0f,\n", sms, clk_khz / 1e3);
  {
    float ms = best_ms([&] { ffma_kernel<<<blocks, threads>>>(iters, 1.0f, fo); });
    printf(" \"ffma_tflops\": %.2f,\n", 2 * ops / (ms * 1e-3) / 1e12);
  }
  {
    float ms = best_ms([&] { ffma2_kernel<<<blocks, threads>>>(iters, 1.0f, fo); });
    printf(" \"ffma2_tflops\": %.2f,\n", 4 * ops / (ms * 1e-3) / 1e12);
  }
  {
    float ms = best_ms([&] { dfma_kernel<<<blocks, threads>>>(iters / 4, 1.0, dd); });
    printf(" \"dfma_tflops\": %.2f,\n", 2 * ops / 4 / (ms * 1e-3) / 1e12);
  }
  {
    // per warp: iters * 4 * CHAINS DMMAs of 8 x 8 x 4 FMAs
    const int dit = iters / 16;
    float ms = best_ms([&] { dmma_kernel<<<blocks, threads>>>(dit, 1.0, dd); });
    const double fl = (double)blocks * (threads / 32) * dit * 4 * CHAINS * 2.0 * 8 * 8 * 4;
    printf(" \"dmma_tflops\": %.2f,\n", fl / (ms * 1e-3) / 1e12);
  }
  {
    float ms = best_ms([&] { mufu_kernel<0><<<blocks, threads>>>(iters / 4, 0.5f, fo); });
    printf(" \"mufu_ex2_gops\": %.1f,\n", ops / 4 / (ms * 1e-3) / 1e9);
  }
  {
    float ms = best_ms([&] { mufu_kernel<1><<<blocks, threads>>>(iters / 4, 0.5f, fo); });
    printf(" \"mufu_sqrt_gops\": %.1f,\n", ops / 4 / (ms * 1e-3) / 1e9);
  }
  const int mi = 20000;
  auto mma = [&](auto kern, int N, const char* name, bool last) {
    float ms = best_ms([&] { kern<<<sms, 128>>>(mi, lo); });
    long long cyc = 0;
    cudaMemcpy(&cyc, lo, 8, cudaMemcpyDeviceToHost);
    const double fl = (double)sms * mi * 4 * 2.0 * 128 * N * 8;
    printf(" \"%s\": {\"tflops\": %.1f, \"cycles_per_mma\": %.1f}%s\n", name, fl / (ms * 1e-3) / 1e12,
           (double)cyc / (mi * 4.0), last ? "" : ",");
  };
  mma(mma_kernel<64, false>, 64, "tf32_ss_n64", false);
  mma(mma_kernel<128, false>, 128, "tf32_ss_n128", false);
  mma(mma_kernel<256, false>, 256, "tf32_ss_n256", false);
  mma(mma_kernel<64, true>, 64, "tf32_ts_n64", false);
  mma(mma_kernel<128, true>, 128, "tf32_ts_n128", false);
  mma(mma_kernel<256, true>, 256, "tf32_ts_n256", false);
  auto mmah = [&](auto kern, int N, const char* name) {   // kind::f16: K = 16 per MMA
    float ms = best_ms([&] { kern<<<sms, 128>>>(mi, lo); });
    long long cyc = 0;
    cudaMemcpy(&cyc, lo, 8, cudaMemcpyDeviceToHost);
    const double fl = (double)sms * mi * 4 * 2.0 * 128 * N * 16;
    printf(" \"%s\": {\"tflops\": %.1f, \"cycles_per_mma\": %.1f},\n", name, fl / (ms * 1e-3) / 1e12,
           (double)cyc / (mi * 4.0));
  };
  mmah(mma_kernel<64, true, true>, 64, "f16_ts_n64");
  mmah(mma_kernel<128, true, true>, 128, "f16_ts_n128");
  mmah(mma_kernel<256, true, true>, 256, "f16_ts_n256");
  auto mma8 = [&](auto kern, int N, const char* name, bool last) {
    float ms = best_ms([&] { kern<<<sms, 128>>>(mi, lo); });
    long long cyc = 0;
    cudaMemcpy(&cyc, lo, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)sms * mi * 4 * 2.0 * 128 * N * 32;
    printf(" \"%s\": {\"tops\": %.1f, \"cycles_per_mma\": %.1f}%s\n", name, ops / (ms * 1e-3) / 1e12,
           (double)cyc / (mi * 4.0), last ? "" : ",");
  };
  mma8(mma_i8_kernel<64>, 64, "i8_ss_n64", false);
  mma8(mma_i8_kernel<128>, 128, "i8_ss_n128", false);
  mma8(mma_i8_kernel<256>, 256, "i8_ss_n256", false);
  {
    // sustained: back-to-back launches for ~4 s (the power-capped clock a long int8 step runs at)
    float ms1 = best_ms([&] { mma_i8_kernel<256, true><<<sms, 128>>>(mi, lo); });
    {
      const double ops1 = (double)sms * mi * 4 * 2.0 * 128 * 256 * 32;
      printf(" \"i8_ss_n256_random_burst\": {\"tops\": %.1f},\n", ops1 / (ms1 * 1e-3) / 1e12);
    }
    const int reps = (int)(4000.0f / (ms1 > 0.01f ? ms1 : 0.01f)) + 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) mma_i8_kernel<256, true><<<sms, 128>>>(mi, lo);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)reps * sms * mi * 4 * 2.0 * 128 * 256 * 32;
    printf(" \"i8_ss_n256_random_sustained\": {\"tops\": %.1f, \"seconds\": %.2f}\n", ops / (ms * 1e-3) / 1e12, ms * 1e-3);
  }
  printf("}\n");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
