// Microbenchmark: cycles per tcgen05.mma kind::tf32 (A from TMEM, B from SMEM)
// as a function of N, one CTA per SM, single issuing thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2405_03474_b200/csrc mma_microbench.cu -o mma_mb
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace rld;

template <int N, int NACC, int COMMIT_EVERY>
__global__ void bench(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t bsm[256 * 128];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<float*>(bsm)[i] = 1.0f;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&bar2, 1); ptx::fence_mbarrier_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32(128, N);
    const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(bsm));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (NACC == 0) {
          const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(bsm)) + 2 * k;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(ad), "l"(bd + 2 * k), "r"(idesc), "r"(1u) : "memory");
        } else {
          ptx::mma_tf32_ts(tmem + (k % NACC) * (256 / NACC), tmem + 256 + 8 * k, bd + 2 * k, idesc, 1u);
        }
      }
      if (COMMIT_EVERY && (i % COMMIT_EVERY) == 0) ptx::tc_commit(&bar2);
    }
    ptx::tc_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

template <int N, int NACC, int CE>
void run() {
  long long* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  bench<N, NACC, CE><<<148, 128>>>(iters, d);
  bench<N, NACC, CE><<<148, 128>>>(iters, d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("N=%3d acc=%d commit_every=%d: %.1f cycles per MMA (128x%dx8 tf32, A in TMEM)  %s\n", N, NACC, CE, (double)h / (iters * 4), N,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, 1, 0>();
  run<64, 1, 1>();
  run<64, 1, 2>();
  run<64, 1, 8>();
  run<128, 1, 0>();
  run<128, 1, 1>();
  return 0;
}
