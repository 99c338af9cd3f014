// Does operand freshness change tcgen05.mma (kind::tf32) throughput?
// VA: A from TMEM cycles over `na` distinct 8-column blocks; VB: B cycles over `nb` distinct 2 KB smem rows blocks.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace rld;

template <int N, bool SS>
__global__ void bench(int iters, int na, int nb, long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* bsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(bsm)[i] = 1.0f + (i & 7);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbarrier_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ai = i % na, bi = i % nb;
      // B: N rows x 128 B blocks of N*128 bytes at bsm + bi * N * 128 (within 64 KB)
      const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(bsm + (size_t)bi * N * 128)) + 2 * (i & 3);
      if (SS) {
        const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(bsm + 32768 + (size_t)(ai % 2) * 16384)) + 2 * (i & 3);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u) : "memory");
      } else {
        ptx::mma_tf32_ts(tmem, tmem + 256 + 8 * ai, bd, idesc, 1u);
      }
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

template <int N, bool SS>
void run(int na, int nb) {
  long long* d;
  cudaMalloc(&d, 8);
  const int iters = 8000;
  cudaFuncSetAttribute(bench<N, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  bench<N, SS><<<148, 128, 66 * 1024>>>(iters, na, nb, d);
  bench<N, SS><<<148, 128, 66 * 1024>>>(iters, na, nb, d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d %s na=%2d nb=%2d: %.1f cycles per MMA  %s\n", N, SS ? "SS" : "TS", na, nb, (double)h / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, false>(4, 1);
  run<64, false>(32, 1);
  run<64, false>(4, 4);
  run<64, false>(32, 4);
  run<64, true>(1, 1);
  run<64, true>(2, 4);
  run<128, false>(4, 1);
  run<128, false>(32, 2);
  run<128, true>(2, 2);
  return 0;
}
