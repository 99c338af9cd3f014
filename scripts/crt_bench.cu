// Feasibility microbenchmark for a CRT ("Ozaki scheme II") float64 product: L int8 modular GEMMs
// (one per modulus) over k-step-tiled, pre-swizzled residue images, tcgen05 kind::i8, one MMA per
// 32-column k-step, KB k-steps per bulk-copied stage.  Times the GEMM core at the config-3 sketch
// shape (n = 65536 rows x n columns, m = 522 vectors as 3 passes of NT = 176, L = 15 moduli) on
// random residues; checks one output tile against a host int64 reference.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2405_03474_b200/csrc crt_bench.cu -o crt_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace rld;

namespace {
constexpr int BM = 128, BK = 32, THREADS = 256;

__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}
constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// grid (passes, tiles, L): CTA (pass, tile, l) computes the int32 product of K-residue tile (tile, l)
// and V-residue block (l, pass) over all KS k-steps, reduces it mod p_l and stores uint8 residues.
template <int NT, int KB, int STAGES, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB)
crt_gemm(const int8_t* __restrict__ Ar, const int8_t* __restrict__ Br, int KS, int tiles, int passes,
         const int* __restrict__ mods, uint8_t* __restrict__ out, int64_t m_pad, int64_t rows) {
  constexpr uint32_t A_STEP = BM * BK, B_STEP = NT * BK;
  constexpr uint32_t STAGE = KB * (A_STEP + B_STEP);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* accfull = empty + STAGES;
  uint32_t* holder = reinterpret_cast<uint32_t*>(accfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pass = blockIdx.x, tile = blockIdx.y, l = blockIdx.z;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accfull, 1);
    ptx::fence_mbarrier_init();
  }
  constexpr uint32_t COLS = NT <= 256 ? 256 : 512;
  if (warp == 2) ptx::tmem_alloc(holder, COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  const int nst = KS / KB;
  if (warp == 0) {
    if (ptx::elect_one()) {
      const int8_t* ga = Ar + ((int64_t)tile * gridDim.z + l) * (int64_t)KS * A_STEP;
      const int8_t* gb = Br + ((int64_t)l * passes + pass) * (int64_t)KS * B_STEP;
      for (int s = 0; s < nst; ++s) {
        const int st = s % STAGES;
        if (s >= STAGES) ptx::mbar_wait(&empty[st], ((s / STAGES) - 1) & 1);
        unsigned char* dst = smem + st * STAGE;
        ptx::mbar_arrive_expect_tx(&full[st], STAGE);
        bulk_load(dst, ga + (int64_t)s * KB * A_STEP, KB * A_STEP, &full[st]);
        bulk_load(dst + KB * A_STEP, gb + (int64_t)s * KB * B_STEP, KB * B_STEP, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      const uint32_t sbase = ptx::smem_u32(smem);
      for (int s = 0; s < nst; ++s) {
        const int st = s % STAGES;
        ptx::mbar_wait(&full[st], (uint32_t)((s / STAGES) & 1));
        ptx::tc_fence_after();
        const uint32_t a0 = sbase + st * STAGE, b0 = a0 + KB * A_STEP;
#pragma unroll
        for (int k = 0; k < KB; ++k)
          mma_i8_ss(tmem, desc_sw32(a0 + k * A_STEP), desc_sw32(b0 + k * B_STEP), idesc_i8(BM, NT),
                    (s > 0 || k > 0) ? 1u : 0u);
        ptx::tc_commit(&empty[st]);
      }
      ptx::tc_commit(accfull);
    }
  } else if (warp >= 4) {
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    ptx::mbar_wait_sleep(accfull, 0);
    ptx::tc_fence_after();
    const int p = mods[l];
    const int64_t r = (int64_t)tile * BM + row;
    uint8_t* o = out + ((int64_t)l * m_pad + (int64_t)pass * NT) * rows + r;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 16) {
      uint32_t v[16];
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + (uint32_t)c0, v);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        int x = (int)v[e] % p;
        if (x < 0) x += p;
        o[(int64_t)(c0 + e) * rows] = (uint8_t)x;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, COLS);
}

__global__ void fill_random(int8_t* p, int64_t n, uint32_t seed, int lim) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (int8_t)((int)(x % (2 * lim + 1)) - lim);
  }
}
}  // namespace

// swizzled byte offset within a [R][32] tile (Swizzle<1,4,3>: 16-byte halves swap in rows 4..7 of each 8-row atom)
static int64_t swz(int r, int c) {
  const int64_t o = (int64_t)r * 32 + c;
  return o ^ (((o >> 7) & 1) << 4);
}

template <int NT, int KB, int STAGES, int MINB = 1>
float run(int n, int m, int L, int reps, bool check) {
  const int KS = n / BK, tiles = n / BM, passes = (m + NT - 1) / NT;
  const int64_t abytes = (int64_t)tiles * L * KS * BM * BK, bbytes = (int64_t)L * passes * KS * NT * BK;
  int8_t *A, *B;
  uint8_t* out;
  int* mods;
  const int64_t m_pad = (int64_t)passes * NT;
  cudaMalloc(&A, abytes);
  cudaMalloc(&B, bbytes);
  cudaMalloc(&out, (int64_t)L * m_pad * n);
  cudaMalloc(&mods, sizeof(int) * 16);
  const int hm[16] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
  cudaMemcpy(mods, hm, sizeof hm, cudaMemcpyHostToDevice);
  fill_random<<<4096, 256>>>(A, abytes, 1234u, 127);
  fill_random<<<4096, 256>>>(B, bbytes, 999u, 127);
  const size_t smem = (size_t)STAGES * KB * (BM * BK + NT * BK) + 1024 + 256;
  cudaFuncSetAttribute(crt_gemm<NT, KB, STAGES, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(passes, tiles, L);
  crt_gemm<NT, KB, STAGES, MINB><<<grid, THREADS, smem>>>(A, B, KS, tiles, passes, mods, out, m_pad, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) crt_gemm<NT, KB, STAGES, MINB><<<grid, THREADS, smem>>>(A, B, KS, tiles, passes, mods, out, m_pad, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(err));
  if (check) {   // tile 1, modulus 2, pass 0: rows 0..127 x first 16 vectors
    const int tile = 1, l = 2, pass = 0;
    std::vector<int8_t> ha((int64_t)KS * BM * BK), hb((int64_t)KS * NT * BK);
    cudaMemcpy(ha.data(), A + ((int64_t)tile * L + l) * KS * BM * BK, ha.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), B + ((int64_t)l * passes + pass) * KS * NT * BK, hb.size(), cudaMemcpyDeviceToHost);
    std::vector<uint8_t> ho((int64_t)m_pad * n);
    cudaMemcpy(ho.data(), out + (int64_t)l * m_pad * n, ho.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < BM; r += 7)
      for (int c = 0; c < 16; ++c) {
        long long s = 0;
        for (int k = 0; k < KS; ++k)
          for (int j = 0; j < BK; ++j)
            s += (long long)ha[(int64_t)k * BM * BK + swz(r, j)] * hb[(int64_t)k * NT * BK + swz(c, j)];
        long long x = s % hm[l];
        if (x < 0) x += hm[l];
        if ((int)ho[(int64_t)c * n + tile * BM + r] != (int)x) ++bad;
      }
    printf("check: %d mismatches\n", bad);
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(out);
  cudaFree(mods);
  return ms;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 65536;
  const int m = 522, L = 15;
  float ms;
  ms = run<176, 4, 5>(n, m, L, 3, true);
  printf("NT=176 KB=4 S=5: %.2f ms  (%.1f int8 TOPS)\n", ms, 2.0 * L * n * (double)n * 528 / (ms * 1e-3) / 1e12);
  ms = run<176, 2, 4, 2>(n, m, L, 3, true);
  printf("NT=176 KB=2 S=4 2/SM: %.2f ms  (%.1f int8 TOPS)\n", ms, 2.0 * L * n * (double)n * 528 / (ms * 1e-3) / 1e12);
  ms = run<176, 4, 2, 2>(n, m, L, 3, false);
  printf("NT=176 KB=4 S=2 2/SM: %.2f ms  (%.1f int8 TOPS)\n", ms, 2.0 * L * n * (double)n * 528 / (ms * 1e-3) / 1e12);
  ms = run<176, 1, 8, 2>(n, m, L, 3, false);
  printf("NT=176 KB=1 S=8 2/SM: %.2f ms  (%.1f int8 TOPS)\n", ms, 2.0 * L * n * (double)n * 528 / (ms * 1e-3) / 1e12);
  return 0;
}
