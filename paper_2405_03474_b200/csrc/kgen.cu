// Dense kernel-matrix generation: K[i, j] = a^2 k(|x_i - x_j|) + jitter [i == j].
//
// Follows src/kernels.py:40-73 (RBF and Matern-5/2 values, diagonal set to
// a^2 + jitter exactly) but forms r^2 from direct coordinate differences
// instead of |x|^2 + |y|^2 - 2 x.y: same value up to rounding, and no
// cancellation for close pairs.  r^2 is float64; the kernel
// function is float64 for a float64 K and float32 (MUFU exp) for a float32 K.
//
// One CTA writes a 32-row x 256-column tile; each thread owns one column and
// walks the 32 rows, so every row store is a coalesced 256-element segment.
// Point dimension and kernel family are template parameters (no per-entry
// branches, the column point stays in registers).
#include "rld_internal.cuh"
#include "rld_device.cuh"

namespace rld {

namespace {

constexpr int KG_ROWS = 32;
constexpr int KG_COLS = 256;

// DIM > 0: compile-time point dimension (registers only); DIM == 0: runtime d <= RLD_MAX_DIM.
// TILED: K is the tiled fp32 layout [ceil(rows/128)][ceil(n/32)][128][32] (ld unused).
template <typename T, int DIM, int FAM, bool TILED = false>
__global__ void __launch_bounds__(KG_COLS)
kgen_kernel(const double* __restrict__ X, int64_t n, KernelParams kp, int64_t row0, int64_t rows,
            T* __restrict__ K, int64_t ld) {
  extern __shared__ double sm[];
  const int d = DIM > 0 ? DIM : kp.d;
  double* xr = sm;                       // KG_ROWS x d
  const int64_t i0 = (int64_t)blockIdx.y * KG_ROWS;
  const int64_t j = (int64_t)blockIdx.x * KG_COLS + threadIdx.x;
  for (int e = threadIdx.x; e < KG_ROWS * d; e += blockDim.x) {
    int64_t r = i0 + e / d;
    xr[e] = (r < rows) ? X[(row0 + r) * d + (e % d)] : 0.0;
  }
  __syncthreads();
  if (j >= n) return;
  constexpr int DD = DIM > 0 ? DIM : RLD_MAX_DIM;
  double xc[DD];
#pragma unroll
  for (int k = 0; k < DD; ++k) xc[k] = (k < d) ? X[j * d + k] : 0.0;
  const int rmax = (int)min64(KG_ROWS, rows - i0);
  T* out = K + i0 * ld + j;
  const int64_t gi0 = row0 + i0;
  const int64_t ks = (n + 31) >> 5;
  for (int r = 0; r < rmax; ++r) {
    double r2 = 0.0;
#pragma unroll
    for (int k = 0; k < DD; ++k) {
      if (DIM > 0 || k < d) {
        const double diff = xr[r * d + k] - xc[k];
        r2 = fma(diff, diff, r2);
      }
    }
    double v;
    if constexpr (sizeof(T) == 4) {
      // float32 K: r^2 from float64 differences as above, the kernel function in float32
      // (relative error ~3e-7, about the float32 rounding of the stored value itself; the fp64
      // exp made this kernel FP64-bound at 3-4x the time of writing K)
      if (FAM == RLD_RBF) {
        v = (double)((float)kp.a2 * __expf(-(float)(r2 * kp.inv_2l2)));
      } else {
        const float u = sqrtf((float)r2) * (float)kp.s5_over_l;
        v = (double)((float)kp.a2 * (1.0f + u + u * u * (1.0f / 3.0f)) * __expf(-u));
      }
    } else if (FAM == RLD_RBF) {
      v = kp.a2 * exp(-r2 * kp.inv_2l2);
    } else {
      const double u = sqrt(r2) * kp.s5_over_l;
      v = kp.a2 * (1.0 + u + u * u * (1.0 / 3.0)) * exp(-u);
    }
    if (gi0 + r == j) v = kp.diag;
    if (TILED) {
      const int64_t i = i0 + r;
      K[(((i >> 7) * ks + (j >> 5)) << 12) + ((i & 127) << 5) + (j & 31)] = (T)v;
    } else {
      out[(int64_t)r * ld] = (T)v;
    }
  }
}

template <typename T, int DIM, bool TILED = false>
void launch_kgen(dim3 grid, size_t smem, const double* X, int64_t n, const KernelParams& kp, int64_t row0,
                 int64_t rows, T* K, int64_t ld, cudaStream_t st) {
  if (kp.family == RLD_RBF)
    kgen_kernel<T, DIM, RLD_RBF, TILED><<<grid, KG_COLS, smem, st>>>(X, n, kp, row0, rows, K, ld);
  else
    kgen_kernel<T, DIM, RLD_MATERN52, TILED><<<grid, KG_COLS, smem, st>>>(X, n, kp, row0, rows, K, ld);
  RLD_LAUNCH_CHECK();
}

}  // namespace

template <typename T>
void build_kernel_rows(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows,
                       T* K, int64_t ld, cudaStream_t st) {
  if (rows <= 0) return;
  dim3 grid((unsigned)ceil_div(n, KG_COLS), (unsigned)ceil_div(rows, KG_ROWS));
  size_t smem = sizeof(double) * KG_ROWS * kp.d;
  switch (kp.d) {   // the BASELINE configs use d = 2, 3, 8
    case 1: launch_kgen<T, 1>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
    case 2: launch_kgen<T, 2>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
    case 3: launch_kgen<T, 3>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
    case 4: launch_kgen<T, 4>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
    case 8: launch_kgen<T, 8>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
    default: launch_kgen<T, 0>(grid, smem, X, n, kp, row0, rows, K, ld, st); break;
  }
}

void build_kernel_tiles(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, float* Kt,
                        cudaStream_t st) {
  if (rows <= 0) return;
  RLD_CUDA(cudaMemsetAsync(Kt, 0, sizeof(float) * tiled_elems(rows, n), st));   // padding rows / columns
  dim3 grid((unsigned)ceil_div(n, KG_COLS), (unsigned)ceil_div(rows, KG_ROWS));
  size_t smem = sizeof(double) * KG_ROWS * kp.d;
  switch (kp.d) {
    case 1: launch_kgen<float, 1, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
    case 2: launch_kgen<float, 2, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
    case 3: launch_kgen<float, 3, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
    case 4: launch_kgen<float, 4, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
    case 8: launch_kgen<float, 8, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
    default: launch_kgen<float, 0, true>(grid, smem, X, n, kp, row0, rows, Kt, 0, st); break;
  }
}

template void build_kernel_rows<double>(const double*, int64_t, const KernelParams&, int64_t, int64_t,
                                        double*, int64_t, cudaStream_t);
template void build_kernel_rows<float>(const double*, int64_t, const KernelParams&, int64_t, int64_t,
                                       float*, int64_t, cudaStream_t);

}  // namespace rld
