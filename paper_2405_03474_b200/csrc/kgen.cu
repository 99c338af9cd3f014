// Dense kernel-matrix generation: K[i, j] = a^2 k(|x_i - x_j|) + jitter [i == j].
//
// Follows src/kernels.py:40-73 (RBF and Matern-5/2 values, diagonal set to
// a^2 + jitter exactly) but forms r^2 from direct coordinate differences
// instead of |x|^2 + |y|^2 - 2 x.y: same value up to rounding, and no
// cancellation for close pairs.  Arithmetic is float64; the
// fp32 store rounds the float64 value once.
//
// One CTA writes a 32-row x 256-column tile; each thread owns one column and
// walks the 32 rows, so every row store is a coalesced 256-element segment.
#include "rld_internal.cuh"
#include "rld_device.cuh"

namespace rld {

namespace {

constexpr int KG_ROWS = 32;
constexpr int KG_COLS = 256;

template <typename T>
__global__ void __launch_bounds__(KG_COLS)
kgen_kernel(const double* __restrict__ X, int64_t n, KernelParams kp, int64_t row0, int64_t rows,
            T* __restrict__ K, int64_t ld) {
  extern __shared__ double sm[];
  const int d = kp.d;
  double* xr = sm;                       // KG_ROWS x d
  const int64_t i0 = (int64_t)blockIdx.y * KG_ROWS;
  const int64_t j = (int64_t)blockIdx.x * KG_COLS + threadIdx.x;
  for (int e = threadIdx.x; e < KG_ROWS * d; e += blockDim.x) {
    int64_t r = i0 + e / d;
    xr[e] = (r < rows) ? X[(row0 + r) * d + (e % d)] : 0.0;
  }
  __syncthreads();
  if (j >= n) return;
  double xc[RLD_MAX_DIM];
#pragma unroll
  for (int k = 0; k < RLD_MAX_DIM; ++k) xc[k] = (k < d) ? X[j * d + k] : 0.0;
  const int rmax = (int)min64(KG_ROWS, rows - i0);
  for (int r = 0; r < rmax; ++r) {
    double r2 = 0.0;
#pragma unroll
    for (int k = 0; k < RLD_MAX_DIM; ++k) {
      if (k < d) {
        double diff = xr[r * d + k] - xc[k];
        r2 = fma(diff, diff, r2);
      }
    }
    const int64_t gi = row0 + i0 + r;
    double v = (gi == j) ? kp.diag : kernel_value_f64(kp, r2);
    K[(i0 + r) * ld + j] = (T)v;
  }
}

}  // namespace

template <typename T>
void build_kernel_rows(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows,
                       T* K, int64_t ld, cudaStream_t st) {
  if (rows <= 0) return;
  dim3 grid((unsigned)ceil_div(n, KG_COLS), (unsigned)ceil_div(rows, KG_ROWS));
  size_t smem = sizeof(double) * KG_ROWS * kp.d;
  kgen_kernel<T><<<grid, KG_COLS, smem, st>>>(X, n, kp, row0, rows, K, ld);
  RLD_LAUNCH_CHECK();
}

template void build_kernel_rows<double>(const double*, int64_t, const KernelParams&, int64_t, int64_t,
                                        double*, int64_t, cudaStream_t);
template void build_kernel_rows<float>(const double*, int64_t, const KernelParams&, int64_t, int64_t,
                                       float*, int64_t, cudaStream_t);

}  // namespace rld
