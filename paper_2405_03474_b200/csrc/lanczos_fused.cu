// Fused step of the preconditioned two-sequence Lanczos recurrence for one GPU:
// the vector work between two K x X products in five kernels instead of ~12, every vector block
// read once per kernel; the two products with U stay cuBLAS DGEMMs (hand-written register-tiled
// FP64 versions measured 4x slower at config 2: 135 vs 32 us per step).
//
// Notation as in vec_kernels.cu (src/lanczos.py:56-72 restated, src/precond.py:102-115 for the
// Woodbury square-root apply):
//   alpha_j = x_j . K x_j ;  u = K x_j - alpha_j p_j - beta_{j-1} p_{j-1} ;  w = u / sqrt(base)
//   T = h o (U^T w) ;  z = (w + U T) / sqrt(base) ;  beta_j = sqrt(u . z)
//   p_{j+1} = u / beta_j ;  x_{j+1} = z / beta_j   (written straight into the tensor-core B operand)
// Rows are processed in 128-row chunks; every reduction is a fixed-order sum of per-chunk
// partials (lane-strided, then a fixed butterfly), so results are deterministic.
#include "rld_internal.cuh"
#include "rld_device.cuh"
#include "rld_kernels.cuh"

namespace rld {

namespace {

constexpr int CH = 128;   // rows per chunk
constexpr int FT = 256;   // threads per CTA

// sum over q of part[q * m + c], by one warp (lane-strided partial sums, then a fixed butterfly):
// every lane returns the same value
__device__ __forceinline__ double chunk_total_warp(const double* __restrict__ part, int nparts, int m, int c) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll 4
  for (int q = lane; q < nparts; q += 32) s += part[(int64_t)q * m + c];
  return warp_sum(s);
}

// dotp[ch * m + c] = sum over chunk ch of a[c, i] * b[c, i]
__global__ void __launch_bounds__(FT)
chunk_dots_kernel(int64_t n, int m, const double* __restrict__ a, const double* __restrict__ b,
                  double* __restrict__ dotp) {
  const int ch = blockIdx.x;
  const int64_t i0 = (int64_t)ch * CH;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < m; c += FT / 32) {
    double s = 0.0;
#pragma unroll
    for (int r = lane; r < CH; r += 32) {
      const int64_t i = i0 + r;
      if (i < n) s = fma(a[(int64_t)c * n + i], b[(int64_t)c * n + i], s);
    }
    s = warp_sum(s);
    if (lane == 0) dotp[(int64_t)ch * m + c] = s;
  }
}

// alpha_j (fixed-order total of the chunk partials of x . K x, masked by live), then the residual
// u = K x - alpha p - beta_{j-1} p_prev and w = u / sqrt(base) of this chunk
__global__ void __launch_bounds__(FT)
residual_kernel(int64_t n, int m, int j, int t, int nch, const double* __restrict__ dotp,
                const int* __restrict__ live, double* __restrict__ alpha, const double* __restrict__ beta,
                const double* __restrict__ KX, const double* __restrict__ p, const double* __restrict__ pp,
                const double* __restrict__ sqrt_base, double* __restrict__ u, double* __restrict__ w) {
  __shared__ double as[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = warp; c < m; c += FT / 32) {
    const double tot = chunk_total_warp(dotp, nch, m, c);
    const double a = live[c] ? tot : 0.0;   // probes past breakdown record 0
    if (lane == 0) {
      as[c] = a;
      if (blockIdx.x == 0) alpha[c * t + j] = a;
    }
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * CH;
  for (int e = tid; e < m * CH; e += FT) {
    const int c = e / CH, r = e % CH;
    const int64_t i = i0 + r;
    if (i >= n) continue;
    const int64_t o = (int64_t)c * n + i;
    double v = KX[o] - as[c] * p[o];
    if (j > 0) v -= beta[c * t + (j - 1)] * pp[o];
    u[o] = v;
    w[o] = v / sqrt_base[i];
  }
}

// z = w / sqrt(base) (w already holds w + U T) over w, dotp2[ch * m + c] = u . z over the chunk
__global__ void __launch_bounds__(FT)
z_dot_kernel(int64_t n, int m, const double* __restrict__ sqrt_base, const double* __restrict__ u,
             double* __restrict__ w, double* __restrict__ dotp2) {
  const int ch = blockIdx.x;
  const int64_t i0 = (int64_t)ch * CH;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < m; c += FT / 32) {
    double s = 0.0;
#pragma unroll
    for (int r = lane; r < CH; r += 32) {
      const int64_t i = i0 + r;
      if (i < n) {
        const int64_t o = (int64_t)c * n + i;
        const double z = w[o] / sqrt_base[i];
        w[o] = z;
        s = fma(u[o], z, s);
      }
    }
    s = warp_sum(s);
    if (lane == 0) dotp2[(int64_t)ch * m + c] = s;
  }
}

// beta_j from the chunk partials of u . z, breakdown test (src/lanczos.py:66-70); one warp per probe
__global__ void beta_chunks_kernel(int m, int nch, int j, int t, double rtol, const double* __restrict__ dotp2,
                                   double* __restrict__ alpha, double* __restrict__ beta, double* __restrict__ beta_ref,
                                   int* __restrict__ live, int* __restrict__ size) {
  const int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (c >= m) return;
  const double b = sqrt(fmax(chunk_total_warp(dotp2, nch, m, c), 0.0));
  if ((threadIdx.x & 31) != 0) return;
  if (j == 0) beta_ref[c] = b;
  if (!live[c]) {
    beta[c * t + j] = 0.0;
    return;
  }
  if (b <= rtol * fmax(beta_ref[c], fabs(alpha[c * t + j]))) {
    live[c] = 0;
    size[c] = j + 1;
    beta[c * t + j] = 0.0;
    return;
  }
  beta[c * t + j] = b;
}

__global__ void alpha_chunks_kernel(int m, int nch, int j, int t, const double* __restrict__ dotp,
                                    const int* __restrict__ live, double* __restrict__ alpha) {
  const int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (c >= m) return;
  const double tot = chunk_total_warp(dotp, nch, m, c);
  if ((threadIdx.x & 31) == 0) alpha[c * t + j] = live[c] ? tot : 0.0;
}

// p_prev <- p ; p <- u / beta ; x <- z / beta (zero past breakdown), and x in the tensor-core
// B layout (the same conversion as kv_tc_split) when bhi != nullptr
__global__ void advance_split_kernel(int64_t n, int m, int j, int t, const double* __restrict__ beta,
                                     const int* __restrict__ live, const double* __restrict__ u,
                                     const double* __restrict__ z, double* __restrict__ p, double* __restrict__ pp,
                                     double* __restrict__ x, float* __restrict__ bhi, float* __restrict__ blo,
                                     int64_t mp, int64_t ks, int blocked, int mode) {
  const int64_t total = (int64_t)m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, i = e % n;
    const double b = beta[c * t + j];
    const bool onp = live[c] != 0;
    pp[e] = p[e];
    p[e] = onp ? u[e] / b : 0.0;
    const double xv = onp ? z[e] / b : 0.0;
    x[e] = xv;
    if (bhi) {
      const int64_t o = blocked ? ((i >> 5) * mp + c) * 32 + (i & 31) : c * (ks * 32) + i;
      float h = (float)xv;
      if (mode == 3) {
        h = __uint_as_float(__float_as_uint(h) & 0xFFFFE000u);
        blo[o] = (float)(xv - (double)h);
      }
      bhi[o] = h;
    }
  }
}

int grid_elems(int64_t total) { return (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(total, 256)), 148 * 16); }

}  // namespace

bool lanczos_fused_fits(int64_t s, int k) { return s >= 1 && s <= 64; }

void lanczos_chunk_dots(int64_t n, int m, const double* a, const double* b, double* dotp, cudaStream_t st) {
  chunk_dots_kernel<<<(unsigned)ceil_div(n, CH), FT, 0, st>>>(n, m, a, b, dotp);
  RLD_LAUNCH_CHECK();
}

void lanczos_alpha_chunks(int m, int64_t n, int j, int t, const double* dotp, const int* live, double* alpha,
                          cudaStream_t st) {
  alpha_chunks_kernel<<<(unsigned)ceil_div(32 * m, 128), 128, 0, st>>>(m, (int)ceil_div(n, CH), j, t, dotp, live,
                                                                       alpha);
  RLD_LAUNCH_CHECK();
}

void lanczos_fused_residual(const LanczosFusedArgs& a, cudaStream_t st) {
  const int nch = (int)ceil_div(a.n, CH);
  residual_kernel<<<nch, FT, 0, st>>>(a.n, a.m, a.j, a.t, nch, a.dotp, a.live, a.alpha, a.beta, a.KX, a.p, a.pp,
                                       a.sqrt_base, a.u, a.w);
  RLD_LAUNCH_CHECK();
}

void lanczos_fused_finish(const LanczosFusedArgs& a, cudaStream_t st) {
  const int nch = (int)ceil_div(a.n, CH);
  z_dot_kernel<<<nch, FT, 0, st>>>(a.n, a.m, a.sqrt_base, a.u, a.w, a.dotp2);
  RLD_LAUNCH_CHECK();
  beta_chunks_kernel<<<(unsigned)ceil_div(32 * a.m, 128), 128, 0, st>>>(a.m, nch, a.j, a.t, a.rtol, a.dotp2, a.alpha,
                                                                       a.beta, a.beta_ref, a.live_rw, a.size);
  RLD_LAUNCH_CHECK();
  advance_split_kernel<<<grid_elems((int64_t)a.m * a.n), 256, 0, st>>>(a.n, a.m, a.j, a.t, a.beta, a.live, a.u, a.w,
                                                                       a.p, a.pp, a.x, a.bl.bhi, a.bl.blo, a.bl.mp,
                                                                       a.bl.ks, a.bl.blocked, a.bl.mode);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
