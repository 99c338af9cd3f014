// Vector / small-matrix kernels of the estimator: per-probe dot products,
// the preconditioned Lanczos recurrence, the multishift Thomas solves with the
// Hutchinson mean, Philox probe generation, and the small preconditioner
// epilogues.  All reductions have a fixed order (deterministic, no atomics).
#include "rld_internal.cuh"
#include "rld_device.cuh"
#include "rld_kernels.cuh"

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

namespace rld {

namespace {

constexpr int RB = 256;  // threads per reduction block

// partial[c * P + p] = sum over chunk p of a[c, j] * b[c, j]
__global__ void __launch_bounds__(RB)
rows_dot_partial(int64_t n, const double* __restrict__ a, int64_t lda, const double* __restrict__ b,
                 int64_t ldb, int64_t chunk, double* __restrict__ partial) {
  __shared__ double red[RB / 32];
  const int64_t c = blockIdx.y;
  const int P = gridDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min64(n, j0 + chunk);
  const double* ar = a + c * lda;
  const double* br = b + c * ldb;
  double s = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += RB) s = fma(ar[j], br[j], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[c * P + blockIdx.x] = s;
}

__global__ void rows_dot_final(int64_t m, int P, const double* __restrict__ partial, double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double s = 0.0;
  for (int p = 0; p < P; ++p) s += partial[c * P + p];
  out[c] = s;
}

}  // namespace

void rows_dot(int64_t m, int64_t n, const double* a, int64_t lda, const double* b, int64_t ldb,
              double* out, DevBuf& scratch, cudaStream_t st, int* launches) {
  if (m <= 0) return;
  int P = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(n, 4 * RB)), std::max<int64_t>(1, 1184 / m));
  const int64_t chunk = ceil_div(n, P);
  P = (int)ceil_div(n, chunk);
  scratch.reserve(sizeof(double) * m * P);
  rows_dot_partial<<<dim3(P, (unsigned)m), RB, 0, st>>>(n, a, lda, b, ldb, chunk, scratch.as<double>());
  RLD_LAUNCH_CHECK();
  rows_dot_final<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(m, P, scratch.as<double>(), out);
  RLD_LAUNCH_CHECK();
  if (launches) *launches += 2;
}

// ---------------------------------------------------------------------------
// Philox Rademacher rows: out[r, j] = +-1 from bit 31 of 32-bit word (r*n + j)
// of the stream (low half of each 64-bit word first) -- numpy's
// integers(0, 2) through buffered_bounded_lemire_uint32 (threshold 0, so no
// rejection), then 2x - 1 (src/linalg.py:84-85).

namespace {
__global__ void rademacher_kernel(uint64_t k0, uint64_t k1, int64_t rows, int64_t n, int64_t col0,
                                  int64_t ncols, int64_t ld, double* __restrict__ out) {
  const int64_t total = rows * ncols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ncols, j = col0 + e % ncols;
    const uint64_t f = (uint64_t)(r * n + j);
    const uint64_t word = philox_word(f >> 1, k0, k1);
    const uint32_t u = (f & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
    out[r * ld + (j - col0)] = (u >> 31) ? 1.0 : -1.0;
  }
}
}  // namespace

void rademacher_rows(const uint64_t key[2], int64_t rows, int64_t n, int64_t col0, int64_t ncols, int64_t ld,
                     double* out, cudaStream_t st) {
  const int64_t total = rows * ncols;
  if (total <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  rademacher_kernel<<<blocks, 256, 0, st>>>(key[0], key[1], rows, n, col0, ncols, ld, out);
  RLD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Lanczos pieces.  Notation (rows layout, probe c, local index i):
//   q_j     Lanczos vector of the symmetric operator A = N^-1 K N^-T (src/estimators.py:71-72)
//   x_j = N^-T q_j,  p_j = N q_j          (so P^-1 p_j = x_j with P = N N^T)
//   alpha_j = x_j . K x_j,  u = K x_j - alpha_j p_j - beta_{j-1} p_{j-1} = N r_j
//   z = P^-1 u = N^-T r_j,  beta_j = sqrt(u . z) = |r_j|
// which is the reference's recurrence (src/lanczos.py:56-72) without storing Q.

namespace {

__global__ void normalize_rows_kernel(int64_t m, int64_t n, const double* __restrict__ z,
                                      const double* __restrict__ nrm2, double* __restrict__ norms,
                                      double* __restrict__ q) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n;
    const double nv = sqrt(nrm2[c]);
    if (e % n == 0) norms[c] = nv;
    q[e] = z[e] / nv;
  }
}

// u = KX - alpha p - beta_prev p_prev ; w = u / sqrt_base
__global__ void lanczos_residual_kernel(int64_t m, int64_t n, int j, int t, const double* __restrict__ KX,
                                        const double* __restrict__ alpha, const double* __restrict__ beta,
                                        const double* __restrict__ p, const double* __restrict__ p_prev,
                                        const double* __restrict__ sqrt_base, int three_term, double* __restrict__ u,
                                        double* __restrict__ w) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, i = e % n;
    double v = KX[e];
    if (three_term) {
      v -= alpha[c * t + j] * p[e];
      if (j > 0) v -= beta[c * t + (j - 1)] * p_prev[e];
    }
    u[e] = v;
    w[e] = v / sqrt_base[i];
  }
}

// beta_j, breakdown test (src/lanczos.py:66-70), per probe
__global__ void lanczos_beta_kernel(int64_t m, int j, int t, double rtol, const double* __restrict__ beta2,
                                    double* __restrict__ alpha, double* __restrict__ beta,
                                    double* __restrict__ beta_ref, int* __restrict__ live,
                                    int* __restrict__ size) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const double b = sqrt(fmax(beta2[c], 0.0));
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

// p_prev <- p ; p <- u / beta ; x <- z / beta  (zero for probes past breakdown)
__global__ void lanczos_advance_kernel(int64_t m, int64_t n, int j, int t, const double* __restrict__ beta,
                                       const int* __restrict__ live, const double* __restrict__ u,
                                       const double* __restrict__ z, double* __restrict__ p,
                                       double* __restrict__ p_prev, double* __restrict__ x) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n;
    const double b = beta[c * t + j];
    const bool on = live[c] != 0;
    p_prev[e] = p[e];
    p[e] = on ? u[e] / b : 0.0;
    x[e] = on ? z[e] / b : 0.0;
  }
}

// For probes already past breakdown, alpha of later steps must not be recorded.
__global__ void lanczos_alpha_mask_kernel(int64_t m, int j, int t, const double* __restrict__ dots,
                                          const int* __restrict__ live, double* __restrict__ alpha) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  alpha[c * t + j] = live[c] ? dots[c] : 0.0;
}

// Multishift Thomas solves (src/linalg.py:125-156 via src/lanczos.py:77-84) and
// the per-probe accumulation b |v|^2 + sum_j c_j v.(Q^T w_j) = |v|^2 b + |v| sum_j c_j w_j[0]
// (src/estimators.py:89-92), then the fixed-order mean (src/estimators.py:93).
__global__ void thomas_hutchinson_kernel(int64_t m, int t, const double* __restrict__ alpha,
                                         const double* __restrict__ beta, const int* __restrict__ size,
                                         const double* __restrict__ norms, int npoles, double offset,
                                         const double* __restrict__ poles, const double* __restrict__ residues,
                                         double* __restrict__ per_probe, double* __restrict__ trace,
                                         int* __restrict__ flags) {
  extern __shared__ double cbuf[];  // t doubles per thread
  const int64_t c = threadIdx.x;
  for (int64_t cc = c; cc < m; cc += blockDim.x) {
    const int ms = size[cc];
    const double nv = norms[cc];
    double* cp = cbuf + threadIdx.x * t;
    double acc = offset * nv * nv;
    for (int q = 0; q < npoles; ++q) {
      const double shift = -poles[q];
      // forward sweep
      double piv = alpha[cc * t] + shift;
      if (fabs(piv) < 1e-300) { atomicOr(flags, RLD_FLAG_SINGULAR); piv = 1e-300; }
      // cp[i] = e_i / pivot_i in the lower half of the scratch, dp[i] in the upper half
      double* dpv = cbuf + blockDim.x * t + threadIdx.x * t;
      dpv[0] = nv / piv;
      if (ms > 1) cp[0] = beta[cc * t] / piv;
      for (int i = 1; i < ms; ++i) {
        const double e = beta[cc * t + (i - 1)];
        piv = (alpha[cc * t + i] + shift) - e * cp[i - 1];
        if (fabs(piv) < 1e-300) { atomicOr(flags, RLD_FLAG_SINGULAR); piv = 1e-300; }
        dpv[i] = (0.0 - e * dpv[i - 1]) / piv;
        if (i < ms - 1) cp[i] = beta[cc * t + i] / piv;
      }
      double xv = dpv[ms - 1];
      for (int i = ms - 2; i >= 0; --i) xv = dpv[i] - cp[i] * xv;
      acc += residues[q] * nv * xv;
    }
    per_probe[cc] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t cc = 0; cc < m; ++cc) s += per_probe[cc];
    *trace = s / (double)m;
  }
}

}  // namespace

static int grid_for(int64_t total) { return (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(total, 256)), 148 * 16); }

void normalize_rows(int64_t m, int64_t n, const double* z, const double* nrm2, double* norms, double* q,
                    cudaStream_t st) {
  normalize_rows_kernel<<<grid_for(m * n), 256, 0, st>>>(m, n, z, nrm2, norms, q);
  RLD_LAUNCH_CHECK();
}

void lanczos_residual(int64_t m, int64_t n, int j, int t, const double* KX, const double* alpha,
                      const double* beta, const double* p, const double* p_prev, const double* sqrt_base, double* u,
                      double* w, cudaStream_t st, bool three_term) {
  lanczos_residual_kernel<<<grid_for(m * n), 256, 0, st>>>(m, n, j, t, KX, alpha, beta, p, p_prev, sqrt_base,
                                                           three_term ? 1 : 0, u, w);
  RLD_LAUNCH_CHECK();
}

void lanczos_alpha(int64_t m, int j, int t, const double* dots, const int* live, double* alpha, cudaStream_t st) {
  lanczos_alpha_mask_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(m, j, t, dots, live, alpha);
  RLD_LAUNCH_CHECK();
}

void lanczos_beta(int64_t m, int j, int t, double rtol, const double* beta2, double* alpha, double* beta,
                  double* beta_ref, int* live, int* size, cudaStream_t st) {
  lanczos_beta_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(m, j, t, rtol, beta2, alpha, beta, beta_ref,
                                                                  live, size);
  RLD_LAUNCH_CHECK();
}

void lanczos_advance(int64_t m, int64_t n, int j, int t, const double* beta, const int* live, const double* u,
                     const double* z, double* p, double* p_prev, double* x, cudaStream_t st) {
  lanczos_advance_kernel<<<grid_for(m * n), 256, 0, st>>>(m, n, j, t, beta, live, u, z, p, p_prev, x);
  RLD_LAUNCH_CHECK();
}

namespace {
// Stochastic Lanczos quadrature epilogue (src/estimators.py:110-120): per probe,
// the eigenvalues theta and first eigenvector components Y[0, :] of its t x t
// tridiagonal T (implicit-shift QL, EISPACK tql2, tracking only the first row
// of the eigenvector matrix), then |v|^2 sum_i Y[0,i]^2 log(max(theta_i, floor))
// and the count of theta_i <= 0; fixed-order mean over probes.  One thread per probe.
__global__ void slq_epilogue_kernel(int64_t m, int t, const double* __restrict__ alpha,
                                    const double* __restrict__ beta, const int* __restrict__ size,
                                    const double* __restrict__ norms, double eig_floor,
                                    double* __restrict__ per_probe, double* __restrict__ trace,
                                    int* __restrict__ clamped, int* __restrict__ flags) {
  extern __shared__ double sbuf[];   // 3 t doubles per thread: d, e, z
  for (int64_t c = threadIdx.x; c < m; c += blockDim.x) {
    double* d = sbuf + (size_t)threadIdx.x * 3 * t;
    double* e = d + t;
    double* z = e + t;
    const int ms = size[c];
    for (int i = 0; i < ms; ++i) {
      d[i] = alpha[c * t + i];
      e[i] = (i + 1 < ms) ? beta[c * t + i] : 0.0;
      z[i] = (i == 0) ? 1.0 : 0.0;
    }
    // tql2 (implicit QL with Wilkinson-type shifts); e[i] couples d[i], d[i+1]
    for (int l = 0; l < ms; ++l) {
      int iter = 0;
      for (;;) {
        int mm = l;
        for (; mm < ms - 1; ++mm) {
          const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
          if (fabs(e[mm]) <= 2.220446049250313e-16 * dd) break;
        }
        if (mm == l) break;
        if (++iter > 60) {
          atomicOr(flags, RLD_FLAG_EIG_NOCONV);
          break;
        }
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
        double sn = 1.0, cs = 1.0, p = 0.0;
        int i = mm - 1;
        for (; i >= l; --i) {
          double f = sn * e[i];
          const double b = cs * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            break;
          }
          sn = f / r;
          cs = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * sn + 2.0 * cs * b;
          p = sn * r;
          d[i + 1] = g + p;
          g = cs * r - b;
          // first row of the accumulated rotations
          f = z[i + 1];
          z[i + 1] = sn * z[i] + cs * f;
          z[i] = cs * z[i] - sn * f;
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    }
    double acc = 0.0;
    int bad = 0;
    for (int i = 0; i < ms; ++i) {
      if (d[i] <= 0.0) ++bad;
      acc += z[i] * z[i] * log(fmax(d[i], eig_floor));
    }
    const double nv = norms[c];
    per_probe[c] = nv * nv * acc;
    if (bad) atomicAdd(clamped, bad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t c = 0; c < m; ++c) s += per_probe[c];
    *trace = s / (double)m;
  }
}
}  // namespace

void slq_epilogue(int64_t m, int t, const double* alpha, const double* beta, const int* size, const double* norms,
                  double eig_floor, double* per_probe, double* trace, int* clamped, int* flags, cudaStream_t st) {
  int threads = (int)std::min<int64_t>(128, std::max<int64_t>(1, m));
  threads = std::max(1, std::min(threads, (int)((48 * 1024) / (24 * std::max(t, 1)))));
  const size_t smem = sizeof(double) * 3 * threads * t;
  slq_epilogue_kernel<<<1, threads, smem, st>>>(m, t, alpha, beta, size, norms, eig_floor, per_probe, trace,
                                                clamped, flags);
  RLD_LAUNCH_CHECK();
}

void thomas_hutchinson(int64_t m, int t, const double* alpha, const double* beta, const int* size,
                       const double* norms, int npoles, double offset, const double* poles,
                       const double* residues, double* per_probe, double* trace, int* flags, cudaStream_t st) {
  int threads = (int)std::min<int64_t>(128, std::max<int64_t>(1, m));
  threads = std::max(1, std::min(threads, (int)((48 * 1024) / (16 * std::max(t, 1)))));
  size_t smem = sizeof(double) * 2 * threads * t;
  thomas_hutchinson_kernel<<<1, threads, smem, st>>>(m, t, alpha, beta, size, norms, npoles, offset, poles,
                                                     residues, per_probe, trace, flags);
  RLD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// elementwise helpers

namespace {
__global__ void scale_rows_kernel(int64_t rows, int64_t cols, int64_t ld, const double* __restrict__ f,
                                  int mode, double* __restrict__ a) {
  // a is col-major rows x cols (ld); multiply row r by f[r] (mode 0) or divide (mode 1)
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    double& v = a[c * ld + r];
    v = mode == 0 ? v * f[r] : v / f[r];
  }
}
__global__ void scale_cols_kernel(int64_t rows, int64_t cols, int64_t ld, const double* __restrict__ f,
                                  double* __restrict__ a) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    a[c * ld + r] *= f[c];
  }
}
__global__ void copy_kernel(int64_t count, const double* __restrict__ s, double* __restrict__ d) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    d[e] = s[e];
}
__global__ void fill_kernel(int64_t count, double v, double* __restrict__ d) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    d[e] = v;
}
}  // namespace

void scale_rows_colmajor(int64_t rows, int64_t cols, int64_t ld, const double* f, bool divide, double* a,
                         cudaStream_t st) {
  if (rows * cols <= 0) return;
  scale_rows_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, ld, f, divide ? 1 : 0, a);
  RLD_LAUNCH_CHECK();
}
void scale_cols_colmajor(int64_t rows, int64_t cols, int64_t ld, const double* f, double* a, cudaStream_t st) {
  if (rows * cols <= 0) return;
  scale_cols_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, ld, f, a);
  RLD_LAUNCH_CHECK();
}
void copy_doubles(int64_t count, const double* s, double* d, cudaStream_t st) {
  if (count <= 0) return;
  copy_kernel<<<grid_for(count), 256, 0, st>>>(count, s, d);
  RLD_LAUNCH_CHECK();
}
namespace {
__global__ void sub_block_kernel(int64_t rows, int64_t cols, const double* __restrict__ T, int64_t ldt,
                                 double* __restrict__ G, int64_t ldg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, r = e - c * rows;
    G[c * ldg + r] -= T[c * ldt + r];
  }
}
__global__ void combine_info_kernel(int* __restrict__ info, const int* __restrict__ i1, const int* __restrict__ i2,
                                    int n1) {
  const int a = *i1, b = *i2;
  *info = a != 0 ? a : (b != 0 ? n1 + b : 0);
}
}  // namespace

// G (column-major, ld ldg) -= T (ld ldt) over a rows x cols block
void sub_block(int64_t rows, int64_t cols, const double* T, int64_t ldt, double* G, int64_t ldg, cudaStream_t st) {
  if (rows * cols <= 0) return;
  sub_block_kernel<<<grid_for(rows * cols), 256, 0, st>>>(rows, cols, T, ldt, G, ldg);
  RLD_LAUNCH_CHECK();
}
// info = i1 (first failing pivot of the leading block) or n1 + i2 (trailing block), 0 on success
void combine_info(int* info, const int* i1, const int* i2, int n1, cudaStream_t st) {
  combine_info_kernel<<<1, 1, 0, st>>>(info, i1, i2, n1);
  RLD_LAUNCH_CHECK();
}

void fill_doubles(int64_t count, double v, double* d, cudaStream_t st) {
  if (count <= 0) return;
  fill_kernel<<<grid_for(count), 256, 0, st>>>(count, v, d);
  RLD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// preconditioner epilogues (src/precond.py:69-100, 231-233, 262-264)

namespace {

// Cholesky check of CholQR pass 1: flag QR_WEAK when potrf failed or a
// projected norm R_ii fell below weak_rtol * |Y_i| (CholQR loses accuracy there).
__global__ void cholqr_check_kernel(int w, const double* __restrict__ R, const double* __restrict__ gdiag,
                                    const int* __restrict__ info, double weak_rtol, int* __restrict__ flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && *info != 0) atomicOr(flags, RLD_FLAG_QR_WEAK);
  if (i >= w) return;
  const double rii = R[(int64_t)i * w + i];
  const double orig = sqrt(fmax(gdiag[i], 0.0));
  if (!(rii >= weak_rtol * fmax(orig, 1e-300))) atomicOr(flags, RLD_FLAG_QR_WEAK);
}

// Householder R: RankDeficient when |R_ii| < rtol |Y_i| (src/linalg.py:177-178); sign of R_ii
__global__ void householder_check_kernel(int w, const double* __restrict__ R, int64_t ldr,
                                         const double* __restrict__ norms2, double rtol, double* __restrict__ sgn,
                                         int* __restrict__ flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w) return;
  const double rii = R[(int64_t)i * ldr + i];
  if (!(fabs(rii) >= rtol * fmax(sqrt(fmax(norms2[i], 0.0)), 1e-300))) atomicOr(flags, RLD_FLAG_RANK_DEFICIENT);
  sgn[i] = rii < 0.0 ? -1.0 : 1.0;
}

// dst (w x w, ld w, column-major) = upper triangle of src (ld lds), zeros below
__global__ void copy_upper_kernel(int w, const double* __restrict__ src, int64_t lds, double* __restrict__ dst) {
  const int64_t total = (int64_t)w * w;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / w), r = (int)(e % w);
    dst[e] = r <= c ? src[(int64_t)c * lds + r] : 0.0;
  }
}

__global__ void diag_copy_kernel(int w, const double* __restrict__ G, double* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < w) d[i] = G[(int64_t)i * w + i];
}

// Vtop[:, r] = V[:, w-1-r] * sqrt(max(theta[w-1-r], 0)); theta_top[r] = theta[w-1-r]
__global__ void top_eigvecs_kernel(int w, int k, const double* __restrict__ V, const double* __restrict__ theta,
                                   double* __restrict__ Vtop, double* __restrict__ theta_top) {
  const int64_t total = (int64_t)w * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / w), i = (int)(e % w);
    const int src = w - 1 - r;
    const double th = theta[src];
    Vtop[e] = V[(int64_t)src * w + i] * sqrt(fmax(th, 0.0));
    if (i == 0) theta_top[r] = th;
  }
}

// base = max(diag - sum_r A^2, floor), sqrt_base, At = A / sqrt_base  (A col-major n x k)
// 32 rows per block, the 8 warps split the k columns; lanes walk adjacent rows (coalesced)
__global__ void __launch_bounds__(256) base_kernel(int64_t n, int k, const double* __restrict__ diag, double floor_v,
                                                   double* __restrict__ A, double* __restrict__ base,
                                                   double* __restrict__ sqrt_base) {
  __shared__ double part[8][33];
  __shared__ double sbs[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < n)
    for (int r = wid; r < k; r += 8) {
      const double a = A[(int64_t)r * n + i];
      s = fma(a, a, s);
    }
  part[wid][lane] = s;
  __syncthreads();
  if (wid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    double sb = 1.0;
    if (i < n) {
      const double b = fmax(diag[i] - t, floor_v);
      sb = sqrt(b);
      base[i] = b;
      sqrt_base[i] = sb;
    }
    sbs[lane] = sb;
  }
  __syncthreads();
  if (i < n) {
    const double inv = sbs[lane];
    for (int r = wid; r < k; r += 8) A[(int64_t)r * n + i] /= inv;
  }
}

__global__ void __launch_bounds__(RB) sum_log_partial(int64_t n, const double* __restrict__ v, int64_t chunk,
                                                      double* __restrict__ partial) {
  __shared__ double red[RB / 32];
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min64(n, j0 + chunk);
  double s = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += RB) s += log(v[j]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void sum_final(int P, const double* __restrict__ partial, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int p = 0; p < P; ++p) s += partial[p];
    *out = s;
  }
}

__global__ void add_identity_kernel(int k, double* __restrict__ C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) C[(int64_t)i * k + i] += 1.0;
}

// 2 sum log diag(L) of the inner Cholesky (src/precond.py:77-80); NotPD on failure
__global__ void chol_logdet_kernel(int k, const double* __restrict__ L, const int* __restrict__ info,
                                   double* __restrict__ out, int* __restrict__ flags) {
  // one warp: lane-strided logs of the diagonal, then a shuffle reduction
  double s = 0.0;
  for (int i = threadIdx.x; i < k; i += 32) s += log(L[(int64_t)i * k + i]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) {
    if (*info != 0) atomicOr(flags, RLD_FLAG_NOT_PD);
    *out = 2.0 * s;
  }
}

// keep filter and spectral factors of (I + At^T At) (src/precond.py:96-99):
// scale_m = 1/sqrt(lam_m) for kept m else 0; h = 1/(1+lam)-1 (P^-1), g = 1/sqrt(1+lam)-1 (N^-T),
// gam = sqrt(1+lam)-1 (N); W columns scaled in place.
__global__ void sqrt_factor_kernel(int k, double keep_rtol, const double* __restrict__ lam, double* __restrict__ W,
                                   double* __restrict__ h, double* __restrict__ g, double* __restrict__ gam,
                                   int* __restrict__ kept) {
  const double lmax = (k > 0) ? lam[k - 1] : 0.0;
  const double thr = keep_rtol * fmax(lmax, 1.0);
  for (int m = blockIdx.x; m < k; m += gridDim.x) {
    const double l = lam[m];
    const bool keep = l > thr;
    const double sc = keep ? 1.0 / sqrt(l) : 0.0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) W[(int64_t)m * k + i] *= sc;
    if (threadIdx.x == 0) {
      h[m] = keep ? 1.0 / (1.0 + l) - 1.0 : 0.0;
      g[m] = keep ? 1.0 / sqrt(1.0 + l) - 1.0 : 0.0;
      gam[m] = keep ? sqrt(1.0 + l) - 1.0 : 0.0;
      if (keep) atomicAdd(kept, 1);
    }
  }
}

__global__ void diag_of_dense_kernel(int64_t rows, int64_t row0, const void* __restrict__ K, int64_t ldk,
                                     int dtype, double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t off = i * ldk + (row0 + i);
  d[i] = dtype == RLD_FP64 ? static_cast<const double*>(K)[off] : (double)static_cast<const float*>(K)[off];
}

__global__ void convert_kernel(const void* __restrict__ src, int sdt, void* __restrict__ dst, int ddt,
                               int64_t count) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = sdt == RLD_FP64 ? static_cast<const double*>(src)[e] : (double)static_cast<const float*>(src)[e];
    if (ddt == RLD_FP64)
      static_cast<double*>(dst)[e] = v;
    else
      static_cast<float*>(dst)[e] = (float)v;
  }
}

__global__ void convert_2d_kernel(const void* __restrict__ src, int sdt, int64_t lds, double* __restrict__ dst,
                                  int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    dst[e] = sdt == RLD_FP64 ? static_cast<const double*>(src)[r * lds + c]
                             : (double)static_cast<const float*>(src)[r * lds + c];
  }
}

__global__ void sqrt_into_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ sb,
                                 int* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = b[i];
  if (!(v > 0.0)) atomicOr(flags, RLD_FLAG_BAD_BASE);
  sb[i] = sqrt(v);
}

__global__ void __launch_bounds__(RB) strided_log_partial(int64_t count, const double* __restrict__ v,
                                                          int64_t stride, int64_t chunk,
                                                          double* __restrict__ partial) {
  __shared__ double red[RB / 32];
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min64(count, j0 + chunk);
  double s = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += RB) s += log(v[j * stride]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

}  // namespace

void convert_rows(const void* src, int sdt, void* dst, int ddt, int64_t count, cudaStream_t st) {
  if (count <= 0) return;
  convert_kernel<<<grid_for(count), 256, 0, st>>>(src, sdt, dst, ddt, count);
  RLD_LAUNCH_CHECK();
}
void convert_rows_2d(const void* src, int sdt, int64_t lds, double* dst, int64_t rows, int64_t cols,
                     cudaStream_t st) {
  if (rows * cols <= 0) return;
  convert_2d_kernel<<<grid_for(rows * cols), 256, 0, st>>>(src, sdt, lds, dst, rows, cols);
  RLD_LAUNCH_CHECK();
}
void sqrt_into(int64_t n, const double* base, double* sqrt_base, int* flags, cudaStream_t st) {
  if (n <= 0) return;
  sqrt_into_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, base, sqrt_base, flags);
  RLD_LAUNCH_CHECK();
}
void strided_sum_log(int64_t count, const double* v, int64_t stride, double* out, DevBuf& scratch,
                     cudaStream_t st) {
  int P = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(count, 4 * RB)), 1184);
  const int64_t chunk = ceil_div(count, P);
  P = (int)ceil_div(count, chunk);
  scratch.reserve(sizeof(double) * P);
  strided_log_partial<<<P, RB, 0, st>>>(count, v, stride, chunk, scratch.as<double>());
  RLD_LAUNCH_CHECK();
  sum_final<<<1, 32, 0, st>>>(P, scratch.as<double>(), out);
  RLD_LAUNCH_CHECK();
}

void cholqr_check(int w, const double* R, const double* gdiag, const int* info, double rtol, int* flags,
                  cudaStream_t st) {
  cholqr_check_kernel<<<(unsigned)ceil_div(std::max(w, 1), 128), 128, 0, st>>>(w, R, gdiag, info, rtol, flags);
  RLD_LAUNCH_CHECK();
}
void copy_upper(int w, const double* src, int64_t lds, double* dst, cudaStream_t st) {
  const int64_t total = (int64_t)w * w;
  copy_upper_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 1024), 256, 0, st>>>(w, src, lds, dst);
  RLD_LAUNCH_CHECK();
}

void householder_check(int w, const double* R, int64_t ldr, const double* norms2, double rtol, double* sgn,
                       int* flags, cudaStream_t st) {
  householder_check_kernel<<<(unsigned)ceil_div(std::max(w, 1), 128), 128, 0, st>>>(w, R, ldr, norms2, rtol, sgn,
                                                                                   flags);
  RLD_LAUNCH_CHECK();
}
void diag_copy(int w, const double* G, double* d, cudaStream_t st) {
  diag_copy_kernel<<<(unsigned)ceil_div(std::max(w, 1), 128), 128, 0, st>>>(w, G, d);
  RLD_LAUNCH_CHECK();
}
void top_eigvecs(int w, int k, const double* V, const double* theta, double* Vtop, double* theta_top,
                 cudaStream_t st) {
  top_eigvecs_kernel<<<grid_for((int64_t)w * k), 256, 0, st>>>(w, k, V, theta, Vtop, theta_top);
  RLD_LAUNCH_CHECK();
}
void precond_base(int64_t n, int k, const double* diag, double floor_v, double* A, double* base, double* sqrt_base,
                  cudaStream_t st) {
  if (n <= 0) return;   // a rank without rows
  base_kernel<<<(unsigned)ceil_div(n, 32), 256, 0, st>>>(n, k, diag, floor_v, A, base, sqrt_base);
  RLD_LAUNCH_CHECK();
}
void sum_log(int64_t n, const double* v, double* out, DevBuf& scratch, cudaStream_t st) {
  int P = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(n, 4 * RB)), 1184);
  const int64_t chunk = ceil_div(n, P);
  P = (int)ceil_div(n, chunk);
  scratch.reserve(sizeof(double) * P);
  sum_log_partial<<<P, RB, 0, st>>>(n, v, chunk, scratch.as<double>());
  RLD_LAUNCH_CHECK();
  sum_final<<<1, 32, 0, st>>>(P, scratch.as<double>(), out);
  RLD_LAUNCH_CHECK();
}
void add_identity(int k, double* C, cudaStream_t st) {
  add_identity_kernel<<<(unsigned)ceil_div(std::max(k, 1), 128), 128, 0, st>>>(k, C);
  RLD_LAUNCH_CHECK();
}
void chol_logdet(int k, const double* L, const int* info, double* out, int* flags, cudaStream_t st) {
  chol_logdet_kernel<<<1, 32, 0, st>>>(k, L, info, out, flags);
  RLD_LAUNCH_CHECK();
}
void sqrt_factors(int k, double keep_rtol, const double* lam, double* W, double* h, double* g, double* gam,
                  int* kept, cudaStream_t st) {
  if (k <= 0) return;
  sqrt_factor_kernel<<<std::min(k, 1024), 128, 0, st>>>(k, keep_rtol, lam, W, h, g, gam, kept);
  RLD_LAUNCH_CHECK();
}
namespace {
// coordinate-major split points [8][ldp]: row k = fp32(x_k) (hi), row 4 + k = fp32(x_k - hi) (lo)
// Float32 points for the on-the-fly tensor-core tiles in k-step blocks
// P[ceil(n/32)][8][32]: rows 0-3 hold x_k * scale (zero for k >= d), rows 4-7 and
// the padding columns are zero (the buffer is cleared first).
__global__ void pad_points_kernel(const double* __restrict__ X, int64_t n, int d, double scale,
                                  float* __restrict__ P) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 4 * n) return;
  const int64_t i = e >> 2;
  const int k = (int)(e & 3);
  const double x = k < d ? X[i * d + k] : 0.0;
  P[(((i >> 5) * 8 + k) << 5) + (i & 31)] = (float)(x * scale);
}
}  // namespace

namespace {
__global__ void relayout_kernel(const double* __restrict__ src, int64_t m, int64_t L, int64_t n,
                                double* __restrict__ dst) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, j = e % n;
    const int64_t g = j / L, jj = j - g * L;
    dst[e] = src[(g * m + c) * L + jj];
  }
}
}  // namespace

void relayout_gathered(const double* src, int G, int64_t m, int64_t L, int64_t n, double* dst, cudaStream_t st) {
  (void)G;
  if (m * n <= 0) return;
  relayout_kernel<<<grid_for(m * n), 256, 0, st>>>(src, m, L, n, dst);
  RLD_LAUNCH_CHECK();
}

namespace {
__global__ void sum_blocks_kernel(int64_t nb, int64_t count, const double* __restrict__ in, double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nb; ++b) s += in[b * count + e];
    out[e] = s;
  }
}
}  // namespace

namespace {
// rows r0 .. r0 + nr - 1 (r0 multiple of 128) of row-major fp32 src (row stride lds) into the tiled layout
__global__ void tile_rows_kernel(const float* __restrict__ src, int64_t lds, int64_t r0, int64_t nr, int64_t n,
                                 float* __restrict__ Kt) {
  const int64_t ks = (n + 31) >> 5;
  const int64_t total = nr * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, j = e % n, i = r0 + r;
    Kt[(((i >> 7) * ks + (j >> 5)) << 12) + ((i & 127) << 5) + (j & 31)] = src[r * lds + j];
  }
}
__global__ void untile_kernel(const float* __restrict__ Kt, int64_t rows, int64_t n, double* __restrict__ out,
                              int64_t ldo) {
  const int64_t ks = (n + 31) >> 5;
  const int64_t total = rows * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    out[i * ldo + j] = (double)Kt[(((i >> 7) * ks + (j >> 5)) << 12) + ((i & 127) << 5) + (j & 31)];
  }
}
__global__ void diag_of_tiled_kernel(int64_t rows, int64_t row0, int64_t n, const float* __restrict__ Kt,
                                     double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t ks = (n + 31) >> 5, j = row0 + i;
  d[i] = (double)Kt[(((i >> 7) * ks + (j >> 5)) << 12) + ((i & 127) << 5) + (j & 31)];
}
}  // namespace

void tile_rows(const float* src, int64_t lds, int64_t r0, int64_t nr, int64_t n, float* Kt, cudaStream_t st) {
  if (nr <= 0) return;
  tile_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nr * n, 256), 148 * 16), 256, 0, st>>>(src, lds, r0, nr, n,
                                                                                                Kt);
  RLD_LAUNCH_CHECK();
}
void untile_to_f64(const float* Kt, int64_t rows, int64_t n, double* out, int64_t ldo, cudaStream_t st) {
  untile_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * n, 256), 148 * 16), 256, 0, st>>>(Kt, rows, n, out, ldo);
  RLD_LAUNCH_CHECK();
}
void diag_of_tiled(int64_t rows, int64_t row0, int64_t n, const float* Kt, double* d, cudaStream_t st) {
  if (rows <= 0) return;
  diag_of_tiled_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, row0, n, Kt, d);
  RLD_LAUNCH_CHECK();
}

namespace {
// base = scale (the "-scaled" kinds, src/precond.py:260-261, 266), sqrt_base, At = A / sqrt(scale)
__global__ void base_scaled_kernel(int64_t n, int k, double scale, double* __restrict__ A, double* __restrict__ base,
                                   double* __restrict__ sqrt_base) {
  const double sb = sqrt(scale), inv = 1.0 / sb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * (int64_t)(k + 1);
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n) {
      base[e] = scale;
      sqrt_base[e] = sb;
    } else {
      A[e - n] *= inv;
    }
  }
}

// first largest entry of d[0..n) (np.argmax tie rule: smallest index), one block per chunk then a final pick;
// out[0] = value, out[1] = global index (row0 + i) as double
// key of index j for first-max ties: j itself, or (points stored in a locality order) the original
// index perm[j], so the pivot is the reference's np.argmax one
__device__ __forceinline__ int64_t amax_key(const int* perm, int64_t j) { return perm ? (int64_t)perm[j] : j; }

__global__ void argmax_partial_kernel(int64_t n, const double* __restrict__ d, int64_t chunk,
                                      double* __restrict__ part, const int* __restrict__ perm) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min64(n, j0 + chunk);
  double bv = -INFINITY;
  int64_t bi = -1;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const double v = d[j];
    if (v > bv || (perm && v == bv && amax_key(perm, j) < amax_key(perm, bi))) { bv = v; bi = j; }   // first max
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int64_t i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 >= 0 &&
                                    (si[threadIdx.x] < 0 || amax_key(perm, i2) < amax_key(perm, si[threadIdx.x])))) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sv[0];
    part[2 * blockIdx.x + 1] = (double)si[0];
  }
}
__global__ void argmax_final_kernel(int P, const double* __restrict__ part, int64_t offset, double* __restrict__ out,
                                    const int* __restrict__ perm) {
  double bv = -INFINITY, bi = -1.0;
  for (int b = 0; b < P; ++b) {   // pairs in increasing index order: strict > keeps the first max
    const double v = part[2 * b], i = part[2 * b + 1];
    if (i >= 0 && (v > bv || (perm && v == bv && bi >= 0 && perm[(int64_t)i] < perm[(int64_t)bi]))) { bv = v; bi = i; }
  }
  out[0] = bv;
  out[1] = bi >= 0 ? bi + (double)offset : -1.0;
}

// column p of K for the local rows (K symmetric: K[row0 + i, p]) from the resident form
__global__ void kernel_column_kernel(int64_t rows, int64_t row0, int64_t n, int64_t p, const void* __restrict__ K,
                                     int64_t ldk, int kdtype, int tiled, const double* __restrict__ X,
                                     KernelParams kp, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double v;
  if (K == nullptr) {   // from the points (src/kernels.py:40-46, 72)
    if (row0 + i == p) {
      v = kp.diag;
    } else {
      double r2 = 0.0;
      for (int c = 0; c < kp.d; ++c) {
        const double df = X[(row0 + i) * kp.d + c] - X[p * kp.d + c];
        r2 = fma(df, df, r2);
      }
      v = kernel_value_f64(kp, r2);
    }
  } else if (tiled) {
    const int64_t ks = (n + 31) >> 5;
    v = (double)static_cast<const float*>(K)[(((i >> 7) * ks + (p >> 5)) << 12) + ((i & 127) << 5) + (p & 31)];
  } else if (kdtype == RLD_FP64) {
    v = static_cast<const double*>(K)[i * ldk + p];
  } else {
    v = (double)static_cast<const float*>(K)[i * ldk + p];
  }
  out[i] = v;
}

// partial-Cholesky column j (src/precond.py:215-228): C[:, j] = col / sqrt(dp); d -= C[:, j]^2
__global__ void pchol_update_kernel(int64_t rows, const double* __restrict__ col, const double* __restrict__ dp,
                                    double* __restrict__ Cj, double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double c = col[i] / sqrt(dp[0]);
  Cj[i] = c;
  d[i] -= c * c;
}

// C[p, 0..j) of the owner rank's rows, zeros elsewhere (then all-reduced)
__global__ void row_of_owner_kernel(int64_t rows, int64_t row0, const double* __restrict__ pv, const double* __restrict__ C,
                                    int j, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= j) return;
  const int64_t p = (int64_t)pv[1] - row0;
  out[c] = (p >= 0 && p < rows) ? C[(int64_t)c * rows + p] : 0.0;
}

__global__ void scale_by_kernel(int64_t n, double* __restrict__ v, const double* __restrict__ f, int mode) {
  // mode 0: v *= 1/sqrt(f[0]) ; mode 1: v *= sqrt(max(f[0], 1e-12))
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  v[i] *= mode == 0 ? 1.0 / sqrt(f[0]) : sqrt(fmax(f[0], 1e-12));
}
}  // namespace

void precond_base_scaled(int64_t n, int k, double scale, double* A, double* base, double* sqrt_base,
                         cudaStream_t st) {
  base_scaled_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n * (k + 1), 256), 148 * 16), 256, 0, st>>>(
      n, k, scale, A, base, sqrt_base);
  RLD_LAUNCH_CHECK();
}
void argmax_first(int64_t n, const double* d, int64_t offset, double* out, DevBuf& scratch, cudaStream_t st,
                  const int* perm) {
  int P = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 2048), 512));
  const int64_t chunk = ceil_div(std::max<int64_t>(n, 1), P);
  P = (int)ceil_div(std::max<int64_t>(n, 1), chunk);
  scratch.reserve(sizeof(double) * 2 * P);
  argmax_partial_kernel<<<P, 256, 0, st>>>(n, d, chunk, scratch.as<double>(), perm);
  RLD_LAUNCH_CHECK();
  argmax_final_kernel<<<1, 1, 0, st>>>(P, scratch.as<double>(), offset, out, perm);
  RLD_LAUNCH_CHECK();
}
void pick_first_max(int P, const double* pairs, double* out, cudaStream_t st, const int* perm) {
  argmax_final_kernel<<<1, 1, 0, st>>>(P, pairs, 0, out, perm);
  RLD_LAUNCH_CHECK();
}
void kernel_column(int64_t rows, int64_t row0, int64_t n, int64_t p, const void* K, int64_t ldk, int kdtype,
                   bool tiled, const double* X, const KernelParams& kp, double* out, cudaStream_t st) {
  if (rows <= 0) return;
  kernel_column_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, row0, n, p, K, ldk, kdtype, tiled ? 1 : 0,
                                                                      X, kp, out);
  RLD_LAUNCH_CHECK();
}
void pchol_update(int64_t rows, const double* col, const double* dp, double* Cj, double* d, cudaStream_t st) {
  if (rows <= 0) return;
  pchol_update_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, col, dp, Cj, d);
  RLD_LAUNCH_CHECK();
}
void row_of_owner(int64_t rows, int64_t row0, const double* pv, const double* C, int j, double* out,
                  cudaStream_t st) {
  if (j <= 0) return;
  row_of_owner_kernel<<<(unsigned)ceil_div(j, 128), 128, 0, st>>>(rows, row0, pv, C, j, out);
  RLD_LAUNCH_CHECK();
}
void scale_by(int64_t n, double* v, const double* f, int mode, cudaStream_t st) {
  if (n <= 0) return;
  scale_by_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, v, f, mode);
  RLD_LAUNCH_CHECK();
}

void sum_blocks(int64_t nb, int64_t count, const double* in, double* out, cudaStream_t st) {
  if (count <= 0) return;
  sum_blocks_kernel<<<(unsigned)std::min<int64_t>(ceil_div(count, 256), 148 * 8), 256, 0, st>>>(nb, count, in, out);
  RLD_LAUNCH_CHECK();
}

void pad_points(const double* X, int64_t n, int d, double scale, float* pts8, cudaStream_t st) {
  RLD_CUDA(cudaMemsetAsync(pts8, 0, sizeof(float) * otf_points_floats(n), st));
  pad_points_kernel<<<(unsigned)ceil_div(4 * n, 256), 256, 0, st>>>(X, n, d, scale, pts8);
  RLD_LAUNCH_CHECK();
}

void diag_of_dense(int64_t rows, int64_t row0, const void* K, int64_t ldk, int dtype, double* d, cudaStream_t st) {
  diag_of_dense_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rows, row0, K, ldk, dtype, d);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld

namespace rld {
namespace {
// dst[c * ldd + i] = src[c * lds + perm[i]] (gather) or dst[c * ldd + perm[i]] = src[c * lds + i] (scatter)
__global__ void permute_rows_kernel(int64_t m, int64_t n, const int* __restrict__ perm, const double* __restrict__ src,
                                    int64_t lds, double* __restrict__ dst, int64_t ldd, int scatter) {
  const int64_t c = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = perm[i];
    if (scatter) dst[c * ldd + j] = src[c * lds + i];
    else dst[c * ldd + i] = src[c * lds + j];
  }
}
}  // namespace

void permute_rows(int64_t m, int64_t n, const int* perm, const double* src, int64_t lds, double* dst, int64_t ldd,
                  bool scatter, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  const dim3 g((unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), (unsigned)m);
  permute_rows_kernel<<<g, 256, 0, st>>>(m, n, perm, src, lds, dst, ldd, scatter ? 1 : 0);
  RLD_LAUNCH_CHECK();
}
}  // namespace rld

namespace rld {
namespace {
// per-dimension bounding box of n points (one block): box[c] = min, box[4 + c] = max
__global__ void morton_box_kernel(const double* __restrict__ X, int64_t n, int d, double* __restrict__ box) {
  __shared__ double lo[4][32], hi[4][32];
  double l[4], h[4];
  for (int c = 0; c < 4; ++c) {
    l[c] = INFINITY;
    h[c] = -INFINITY;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int c = 0; c < d; ++c) {
      const double x = X[i * d + c];
      l[c] = fmin(l[c], x);
      h[c] = fmax(h[c], x);
    }
  for (int c = 0; c < 4; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      l[c] = fmin(l[c], __shfl_xor_sync(0xffffffffu, l[c], o));
      h[c] = fmax(h[c], __shfl_xor_sync(0xffffffffu, h[c], o));
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int c = 0; c < 4; ++c) {
      lo[c][w] = l[c];
      hi[c][w] = h[c];
    }
  __syncthreads();
  if (threadIdx.x < 4) {
    double a = INFINITY, b = -INFINITY;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a = fmin(a, lo[threadIdx.x][k]);
      b = fmax(b, hi[threadIdx.x][k]);
    }
    box[threadIdx.x] = a;
    box[4 + threadIdx.x] = b;
  }
}

// Z-curve code: 63 / d bits per coordinate over the box, interleaved
__global__ void morton_code_kernel(const double* __restrict__ X, int64_t n, int d, const double* __restrict__ box,
                                   unsigned long long* __restrict__ code, int* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = 63 / d;
  const double top = ldexp(1.0, b) - 1.0;
  unsigned long long k = 0;
  for (int c = 0; c < d; ++c) {
    const double span = box[4 + c] - box[c];
    const double f = span > 0 ? (X[i * d + c] - box[c]) / span : 0.0;
    const unsigned long long q = (unsigned long long)fmin(top, fmax(0.0, floor(f * top)));
    for (int bit = 0; bit < b; ++bit) k |= ((q >> bit) & 1ull) << (bit * d + c);
  }
  code[i] = k;
  idx[i] = (int)i;
}

__global__ void gather_points_kernel(const double* __restrict__ X, int64_t n, int d, const int* __restrict__ perm,
                                     double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const int64_t i = e / d;
  out[e] = X[(int64_t)perm[i] * d + (e - i * d)];
}
}  // namespace

// Morton (Z-curve) order of n device points (d <= 3), stable: perm[i] = original index of point i;
// Xs = the points in that order.  scratch holds the codes.
void morton_order_device(const double* X, int64_t n, int d, int* perm, double* Xs, DevBuf& scratch, cudaStream_t st) {
  scratch.reserve(sizeof(unsigned long long) * (n + 1) + sizeof(double) * 8);
  double* box = scratch.as<double>();
  unsigned long long* code = reinterpret_cast<unsigned long long*>(box + 8);
  morton_box_kernel<<<1, 1024, 0, st>>>(X, n, d, box);
  RLD_LAUNCH_CHECK();
  morton_code_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(X, n, d, box, code, perm);
  RLD_LAUNCH_CHECK();
  thrust::stable_sort_by_key(thrust::cuda::par.on(st), thrust::device_pointer_cast(code),
                             thrust::device_pointer_cast(code + n), thrust::device_pointer_cast(perm));
  gather_points_kernel<<<(unsigned)ceil_div(n * d, 256), 256, 0, st>>>(X, n, d, perm, Xs);
  RLD_LAUNCH_CHECK();
}
}  // namespace rld
