// Matrix-free float64 K x V for the CPU oracle.
//
// TEST INFRASTRUCTURE ONLY (see oracle/rstar_oracle.py): the checker the GPU path is compared
// against at BASELINE sizes where the reference's dense K does not fit in host RAM
// (n = 65536 / 262144 / 2^20).  Never linked into, or called by, the product library.
//
// What it restates (reference paths relative to /root/reference/pkg/src/ratlogdet/):
//   * build_covariance (kernels.py:59-73): r^2 = (|x_i|^2 + |x_j|^2) - 2 x_i.x_j (exactly
//     symmetric here: x_i.x_j is one fused multiply-add per coordinate in coordinate order, the
//     order OpenBLAS's dgemm uses for X X^T in all but ~0.5 % of entries), clamped at 0,
//     r = sqrt(r^2); the diagonal is amplitude^2 + jitter (kernels.py:72);
//   * _kernel_of_r (kernels.py:40-46): RBF a^2 exp(-(r r) / (2 l l)),
//     Matern-5/2 a^2 (1 + u + u u / 3) exp(-u) with u = sqrt(5) r / l (same operation order;
//     exp from glibc's libmvec, <= 4 ulp);
//   * the operator product M @ y of estimators.py:72 / precond.py:186, 189, for a block of
//     vectors at once.
// K is never stored: every OpenMP thread owns a block of output rows and walks the columns in
// fixed chunks.  Narrow blocks (m <= 16, the Lanczos shape) are contracted in registers as the
// entries are generated; wide blocks (the sketch) write the tile and multiply it into the block
// with a single-threaded float64 GEMM from numpy's OpenBLAS (dlopen'ed; a plain loop if no BLAS
// is found).  The summation order is fixed, so results do not depend on the thread count.
//
// Build: oracle/mf.py build() -- two variants, x86-64-v3 (AVX2) and x86-64-v4 (AVX-512),
// picked at load time by the host's CPU flags.
#include <dlfcn.h>
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#if defined(__AVX512F__)
typedef __m512d vd;
constexpr int W = 8;
extern "C" __m512d _ZGVeN8v_exp(__m512d);
static inline vd vset(double x) { return _mm512_set1_pd(x); }
static inline vd vload(const double* p) { return _mm512_loadu_pd(p); }
static inline void vstore(double* p, vd v) { _mm512_storeu_pd(p, v); }
static inline vd vfma(vd a, vd b, vd c) { return _mm512_fmadd_pd(a, b, c); }
static inline vd vadd(vd a, vd b) { return _mm512_add_pd(a, b); }
static inline vd vsub(vd a, vd b) { return _mm512_sub_pd(a, b); }
static inline vd vmul(vd a, vd b) { return _mm512_mul_pd(a, b); }
static inline vd vdiv(vd a, vd b) { return _mm512_div_pd(a, b); }
static inline vd vsqrt(vd a) { return _mm512_sqrt_pd(a); }
static inline vd vmax0(vd a) { return _mm512_max_pd(a, _mm512_setzero_pd()); }
static inline vd vexp(vd a) { return _ZGVeN8v_exp(a); }
#else
typedef __m256d vd;
constexpr int W = 4;
extern "C" __m256d _ZGVdN4v_exp(__m256d);
static inline vd vset(double x) { return _mm256_set1_pd(x); }
static inline vd vload(const double* p) { return _mm256_loadu_pd(p); }
static inline void vstore(double* p, vd v) { _mm256_storeu_pd(p, v); }
static inline vd vfma(vd a, vd b, vd c) { return _mm256_fmadd_pd(a, b, c); }
static inline vd vadd(vd a, vd b) { return _mm256_add_pd(a, b); }
static inline vd vsub(vd a, vd b) { return _mm256_sub_pd(a, b); }
static inline vd vmul(vd a, vd b) { return _mm256_mul_pd(a, b); }
static inline vd vdiv(vd a, vd b) { return _mm256_div_pd(a, b); }
static inline vd vsqrt(vd a) { return _mm256_sqrt_pd(a); }
static inline vd vmax0(vd a) { return _mm256_max_pd(a, _mm256_setzero_pd()); }
static inline vd vexp(vd a) { return _ZGVdN4v_exp(a); }
#endif

namespace {

typedef void (*dgemm_fn)(int layout, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
                         const double* B, int ldb, double beta, double* C, int ldc);
typedef void (*setthreads_fn)(int);
dgemm_fn g_dgemm = nullptr;
constexpr int ROW_MAJOR = 101, NO_TRANS = 111, TRANS = 112;
constexpr int MAXD = 32, FUSED_M = 16;

constexpr double SQRT5 = 2.23606797749979;   // np.sqrt(5.0), kernels.py:14

struct Spec {
  int family;   // 0 = rbf, 1 = matern52
  double a2, ell, two_ll, diag;
  double pert = 0.0;   // perturbation screen: K_ij (1 + pert h(i, j)), h symmetric in [-1, 1)
};

// symmetric hash of (i, j) to [-1, 1) (splitmix64 finaliser)
static inline double sym_hash(int64_t i, int64_t j) {
  uint64_t a = (uint64_t)(i < j ? i : j), b = (uint64_t)(i < j ? j : i);
  uint64_t z = (a << 32) ^ b ^ 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// |x|^2 as numpy's np.sum(points * points, axis=1): a plain loop below 8 terms, numpy's
// 8-accumulator pairwise block from 8 to 128 terms.
double sqnorm(const double* x, int d) {
  if (d < 8) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) s += x[k] * x[k];
    return s;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = x[k] * x[k];
  int k = 8;
  for (; k + 8 <= d; k += 8)
    for (int q = 0; q < 8; ++q) r[q] += x[k + q] * x[k + q];
  double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; k < d; ++k) s += x[k] * x[k];
  return s;
}

// Column chunk in structure-of-arrays form: coordinate k of column j at xs[k * Cp + j], the
// squared norms at sq[j]; padded to a multiple of W with copies of the last column.
struct Chunk {
  int C = 0, Cp = 0;
  std::vector<double> xs, sq;
  void load(const double* X, const double* sqall, int d, int64_t j0, int c) {
    C = c;
    Cp = (c + W - 1) / W * W;
    xs.resize((size_t)d * Cp);
    sq.resize(Cp);
    for (int j = 0; j < Cp; ++j) {
      const int64_t jj = j0 + std::min(j, c - 1);
      for (int k = 0; k < d; ++k) xs[(size_t)k * Cp + j] = X[jj * d + k];
      sq[j] = sqall[jj];
    }
  }
};

// W entries K[i, j..j+W) (off-diagonal formula; the caller patches the diagonal)
static inline vd entries(const Spec& sp, const double* xi, double sqi, const Chunk& ch, int d, int j) {
  vd g = vset(0.0);
  for (int k = 0; k < d; ++k) g = vfma(vset(xi[k]), vload(&ch.xs[(size_t)k * ch.Cp + j]), g);
  // r2 = (sq_i + sq_j) - 2 g, clamped at 0
  const vd r2 = vmax0(vsub(vadd(vset(sqi), vload(&ch.sq[j])), vmul(vset(2.0), g)));
  const vd r = vsqrt(r2);
  if (sp.family == 0) {   // a2 * exp(-(r * r) / (2 l l))
    const vd arg = vdiv(vsub(vset(0.0), vmul(r, r)), vset(sp.two_ll));
    return vmul(vset(sp.a2), vexp(arg));
  }
  // u = sqrt5 r / l ; a2 (1 + u + u u / 3) exp(-u)
  const vd u = vdiv(vmul(vset(SQRT5), r), vset(sp.ell));
  const vd e = vexp(vsub(vset(0.0), u));
  const vd poly = vadd(vadd(vset(1.0), u), vdiv(vmul(u, u), vset(3.0)));
  return vmul(vmul(vset(sp.a2), poly), e);
}

}  // namespace

extern "C" {

// Load a CBLAS dgemm from `path` (numpy / scipy OpenBLAS), 1 thread per call.  Returns 1 on success.
int mf_init(const char* path, const char* dgemm_sym, const char* threads_sym) {
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return 0;
  g_dgemm = (dgemm_fn)dlsym(h, dgemm_sym);
  setthreads_fn st = threads_sym ? (setthreads_fn)dlsym(h, threads_sym) : nullptr;
  if (st) st(1);
  return g_dgemm != nullptr;
}

int mf_threads(void) { return omp_get_max_threads(); }
int mf_simd_width(void) { return W; }

// Y = K[row0 : row0 + rows, :] V for m vectors.
//   X: n x d points (row-major).  V: m x n, vectors as rows (ld ldv >= n).
//   Y: m x rows, vectors as rows (ld ldy >= rows).
// family 0 = rbf, 1 = matern52.
int mf_kv(int family, double amplitude, double ell, double jitter, const double* X, int64_t n, int d, int64_t row0,
          int64_t rows, const double* V, int64_t m, int64_t ldv, double* Y, int64_t ldy, int rb, int cb,
          double pert) {
  if (n < 1 || d < 1 || d > MAXD || m < 1 || rows < 0 || row0 < 0 || row0 + rows > n) return 1;
  Spec sp;
  sp.pert = pert;
  sp.family = family;
  sp.a2 = amplitude * amplitude;   // spec.amplitude**2
  sp.ell = ell;
  sp.two_ll = 2.0 * ell * ell;
  sp.diag = sp.a2 + jitter;
  std::vector<double> sq(n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) sq[i] = sqnorm(X + i * d, d);
  if (rb < 1) rb = 64;
  if (cb < 1) cb = 1024;
  cb = (cb + W - 1) / W * W;
  const bool fused = m <= FUSED_M;
  const int64_t nblk = (rows + rb - 1) / rb;
#pragma omp parallel
  {
    Chunk ch;
    std::vector<double> T(fused ? 0 : (size_t)rb * cb), Yb((size_t)rb * m);
    alignas(64) double lanes[W];
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < nblk; ++b) {
      const int64_t i0 = row0 + b * rb;
      const int R = (int)std::min<int64_t>(rb, row0 + rows - i0);
      std::fill(Yb.begin(), Yb.begin() + (size_t)R * m, 0.0);
      for (int64_t j0 = 0; j0 < n; j0 += cb) {
        const int C = (int)std::min<int64_t>(cb, n - j0);
        ch.load(X, sq.data(), d, j0, C);
        for (int i = 0; i < R; ++i) {
          const int64_t gi = i0 + i;
          const double* xi = X + gi * d;
          const bool diag_here = gi >= j0 && gi < j0 + C;
          if (fused) {
            vd acc[FUSED_M];
            for (int c = 0; c < m; ++c) acc[c] = vset(0.0);
            for (int j = 0; j < ch.Cp; j += W) {
              vd kv = entries(sp, xi, sq[gi], ch, d, j);
              if (j + W > C || (diag_here && gi - j0 >= j && gi - j0 < j + W) || sp.pert != 0.0) {
                vstore(lanes, kv);
                for (int l = 0; l < W; ++l) {
                  if (j + l >= C) lanes[l] = 0.0;
                  else if (j0 + j + l == gi) lanes[l] = sp.diag;
                  if (sp.pert != 0.0 && j + l < C) lanes[l] *= 1.0 + sp.pert * sym_hash(gi, j0 + j + l);
                }
                kv = vload(lanes);
              }
              for (int c = 0; c < m; ++c) {
                const double* vc = V + c * ldv + j0 + j;
                vd v;
                if (j + W <= C) {
                  v = vload(vc);
                } else {
                  for (int l = 0; l < W; ++l) lanes[l] = j + l < C ? vc[l] : 0.0;
                  v = vload(lanes);
                }
                acc[c] = vfma(kv, v, acc[c]);
              }
            }
            for (int c = 0; c < m; ++c) {
              vstore(lanes, acc[c]);
              double s = 0.0;
              for (int l = 0; l < W; ++l) s += lanes[l];
              Yb[(size_t)i * m + c] += s;
            }
          } else {
            double* row = T.data() + (size_t)i * C;
            for (int j = 0; j < ch.Cp; j += W) {
              vstore(lanes, entries(sp, xi, sq[gi], ch, d, j));
              const int L = std::min(W, C - j);
              for (int l = 0; l < L; ++l) row[j + l] = (j0 + j + l == gi) ? sp.diag : lanes[l];
              if (sp.pert != 0.0)
                for (int l = 0; l < L; ++l) row[j + l] *= 1.0 + sp.pert * sym_hash(gi, j0 + j + l);
            }
          }
        }
        if (!fused) {
          const double* Vc = V + j0;
          if (g_dgemm) {
            g_dgemm(ROW_MAJOR, NO_TRANS, TRANS, R, (int)m, C, 1.0, T.data(), C, Vc, (int)ldv, 1.0, Yb.data(), (int)m);
          } else {
            for (int i = 0; i < R; ++i)
              for (int64_t c = 0; c < m; ++c) {
                double s = 0.0;
                for (int j = 0; j < C; ++j) s += T[(size_t)i * C + j] * Vc[c * ldv + j];
                Yb[(size_t)i * m + c] += s;
              }
          }
        }
      }
      const int64_t o = i0 - row0;
      for (int i = 0; i < R; ++i)
        for (int64_t c = 0; c < m; ++c) Y[c * ldy + o + i] = Yb[(size_t)i * m + c];
    }
  }
  return 0;
}

// Rows [row0, row0 + rows) of K, row-major (ld n): the tile generator alone, for tests.
int mf_kblock(int family, double amplitude, double ell, double jitter, const double* X, int64_t n, int d, int64_t row0,
              int64_t rows, double* out) {
  if (n < 1 || d < 1 || d > MAXD || rows < 0 || row0 < 0 || row0 + rows > n) return 1;
  Spec sp;
  sp.family = family;
  sp.a2 = amplitude * amplitude;
  sp.ell = ell;
  sp.two_ll = 2.0 * ell * ell;
  sp.diag = sp.a2 + jitter;
  std::vector<double> sq(n);
  for (int64_t i = 0; i < n; ++i) sq[i] = sqnorm(X + i * d, d);
#pragma omp parallel
  {
    Chunk ch;
    alignas(64) double lanes[W];
#pragma omp for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
      const int64_t gi = row0 + i;
      for (int64_t j0 = 0; j0 < n; j0 += 4096) {
        const int C = (int)std::min<int64_t>(4096, n - j0);
        ch.load(X, sq.data(), d, j0, C);
        for (int j = 0; j < ch.Cp; j += W) {
          vstore(lanes, entries(sp, X + gi * d, sq[gi], ch, d, j));
          for (int l = 0; l < std::min(W, C - j); ++l) out[i * n + j0 + j + l] = (j0 + j + l == gi) ? sp.diag : lanes[l];
        }
      }
    }
  }
  return 0;
}

}  // extern "C"
