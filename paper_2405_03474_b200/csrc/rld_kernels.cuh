// Host wrappers of the small kernels in vec_kernels.cu.
#pragma once

#include "rld_internal.cuh"

namespace rld {

enum : int {
  RLD_FLAG_RANK_DEFICIENT = 1,
  RLD_FLAG_NOT_PD = 2,
  RLD_FLAG_SINGULAR = 4,
  RLD_FLAG_BAD_BASE = 8,
  RLD_FLAG_QR_WEAK = 16,
  RLD_FLAG_EIG_NOCONV = 32,
};

void normalize_rows(int64_t m, int64_t n, const double* z, const double* nrm2, double* norms, double* q,
                    cudaStream_t st);

// u = KX - alpha_j p - beta_{j-1} p_prev (or u = KX when !three_term: the residual is then
// reorthogonalised against the whole basis, src/lanczos.py:58-62); w = u / sqrt_base
void lanczos_residual(int64_t m, int64_t n, int j, int t, const double* KX, const double* alpha,
                      const double* beta, const double* p, const double* p_prev, const double* sqrt_base, double* u,
                      double* w, cudaStream_t st, bool three_term = true);
void lanczos_alpha(int64_t m, int j, int t, const double* dots, const int* live, double* alpha, cudaStream_t st);
void lanczos_beta(int64_t m, int j, int t, double rtol, const double* beta2, double* alpha, double* beta,
                  double* beta_ref, int* live, int* size, cudaStream_t st);
void lanczos_advance(int64_t m, int64_t n, int j, int t, const double* beta, const int* live, const double* u,
                     const double* z, double* p, double* p_prev, double* x, cudaStream_t st);
void thomas_hutchinson(int64_t m, int t, const double* alpha, const double* beta, const int* size,
                       const double* norms, int npoles, double offset, const double* poles,
                       const double* residues, double* per_probe, double* trace, int* flags, cudaStream_t st);

void slq_epilogue(int64_t m, int t, const double* alpha, const double* beta, const int* size, const double* norms,
                  double eig_floor, double* per_probe, double* trace, int* clamped, int* flags, cudaStream_t st);

void scale_rows_colmajor(int64_t rows, int64_t cols, int64_t ld, const double* f, bool divide, double* a,
                         cudaStream_t st);
void scale_cols_colmajor(int64_t rows, int64_t cols, int64_t ld, const double* f, double* a, cudaStream_t st);
void copy_doubles(int64_t count, const double* s, double* d, cudaStream_t st);
void sub_block(int64_t rows, int64_t cols, const double* T, int64_t ldt, double* G, int64_t ldg, cudaStream_t st);
void combine_info(int* info, const int* i1, const int* i2, int n1, cudaStream_t st);
void fill_doubles(int64_t count, double v, double* d, cudaStream_t st);

void cholqr_check(int w, const double* R, const double* gdiag, const int* info, double rtol, int* flags,
                  cudaStream_t st);
void householder_check(int w, const double* R, int64_t ldr, const double* norms2, double rtol, double* sgn,
                       int* flags, cudaStream_t st);
void copy_upper(int w, const double* src, int64_t lds, double* dst, cudaStream_t st);
void diag_copy(int w, const double* G, double* d, cudaStream_t st);
void top_eigvecs(int w, int k, const double* V, const double* theta, double* Vtop, double* theta_top,
                 cudaStream_t st);
void precond_base(int64_t n, int k, const double* diag, double floor_v, double* A, double* base, double* sqrt_base,
                  cudaStream_t st);
void sum_log(int64_t n, const double* v, double* out, DevBuf& scratch, cudaStream_t st);
void add_identity(int k, double* C, cudaStream_t st);
void chol_logdet(int k, const double* L, const int* info, double* out, int* flags, cudaStream_t st);
// One-cluster Cholesky G = R^T R (upper, in place, info as LAPACK potrf) for n <= 640; false if n is
// out of range (caller falls back to cuSOLVER).  small_chol.cu
// With Rinv != nullptr also writes R^-1 (upper, n x n, ld n, lower part zero).
bool small_potrf_upper(int n, double* G, int ld, int* info, cudaStream_t st, double* Rinv = nullptr);
// Eigen-decomposition of a symmetric n x n matrix (3 <= n <= 288) up to the last two steps
// (tri_eig.cu): eigenvalues ascending into w; Z (n x n) = eigenvectors of the tridiagonal T from
// inverse iteration (orthogonal up to eps |T| / gap: the caller runs one Cholesky-QR pass) and
// Q (n x n) with A = Q T Q^T, both in `scratch`; eigenvectors of A = Q orth(Z).  `spare` points to
// 3 n^2 free doubles.  Q is formed on st2 (fork / join events), joined into st before returning.
// false if n is out of range or RLD_TRI_EIG=0.
bool tri_eigh(int n, const double* A, double* w, DevBuf& scratch, double** Z, double** Q, double** spare,
              cudaStream_t st, cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join);
// *out = max |G - I| of the n x n matrix G (NaN reads as 1e300)
void orth_defect(int n, const double* G, double* out, cudaStream_t st);
void sqrt_factors(int k, double keep_rtol, const double* lam, double* W, double* h, double* g, double* gam,
                  int* kept, cudaStream_t st);
void convert_rows(const void* src, int sdt, void* dst, int ddt, int64_t count, cudaStream_t st);
void convert_rows_2d(const void* src, int sdt, int64_t lds, double* dst, int64_t rows, int64_t cols,
                     cudaStream_t st);
void sqrt_into(int64_t n, const double* base, double* sqrt_base, int* flags, cudaStream_t st);
void strided_sum_log(int64_t count, const double* v, int64_t stride, double* out, DevBuf& scratch,
                     cudaStream_t st);
// rows x n standard normals of numpy stream `key` (Generator(Philox).standard_normal, bit-exact),
// columns [col0, col0 + ncols) of each row to out (row stride ld); dflags bit set on overflow
// end_word (device, optional): the stream word index following the last draw (where a
// host continuation of the same numpy stream starts, see rng_host.cu)
void normal_rows(const uint64_t key[2], int64_t rows, int64_t n, int64_t col0, int64_t ncols, int64_t ld,
                 double* out, DevBuf& scratch, int* dflags, cudaStream_t st, int64_t* end_word = nullptr);
void chi_radii_host(const uint64_t key[2], uint64_t word0, int64_t df, int64_t count, double* out);
// [G][m][L] (all-gathered shards) -> m x n rows, n <= G L
void relayout_gathered(const double* src, int G, int64_t m, int64_t L, int64_t n, double* dst, cudaStream_t st);
// tiled fp32 K (kgen.cu layout): relayout of row-major rows, back to float64 rows, diagonal
void tile_rows(const float* src, int64_t lds, int64_t r0, int64_t nr, int64_t n, float* Kt, cudaStream_t st);
void untile_to_f64(const float* Kt, int64_t rows, int64_t n, double* out, int64_t ldo, cudaStream_t st);
void diag_of_tiled(int64_t rows, int64_t row0, int64_t n, const float* Kt, double* d, cudaStream_t st);
// preconditioner kinds beyond rand-svd (src/precond.py:201-267)
void precond_base_scaled(int64_t n, int k, double scale, double* A, double* base, double* sqrt_base,
                         cudaStream_t st);
void argmax_first(int64_t n, const double* d, int64_t offset, double* out, DevBuf& scratch, cudaStream_t st,
                  const int* perm = nullptr);
// Morton order of n device points (d <= 3): perm[i] = original index of point i, Xs the sorted points
void morton_order_device(const double* X, int64_t n, int d, int* perm, double* Xs, DevBuf& scratch, cudaStream_t st);
// m rows of length n: gather dst[c][i] = src[c][perm[i]], or scatter dst[c][perm[i]] = src[c][i]
void permute_rows(int64_t m, int64_t n, const int* perm, const double* src, int64_t lds, double* dst, int64_t ldd,
                  bool scatter, cudaStream_t st);
// out = the (value, index) pair with the largest value, first on ties, of P pairs ordered by index
// perm != null: equal values go to the pair whose (global resident) index has the smallest perm[]
void pick_first_max(int P, const double* pairs, double* out, cudaStream_t st, const int* perm = nullptr);
void kernel_column(int64_t rows, int64_t row0, int64_t n, int64_t p, const void* K, int64_t ldk, int kdtype,
                   bool tiled, const double* X, const KernelParams& kp, double* out, cudaStream_t st);
void pchol_update(int64_t rows, const double* col, const double* dp, double* Cj, double* d, cudaStream_t st);
void row_of_owner(int64_t rows, int64_t row0, const double* pv, const double* C, int j, double* out,
                  cudaStream_t st);
void scale_by(int64_t n, double* v, const double* f, int mode, cudaStream_t st);
// out[e] = sum_{b < nb} in[b * count + e] (fixed order)
void sum_blocks(int64_t nb, int64_t count, const double* in, double* out, cudaStream_t st);
void pad_points(const double* X, int64_t n, int d, double scale, float* pts8, cudaStream_t st);
void diag_of_dense(int64_t rows, int64_t row0, const void* K, int64_t ldk, int dtype, double* d, cudaStream_t st);

}  // namespace rld
