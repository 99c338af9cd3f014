// Internal declarations shared by the rld CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "rld.h"

namespace rld {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void cublas_check(cublasStatus_t s, const char* what, const char* file, int line);
void cusolver_check(cusolverStatus_t s, const char* what, const char* file, int line);

#define RLD_CUDA(x) ::rld::cuda_check((x), #x, __FILE__, __LINE__)
#define RLD_CUBLAS(x) ::rld::cublas_check((x), #x, __FILE__, __LINE__)
#define RLD_CUSOLVER(x) ::rld::cusolver_check((x), #x, __FILE__, __LINE__)
extern thread_local int g_launches;
#define RLD_LAUNCH_CHECK()                                                    \
  do {                                                                        \
    ++::rld::g_launches;                                                      \
    ::rld::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
  } while (0)

// Live handles in the process.  With more than one, K x V launches from different streams may
// run concurrently and interleave on the SMs, so the tensor-core kernel drops its inter-CTA epoch
// barrier (a spin on CTAs that another kernel's blocks could keep off the SMs).
extern std::atomic<int> g_live_handles;

// Run `f` once per CUDA device (kernel attributes such as the dynamic shared-memory limit are per
// device); safe from several host threads (f is idempotent, so a concurrent double call is harmless).
template <typename F>
void once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// Grow-only device buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void reserve(size_t nbytes);
  void release();
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
  ~DevBuf() { release(); }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Kernel-matrix description as the device sees it.
struct KernelParams {
  int family;        // rld_family
  int d;
  double a2;         // amplitude^2
  double inv_2l2;    // 1 / (2 ell^2)          (RBF)
  double s5_over_l;  // sqrt(5) / ell          (Matern-5/2)
  double diag;       // amplitude^2 + jitter   (src/kernels.py:72)
};

// K rows [row0, row0 + rows) x all n columns, written as T with row stride ld.
// fp32 K rows [row0, row0 + rows) in the tiled layout Kt[ceil(rows/128)][ceil(n/32)][128][32]
// (zero padded): every tensor-core pipeline step streams one contiguous 16 KB tile.
void build_kernel_tiles(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, float* Kt,
                        cudaStream_t st);
inline int64_t tiled_elems(int64_t rows, int64_t n) { return ceil_div(rows, 128) * 128 * ceil_div(n, 32) * 32; }

template <typename T>
void build_kernel_rows(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows,
                       T* K, int64_t ld, cudaStream_t st);

// ---------------------------------------------------------------------------
// Block products with K.  Y[c, i] = sum_j K[row0 + i, j] * V[c, j] for the m rows
// of V (each of length n) and the local K rows i in [0, rows).  Y is float64,
// rows layout with row stride ldy.
struct KvOperand {
  // Exactly one source of K.
  const void* K = nullptr;   // dense rows (rows x n, row stride ldk), dtype below
  int64_t ldk = 0;
  bool tiled = false;        // fp32 K in 16 KB tiles [ceil(rows/128)][ceil(n/32)][128][32] (see kgen.cu)
  const double* X = nullptr; // points (n x d) for on-the-fly generation
  const float* pts4 = nullptr;  // points as n x 8 fp32 (hi x,y,z,w; lo x,y,z,w) for the tensor-core on-the-fly path, d <= 4
  KernelParams kp{};
  int dtype = RLD_FP64;      // product arithmetic
  const int8_t* kq = nullptr;      // K as exact int8 slices, k-step-tiled image (kv_ozaki.cu), or null
  int kslices = 7;                 // 7: float64 K; 3: float32 K (Morton-ordered points)
  const uint32_t* koff = nullptr;  // sparse 3-slice image: slice offset of every block's kept slices
  const double* ksigma = nullptr;  // per-row power-of-two scales of the slices
  const int* knz = nullptr;        // per (tile, k-step) block: slices from the first nonzero one (or null)
  int64_t n = 0;             // columns of K (global order)
  int64_t row0 = 0;          // first global row held locally
  int64_t rows = 0;          // local rows
  int tc_mode = 3;           // tensor-core product: 3 = 3xTF32 (Lanczos), 1 = 1xTF32 (sketch)
  int oz_diags = 7;          // float64 int8-slice product: slice-pair diagonals kept (7 = all 28 pairs)
  const int8_t* kr = nullptr;      // K' residues modulo the CRT moduli (kv_crt.cu), or null
  const float* rowscale = nullptr; // tiled fp32 K: per-row power-of-two scales (kv_otf.cu stored products)
  const uint32_t* otf_skip = nullptr;  // on the fly: (tile, k-step) far-field skip bits (kv_otf.cu), or null
};

struct KvWorkspace {
  DevBuf vcast;       // V converted to the product dtype
  DevBuf partial;     // split-K partial sums
  DevBuf bhi, blo;    // tensor-core B operand (tf32 hi / lo rows)
  DevBuf tc_partial;  // stream-K partial accumulators
  DevBuf tc_sync;     // epoch-barrier counters of the tensor-core kernel
  cublasHandle_t blas = nullptr;   // the handle's cuBLAS (bound to the same stream): fp64 stored K
  DevBuf oz_vq, oz_tau;            // int8 slices of V and their column scales (kv_ozaki.cu)
  DevBuf otf_vmax;                 // per-vector max |V| of the fp16 on-the-fly product (kv_otf.cu)
  DevBuf crt_vmax, crt_vr, crt_out;   // CRT product (kv_crt.cu): V scales, V residues, output residues
};

bool kv_tc_supported(const KvOperand& op);
// On-the-fly float32 product on the kind::f16 tensor cores (kv_otf.cu; default, RLD_OTF_KIND=tf32
// selects the 3xTF32 kernel).  Points in op.pts4 padded to otf_points_floats(n) floats.
bool kv_otf_f16_enabled();
int64_t otf_points_floats(int64_t n);
// far-field skip map of the on-the-fly fp16 product (otf_skip_words(rows, n) words)
int64_t otf_skip_words(int64_t rows, int64_t n);
double otf_skip_fraction(const uint32_t* bits, int64_t rows, int64_t n, DevBuf& scratch, cudaStream_t st);
void otf_skip_map(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, uint32_t* bits,
                  DevBuf& scratch, cudaStream_t st);
// per-row scales of a tiled fp32 K for the fp16 stored products (wide products, m > 64)
void kv_rowscales(const float* Kt, int64_t rows, int64_t n, float* rs, cudaStream_t st);
void kv_product_otf16(const KvOperand& op, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                      KvWorkspace& ws, cudaStream_t st);
// presplit: the B operand (tf32 hi / lo of V in the k-step blocked layout) was already written
// into ws.bhi / ws.blo by the caller (see kv_tc_b_layout); V is then unused.
void kv_product_tc(const KvOperand& op, int mode, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                   KvWorkspace& ws, cudaStream_t st, bool presplit = false);

// Layout of the tensor-core B operand of an m-vector product: element (vector c, column j) at
// ((j >> 5) * mp + c) * 32 + (j & 31) when blocked (else c * ks * 32 + j); hi = tf32(v) (mode 3)
// or fp32(v) (mode 1), lo = fp32(v - hi).  Reserves the buffers; false if the product does not
// run on the tensor cores.
struct TcBLayout {
  float* bhi = nullptr;
  float* blo = nullptr;
  int64_t mp = 0, ks = 0;
  int blocked = 1, mode = 3;
};
bool kv_tc_b_layout(const KvOperand& op, int64_t m, KvWorkspace& ws, TcBLayout& out);

// V: m x n rows (float64, device).  Y: m x rows (float64, device, row stride ldy).
void kv_product(const KvOperand& op, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                KvWorkspace& ws, cudaStream_t st, int* launches, bool presplit = false);

// Float64 products on the FP64 tensor cores (kv_dmma.cu):
// C (q x p, ld ldc) = beta C + A B^T for A: p x n (ld lda), B: q x n (ld ldb), rows layout.
// Rows must start 16-byte aligned (gemm_nt_f64_ok); deterministic split-k.
bool gemm_nt_f64_ok(const double* A, int64_t lda, const double* B, int64_t ldb);
void gemm_nt_f64(const double* A, int64_t lda, int64_t p, const double* B, int64_t ldb, int64_t q, int64_t n,
                 double* C, int64_t ldc, double beta, DevBuf& partial, cudaStream_t st);
// C (q x N, rows layout) = beta C + alpha S^T X for S: p x q column-major (small), X: p x N rows
// layout (the expansions U T, Q R^-1, Q^T V of the preconditioner and its Woodbury apply).
void gemm_expand_f64(const double* S, int64_t lds, int64_t p, int64_t q, const double* X, int64_t ldx, int64_t N,
                     double* C, int64_t ldc, double alpha, double beta, cudaStream_t st, bool tri_upper = false);
// tri_upper: S is upper triangular (S[k][b] = 0 for k > b): the k loop of an output tile stops at its last row

// Float64-accurate products on the INT8 tensor cores (kv_ozaki.cu): exact 7 x 8-bit slicing
// (`slices` = 7; a float32 K from Morton-ordered points is held as 3 slices and multiplied with 4 of V).
int64_t ozaki_bytes(int64_t rows, int64_t n, int tile_rows, int slices = 7);   // size of a sliced image (tiles of 128 / 64 rows)
void ozaki_slice(const double* A, int64_t lda, int64_t rows, int64_t n, int tile_rows, int8_t* q, double* scale,
                 cudaStream_t st, int slices = 7);
// the same image straight from the points (no float64 K): stationary kernel, row max = diagonal
// Kr != null: also K's CRT residue image (kv_crt.cu), crt_bytes(rows, n) bytes
// knz != null: per (128-row tile, 32-column k-step) block, slices - the number of leading all-zero slices
// (int [ceil(rows/128)][ceil(n/32)]), which the product skips
void ozaki_slice_points(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, int8_t* q,
                        double* scale, cudaStream_t st, int8_t* Kr = nullptr, int* knz = nullptr, int slices = 7,
                        const uint32_t* koff = nullptr);
// sparse 3-slice image of a float32 K (Morton-ordered points): per block the slices kept (a bound from
// the point boxes) and their slice offsets; returns the slices kept in all (4096 bytes each).  The
// image is then written by ozaki_slice_points(..., knz = keep, slices = 3, koff)
int64_t ozaki_sparse_plan(const double* X, int64_t n, const KernelParams& kp, int64_t row0, int64_t rows, int* keep,
                          uint32_t* koff, DevBuf& scratch, cudaStream_t st);
void kv_product_ozaki(const int8_t* Kq, const double* ksigma, int64_t rows, int64_t n, const double* V, int64_t ldv,
                      int64_t m, double* Y, int64_t ldy, KvWorkspace& ws, cudaStream_t st, int diags = 7,
                      const int* knz = nullptr, int kslices = 7, const uint32_t* koff = nullptr);
// Wide float64 products as 15 modular int8 GEMMs + CRT (kv_crt.cu); the residue image of K comes
// from its slice image (crt_residues, 15 bytes per entry).
bool crt_supported(int64_t n);
int64_t crt_bytes(int64_t rows, int64_t n);
void crt_residues(const int8_t* Kq, int64_t rows, int64_t n, int8_t* Kr, cudaStream_t st);
void kv_product_crt(const int8_t* Kr, const double* ksigma, int64_t rows, int64_t n, const double* V, int64_t ldv,
                    int64_t m, double* Y, int64_t ldy, KvWorkspace& ws, cudaStream_t st);
constexpr int64_t CRT_MIN_M = 96;   // narrower products (the Lanczos block) stay on the slices
// Which float64 stored-K product a prepare sets up: the int8 slices (default) or, with
// RLD_FP64_PRODUCT=dmma, the DMMA kernel on the float64 K.
bool fp64_product_ozaki();
// float32 stored K from Morton-ordered points as 3 int8 slices (default; RLD_FP32_PRODUCT=tf32: fp32 tiles)
bool fp32_product_slices();

// ---------------------------------------------------------------------------
// RNG
void rademacher_rows(const uint64_t key[2], int64_t rows, int64_t n, int64_t row0_col, int64_t ncols,
                     int64_t ld, double* out, cudaStream_t st);

// ---------------------------------------------------------------------------
// Small vector kernels (rows layout).
void rows_dot(int64_t m, int64_t n, const double* a, int64_t lda, const double* b, int64_t ldb,
              double* out, DevBuf& scratch, cudaStream_t st, int* launches);

}  // namespace rld
