// C ABI (include/rld.h) and the device-side orchestration of one estimate.
//
// rld_logdet follows src/estimators.py:77-96 end to end on the GPU:
//   preconditioner (src/precond.py:168-198, 231-267, 69-100)
//     -> probes (src/estimators.py:64)
//     -> s-probe Lanczos on N^-1 K N^-T (src/estimators.py:68-72, src/lanczos.py:34-74)
//     -> multishift Thomas solves + Hutchinson mean (src/lanczos.py:77-84, src/estimators.py:86-95).
// Everything is ordered on the handle's stream; the host synchronises only to
// decide the RankDeficient retry (src/precond.py:181-197) and to read the result.
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <algorithm>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.cuh"
#include "rld_internal.cuh"
#include "rld_kernels.cuh"

namespace rld {

thread_local int g_launches = 0;
std::atomic<int> g_live_handles{0};  // own kernel launches (RLD_LAUNCH_CHECK)

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

// NVTX phase ranges (nsys / ncu --nvtx): a no-op unless a tool injects itself
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  (void)cudaGetLastError();
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  fail(e == cudaErrorMemoryAllocation ? RLD_ERR_OUT_OF_MEMORY : RLD_ERR_CUDA, buf);
}

void cublas_check(cublasStatus_t s, const char* what, const char* file, int line) {
  if (s == CUBLAS_STATUS_SUCCESS) return;
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: cublas status %d (%s:%d)", what, (int)s, file, line);
  fail(s == CUBLAS_STATUS_ALLOC_FAILED ? RLD_ERR_OUT_OF_MEMORY : RLD_ERR_CUDA, buf);
}

void cusolver_check(cusolverStatus_t s, const char* what, const char* file, int line) {
  if (s == CUSOLVER_STATUS_SUCCESS) return;
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: cusolver status %d (%s:%d)", what, (int)s, file, line);
  fail(s == CUSOLVER_STATUS_ALLOC_FAILED ? RLD_ERR_OUT_OF_MEMORY : RLD_ERR_CUDA, buf);
}

void DevBuf::reserve(size_t nbytes) {
  if (nbytes <= bytes) return;
  release();
  if (nbytes == 0) return;
  RLD_CUDA(cudaMalloc(&ptr, nbytes));
  bytes = nbytes;
  // RLD_POISON=1 (debugging): fresh workspace is filled with NaN bytes, so a kernel that reads
  // memory nothing wrote shows up as a NaN / wrong result instead of silently reusing stale values
  static const bool poison = getenv("RLD_POISON") && getenv("RLD_POISON")[0] == '1';
  if (poison) {   // the handle's stream does not order against the legacy stream: wait here
    RLD_CUDA(cudaMemset(ptr, 0xFF, nbytes));
    RLD_CUDA(cudaDeviceSynchronize());
  }
}

void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

namespace {

struct Resident {
  bool ready = false;
  int source = 0, path = 0, dtype = 0, family = 0;
  int64_t n = 0;
  int d = 0;
  double amplitude = 1, ell = 1, jitter = 0;
  int64_t row0 = 0, rows = 0;
  DevBuf Kbuf;               // owned stored rows
  const void* K = nullptr;   // stored rows (owned or aliased)
  int64_t ldk = 0;
  bool tiled = false;        // fp32 K in the 16 KB-tile layout (kgen.cu build_kernel_tiles)
  DevBuf X;                  // points n x d
  DevBuf pts4;               // points split to n x 8 fp32 hi/lo (d <= 4; tensor-core on-the-fly tiles)
  DevBuf diag;               // local diagonal of K (float64)
  DevBuf Kq, ksigma;         // K as exact int8 slices (kv_ozaki.cu): float64 (7 slices, RLD_FP64_PRODUCT=ozaki)
  bool kq_ready = false;     // or float32 from Morton-ordered points (3 slices, sparse image)
  int kslices = 7;
  DevBuf koff;               // sparse 3-slice image: slice offset of every block (kv_ozaki.cu)
  bool koff_ready = false;
  bool cached = false;       // on-the-fly float32 problem whose sparse slice image fits in HBM: served from it
  DevBuf perm;               // points held in Morton (Z-curve) order: perm[i] = original index of point i
  bool permuted = false;     // (every rank alike; far-field slice blocks are then all-zero and skipped)
  DevBuf knz;                // per slice-image block: slices from the first nonzero one (skipped leading zeros)
  DevBuf otf_skip;           // on the fly (fp32, Morton order): far-field (tile, k-step) skip bits
  bool otf_skip_ready = false;
  bool knz_ready = false;
  DevBuf Kr;                 // residues of K' modulo the CRT moduli (kv_crt.cu), for the wide products
  bool kr_ready = false;
  DevBuf rowscale;           // tiled fp32 K: per-row power-of-two scales (fp16 wide products, kv_otf.cu)
  KernelParams kp{};

  KvOperand op() const {
    KvOperand o;
    o.K = (path == RLD_PATH_ON_THE_FLY) ? nullptr : K;
    o.ldk = ldk;
    o.tiled = tiled;
    o.rowscale = (tiled && path != RLD_PATH_ON_THE_FLY) ? rowscale.as<float>() : nullptr;
    o.otf_skip = (otf_skip_ready && path == RLD_PATH_ON_THE_FLY) ? otf_skip.as<uint32_t>() : nullptr;
    o.X = X.as<double>();
    o.pts4 = (source == RLD_SOURCE_POINTS && d <= 4) ? pts4.as<float>() : nullptr;
    o.kp = kp;
    o.dtype = dtype;
    if (kq_ready && (path != RLD_PATH_ON_THE_FLY || cached)) {
      o.kq = Kq.as<int8_t>();
      o.kslices = kslices;
      if (koff_ready) o.koff = koff.as<uint32_t>();
      o.ksigma = ksigma.as<double>();
      if (knz_ready) o.knz = knz.as<int>();
      if (kr_ready) o.kr = Kr.as<int8_t>();
    }
    o.n = n;
    o.row0 = row0;
    o.rows = rows;
    return o;
  }
};

struct Work {
  DevBuf Y, Z, A, G, gdiag, theta, Vtop, theta_top, C, inner, lam, hgg, base, sqrt_base;
  DevBuf omega, probes;
  DevBuf ptmp, ptmp2;  // n-vector blocks moved into / out of the resident (Morton) order
  DevBuf x, p, pp, u, w, KX, T, Tg;
  DevBuf scal;     // small scalars / per-probe arrays
  DevBuf ints;     // flags, info, live, size, kept
  DevBuf scratch, scratch2, solver_work, rng_scratch, gram_scratch, qtile;
  DevBuf gsend, grecv;   // row-shard all-gather staging
  DevBuf qbasis, pbasis, coef;   // reorthogonalised Lanczos: bases (t x s x rows) and coefficients
  DevBuf endw, radii;            // normal-orthogonal probes: stream position, chi radii
  DevBuf rinv;                   // CholQR: explicit R^-1
  DevBuf eig_scratch;            // one-cluster eigensolver: V and singular values
  DevBuf flagbuf;        // flag OR over ranks
  KvWorkspace kv;
};

}  // namespace
}  // namespace rld

struct rld_handle {
  int device = 0, rank = 0, world = 1;
  bool counted = false;   // included in rld::g_live_handles
  cudaStream_t st = nullptr;
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  std::unique_ptr<rld::Comm> comm;   // world > 1: NCCL or virtual shards (comm.cu)
  int precond_k = -1;                 // columns of U of the last preconditioner build (-1: none)
  std::string last_error;
  rld::Resident res;
  rld::Work wk;
  cudaEvent_t ev[8] = {};
  cudaStream_t st2 = nullptr;        // side stream for independent small work (joined before use)
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t efork = nullptr, ejoin = nullptr;   // the eigensolver's own side-stream branch
};

namespace rld {
namespace {

constexpr double ONE = 1.0, ZERO = 0.0;

struct Partial {
  double offset;
  int npoles;
  double poles[5], residues[5];
};

// Table 1 (src/rational.py:70-96)
Partial partial_fraction(int order) {
  Partial p{};
  if (order == 1) {
    p = {2.0, 1, {-1.0}, {-4.0}};
  } else if (order == 3) {
    p = {14.0 / 3.0, 3, {-13.92820323027551, -1.0, -0.0717967697244908},
         {-49.52250037431294, -20.0 / 9.0, -0.2552774034648563}};
  } else if (order == 5) {
    p = {86.0 / 15.0, 5,
         {-39.863458189061411, -3.8518399963191827, -1.0, -0.25961618368249978, -0.025085630936916615},
         {-140.08241129102026, -6.1858406006156228, -92.0 / 75.0, -0.41692913805732562,
          -0.088152303639431204}};
  } else {
    fail(RLD_ERR_INVALID_ARGUMENT, "partial fractions exist for odd orders 1, 3, 5; got " + std::to_string(order));
  }
  return p;
}

void set_device(rld_handle* h) { RLD_CUDA(cudaSetDevice(h->device)); }

// --- collectives (row shards).  world == 1: no-ops. --------------------------
void allreduce_sum(rld_handle* h, double* buf, int64_t count) {
  if (h->world == 1 || count <= 0) return;
  h->comm->allreduce_sum(buf, count, h->st);
}

// Bitwise OR of the host copies of the status flags over ranks.  Flags raised on
// local rows only (BAD_BASE, generator overflow) must stop every rank alike.
void allreduce_flags(rld_handle* h, int* hflags, int count) {
  if (h->world == 1) return;
  std::vector<int> bits(32 * count);
  for (int i = 0; i < count; ++i)
    for (int b = 0; b < 32; ++b) bits[32 * i + b] = (hflags[i] >> b) & 1;
  DevBuf& d = h->wk.flagbuf;
  d.reserve(sizeof(int) * bits.size());
  RLD_CUDA(cudaMemcpyAsync(d.ptr, bits.data(), sizeof(int) * bits.size(), cudaMemcpyHostToDevice, h->st));
  h->comm->allreduce_max(d.as<int>(), (int64_t)bits.size(), h->st);
  RLD_CUDA(cudaMemcpyAsync(bits.data(), d.ptr, sizeof(int) * bits.size(), cudaMemcpyDeviceToHost, h->st));
  RLD_CUDA(cudaStreamSynchronize(h->st));
  for (int i = 0; i < count; ++i) {
    hflags[i] = 0;
    for (int b = 0; b < 32; ++b) hflags[i] |= bits[32 * i + b] << b;
  }
}

// Locality order (Morton, morton_order_device) for the points of the products that skip exactly-zero
// work: d <= 3; RLD_SORT=0 keeps the given order.
bool sort_points(const rld_handle* h, const rld_problem* p) {
  const char* e = getenv("RLD_SORT");
  if (e && e[0] == '0') return false;
  // float64 stored on int8 slices (all-zero leading slices skipped) or float32 on the fly (far-field
  // k-steps with exactly-zero fp16 operands skipped)
  const bool slices = p->path == RLD_PATH_STORED &&
                      (p->dtype == RLD_FP64 ? fp64_product_ozaki() : fp32_product_slices());
  const bool otf = p->path == RLD_PATH_ON_THE_FLY && p->dtype == RLD_FP32 && kv_otf_f16_enabled();
  // (every rank sorts all n points the same way; its rows are a block of the sorted order)
  return p->source == RLD_SOURCE_POINTS && (slices || otf) && p->d >= 1 && p->d <= 3 && p->n < (int64_t)1 << 31;
}

// plain: the points as given (no Morton order, no slice image): rld_build_covariance's upload
void prepare(rld_handle* h, const rld_problem* p, bool plain = false) {
  NvtxRange nv("rld:prepare (K rows / points to HBM)");
  if (!p) fail(RLD_ERR_INVALID_ARGUMENT, "problem is NULL");
  if (p->n < 1) fail(RLD_ERR_INVALID_ARGUMENT, "n must be >= 1");
  if (p->dtype != RLD_FP64 && p->dtype != RLD_FP32) fail(RLD_ERR_INVALID_ARGUMENT, "dtype must be fp64 or fp32");
  if (!p->data) fail(RLD_ERR_INVALID_ARGUMENT, "problem data is NULL");
  Resident& r = h->res;
  r.ready = false;
  r.tiled = false;
  r.kq_ready = false;
  r.koff_ready = false;
  r.cached = false;
  r.kslices = 7;
  r.kr_ready = false;
  r.knz_ready = false;
  r.permuted = false;
  r.otf_skip_ready = false;
  h->precond_k = -1;
  r.source = p->source;
  r.dtype = p->dtype;
  r.n = p->n;
  const int64_t L = ceil_div(p->n, h->world);
  if (h->world > 1 && (int64_t)(h->world - 1) * L >= p->n)   // (every rank sees the same condition)
    fail(RLD_ERR_NOT_SUPPORTED, "row sharding needs at least one row of K on every rank (n too small for this world size)");
  r.row0 = std::min<int64_t>(p->n, (int64_t)h->rank * L);
  r.rows = std::min<int64_t>(L, p->n - r.row0);
  cudaStream_t st = h->st;

  if (p->source == RLD_SOURCE_POINTS) {
    if (p->family != RLD_RBF && p->family != RLD_MATERN52) fail(RLD_ERR_INVALID_ARGUMENT, "unknown kernel family");
    if (!(p->amplitude > 0) || !(p->length_scale > 0))
      fail(RLD_ERR_INVALID_ARGUMENT, "amplitude and length_scale must be positive");
    if (!(p->jitter >= 0)) fail(RLD_ERR_INVALID_ARGUMENT, "jitter must be non-negative");
    if (p->d < 1) fail(RLD_ERR_INVALID_ARGUMENT, "n and d must be >= 1");
    if (p->d > 32) fail(RLD_ERR_NOT_SUPPORTED, "point dimension d > 32 is not supported by the device kernels");
    r.path = p->path;
    r.family = p->family;
    r.d = p->d;
    r.amplitude = p->amplitude;
    r.ell = p->length_scale;
    r.jitter = p->jitter;
    r.kp.family = p->family;
    r.kp.d = p->d;
    r.kp.a2 = p->amplitude * p->amplitude;
    r.kp.inv_2l2 = 1.0 / (2.0 * p->length_scale * p->length_scale);
    r.kp.s5_over_l = std::sqrt(5.0) / p->length_scale;
    r.kp.diag = r.kp.a2 + p->jitter;
    const size_t xb = sizeof(double) * p->n * p->d;
    r.X.reserve(xb);
    if (!plain && sort_points(h, p)) {
      // float64 stored products on int8 slices: points in Morton order make the K blocks away from
      // the diagonal small, and their leading slices all zero, which the product skips (kv_ozaki.cu).
      // Every n-vector entering or leaving the resident frame is permuted (probes, sketch rows, the
      // rank-one start, kv_apply / precond_apply operands); pivot ties go to the original index.
      h->wk.ptmp.reserve(xb);   // the caller's points on the device, then sorted into r.X
      RLD_CUDA(cudaMemcpyAsync(h->wk.ptmp.ptr, p->data, xb,
                               p->data_memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
      r.perm.reserve(sizeof(int) * p->n);
      morton_order_device(h->wk.ptmp.as<double>(), p->n, p->d, r.perm.as<int>(), r.X.as<double>(), h->wk.scratch2, st);
      r.permuted = true;
    } else {
      RLD_CUDA(cudaMemcpyAsync(r.X.ptr, p->data, xb,
                               p->data_memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    }
    r.diag.reserve(sizeof(double) * std::max<int64_t>(1, r.rows));
    fill_doubles(r.rows, r.kp.diag, r.diag.as<double>(), st);
    if (p->d <= 4) {
      r.pts4.reserve(sizeof(float) * otf_points_floats(p->n));
      // coordinates pre-scaled so the tile generator's r^2 is the kernel argument
      const double scale = p->family == RLD_MATERN52 ? r.kp.s5_over_l : std::sqrt(r.kp.inv_2l2 * 1.4426950408889634);
      pad_points(r.X.as<double>(), p->n, p->d, scale, r.pts4.as<float>(), st);
      if (r.permuted && p->dtype == RLD_FP32 && fp32_product_slices()) {   // (collective: ranks without rows too)
        // float32 K from Morton-ordered points (d <= 3) as a SPARSE image of 3 int8 slices:
        // the float64 kernel value rounded to 24 bits of its row scale (float32-grade next to the
        // diagonal; far-field entries below 2^-25 of the scale are exactly zero), only the slices a
        // bound from the point boxes allows to be nonzero are evaluated and stored, and the product
        // multiplies them with 4 slices of V on the INT8 tensor cores (kv_ozaki.cu <3, 4>).  A
        // stored problem always takes it (<= 3 bytes per entry, no fp32 K); an on-the-fly problem
        // when the image leaves a quarter of HBM free (config 4: clustered points, most blocks
        // empty), and is then served from HBM instead of regenerating K for every product.
        const int64_t nb = ceil_div(r.rows, 128) * ceil_div(p->n, 32);
        r.knz.reserve(sizeof(int) * std::max<int64_t>(nb, 1));
        r.koff.reserve(sizeof(uint32_t) * std::max<int64_t>(nb, 1));
        const int64_t kept = ozaki_sparse_plan(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.knz.as<int>(),
                                               r.koff.as<uint32_t>(), h->wk.scratch2, st);   // 0 without rows
        const int64_t bytes = std::max<int64_t>(kept, 1) * 4096;
        bool take = r.path == RLD_PATH_STORED;
        const char* ce = getenv("RLD_OTF_CACHE");   // 0: always regenerate K on the fly (read per prepare)
        if (!take && !(ce && ce[0] == '0')) {
          size_t fr = 0, tot = 0;
          RLD_CUDA(cudaMemGetInfo(&fr, &tot));
          // room for the estimate's workspaces: ~6 blocks of w x n float64 at the largest BASELINE
          // sketch width (w = 2058; the configuration is not known at prepare) and 8 GB of slack
          const int64_t need = 6 * 2058 * p->n * (int64_t)sizeof(double) + ((int64_t)8 << 30);
          (void)tot;
          take = kept < ((int64_t)1 << 32) && bytes + need <= (int64_t)fr + (int64_t)r.Kq.bytes;
        }
        if (h->world > 1 && r.path == RLD_PATH_ON_THE_FLY) {   // all ranks serve from the image, or none
          int no = take ? 0 : 1;
          allreduce_flags(h, &no, 1);
          take = no == 0;
        }
        if (take) {
          r.Kq.reserve((size_t)bytes);
          r.ksigma.reserve(sizeof(double) * std::max<int64_t>(r.rows, 1));
          ozaki_slice_points(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.Kq.as<int8_t>(), r.ksigma.as<double>(),
                             st, nullptr, r.knz.as<int>(), 3, r.koff.as<uint32_t>());
          r.kslices = 3;
          r.kq_ready = r.knz_ready = r.koff_ready = r.rows > 0;
          r.cached = r.path == RLD_PATH_ON_THE_FLY;
        }
      }
      if (!r.cached && !(r.kq_ready && r.path == RLD_PATH_STORED) && r.permuted && r.path == RLD_PATH_ON_THE_FLY &&
          p->dtype == RLD_FP32) {
        int thin = 0;
        if (r.rows > 0) {
          r.otf_skip.reserve(sizeof(uint32_t) * otf_skip_words(r.rows, p->n));
          otf_skip_map(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.otf_skip.as<uint32_t>(), h->wk.scratch2, st);
          // the order pays only where it skips enough: its per-k-step flushes (kv_otf.cu) cost ~13 %
          // (config 4's clustered points skip ~nothing; config 5 skips most k-steps)
          thin = otf_skip_fraction(r.otf_skip.as<uint32_t>(), r.rows, p->n, h->wk.scratch2, st) >= 0.3 ? 0 : 1;
        }
        if (h->world > 1) allreduce_flags(h, &thin, 1);   // one order for all ranks
        if (!thin) {
          r.otf_skip_ready = r.rows > 0;
        } else {   // back to the caller's order
          std::vector<double> hx((size_t)p->n * p->d), hy((size_t)p->n * p->d);
          std::vector<int> pm((size_t)p->n);
          RLD_CUDA(cudaMemcpyAsync(hx.data(), r.X.ptr, xb, cudaMemcpyDeviceToHost, st));
          RLD_CUDA(cudaMemcpyAsync(pm.data(), r.perm.ptr, sizeof(int) * p->n, cudaMemcpyDeviceToHost, st));
          RLD_CUDA(cudaStreamSynchronize(st));
          for (int64_t i = 0; i < p->n; ++i)
            for (int c = 0; c < p->d; ++c) hy[(size_t)pm[i] * p->d + c] = hx[(size_t)i * p->d + c];
          RLD_CUDA(cudaMemcpyAsync(r.X.ptr, hy.data(), xb, cudaMemcpyHostToDevice, st));
          RLD_CUDA(cudaStreamSynchronize(st));
          r.permuted = false;
          pad_points(r.X.as<double>(), p->n, p->d, scale, r.pts4.as<float>(), st);
        }
      }
    }
    if (r.path == RLD_PATH_STORED) {
      if (p->dtype == RLD_FP64 && fp64_product_ozaki()) {
        // float64 products on exact int8 slices generated straight from the points (kv_ozaki.cu):
        // no float64 K in HBM (column reads and rebuilds go back to the points)
        r.K = nullptr;
        r.ldk = 0;
        if (r.rows > 0) {
          r.Kq.reserve((size_t)ozaki_bytes(r.rows, p->n, 128));
          r.ksigma.reserve(sizeof(double) * r.rows);
          // the CRT residue image for the wide (sketch) products in the same pass, where it fits
          int8_t* kr = nullptr;
          if (crt_supported(p->n) && !r.permuted) {   // Morton-ordered points: the slices skip their
                                                      // all-zero blocks and beat the CRT product
            const int64_t bytes = crt_bytes(r.rows, p->n);
            size_t fr = 0, tot = 0;
            RLD_CUDA(cudaStreamSynchronize(st));
            RLD_CUDA(cudaMemGetInfo(&fr, &tot));
            if ((int64_t)r.Kr.bytes >= bytes || (int64_t)fr > bytes + (int64_t)(tot / 16)) {
              r.Kr.reserve((size_t)bytes);
              kr = r.Kr.as<int8_t>();
            }
          }
          r.knz.reserve(sizeof(int) * ceil_div(r.rows, 128) * ceil_div(p->n, 32));
          ozaki_slice_points(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.Kq.as<int8_t>(), r.ksigma.as<double>(),
                             st, kr, r.knz.as<int>());
          r.kr_ready = kr != nullptr;
          r.knz_ready = true;
        }
        r.kq_ready = r.rows > 0;
      } else if (p->dtype == RLD_FP64) {
        r.ldk = ceil_div(p->n, 4) * 4;
        r.Kbuf.reserve(sizeof(double) * r.rows * r.ldk);
        r.K = r.Kbuf.ptr;
        build_kernel_rows<double>(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.Kbuf.as<double>(), r.ldk, st);
      } else if (r.kq_ready) {   // float32 K held as the sparse 3-slice image built above: no fp32 K
        r.K = nullptr;
        r.ldk = 0;
      } else {   // fp32: 16 KB tiles, one contiguous TMA box per tensor-core step
        r.tiled = true;
        r.ldk = 0;
        r.Kbuf.reserve(sizeof(float) * tiled_elems(r.rows, p->n));
        r.K = r.Kbuf.ptr;
        build_kernel_tiles(r.X.as<double>(), p->n, r.kp, r.row0, r.rows, r.Kbuf.as<float>(), st);
      }
    } else if (r.path != RLD_PATH_ON_THE_FLY) {
      fail(RLD_ERR_INVALID_ARGUMENT, "unknown path");
    }
  } else if (p->source == RLD_SOURCE_DENSE) {
    const int64_t ld = p->ld ? p->ld : p->n;
    if (ld < p->n) fail(RLD_ERR_INVALID_ARGUMENT, "ld < n");
    if (p->data_dtype != RLD_FP64 && p->data_dtype != RLD_FP32) fail(RLD_ERR_INVALID_ARGUMENT, "bad data_dtype");
    r.path = RLD_PATH_STORED;
    r.d = 0;
    const size_t es = p->dtype == RLD_FP64 ? 8 : 4;
    const size_t ses = p->data_dtype == RLD_FP64 ? 8 : 4;
    const char* src = static_cast<const char*>(p->data) + ses * (r.row0 * ld);
    const cudaMemcpyKind kind = p->data_memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (p->dtype == RLD_FP32) {
      // fp32 products read K in 16 KB tiles: stage 128-row chunks, convert, relayout
      r.tiled = true;
      r.ldk = 0;
      r.Kbuf.reserve(sizeof(float) * tiled_elems(r.rows, p->n));
      r.K = r.Kbuf.ptr;
      RLD_CUDA(cudaMemsetAsync(r.Kbuf.ptr, 0, sizeof(float) * tiled_elems(r.rows, p->n), st));
      const int64_t chunk = std::max<int64_t>(128, ((256ll << 20) / (int64_t)(ses * p->n)) / 128 * 128);
      DevBuf& stage = h->wk.scratch2;
      DevBuf& stage32 = h->wk.qtile;
      stage.reserve(ses * chunk * p->n);
      if (ses == 8) stage32.reserve(sizeof(float) * chunk * p->n);
      for (int64_t r0 = 0; r0 < r.rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, r.rows - r0);
        RLD_CUDA(cudaMemcpy2DAsync(stage.ptr, ses * p->n, src + ses * r0 * ld, ses * ld, ses * p->n, nr, kind, st));
        const float* t = stage.as<float>();
        if (ses == 8) {
          convert_rows(stage.ptr, RLD_FP64, stage32.ptr, RLD_FP32, nr * p->n, st);
          t = stage32.as<float>();
        }
        tile_rows(t, p->n, r0, nr, p->n, r.Kbuf.as<float>(), st);
      }
      RLD_CUDA(cudaStreamSynchronize(st));
    } else if (p->data_memory == RLD_DEVICE && p->data_dtype == p->dtype) {
      r.K = src;  // alias the caller's device rows (caller keeps them alive)
      r.ldk = ld;
    } else {
      r.ldk = ceil_div(p->n, 4) * 4;
      r.Kbuf.reserve(es * r.rows * r.ldk);
      r.K = r.Kbuf.ptr;
      if (p->data_dtype == p->dtype) {
        RLD_CUDA(cudaMemcpy2DAsync(r.Kbuf.ptr, es * r.ldk, src, ses * ld, es * p->n, r.rows,
                                   p->data_memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                   st));
      } else {
        // stage in chunks of rows and convert on the device
        const int64_t chunk = std::max<int64_t>(1, (int64_t)((256ull << 20) / (ses * p->n)));
        DevBuf& stage = h->wk.scratch2;
        stage.reserve(ses * chunk * r.ldk);
        for (int64_t r0 = 0; r0 < r.rows; r0 += chunk) {
          const int64_t nr = std::min(chunk, r.rows - r0);
          RLD_CUDA(cudaMemcpy2DAsync(stage.ptr, ses * r.ldk, src + ses * r0 * ld, ses * ld, ses * p->n, nr,
                                     p->data_memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyHostToDevice,
                                     st));
          convert_rows(stage.ptr, p->data_dtype, static_cast<char*>(r.Kbuf.ptr) + es * r0 * r.ldk, p->dtype,
                       nr * r.ldk, st);
        }
        RLD_CUDA(cudaStreamSynchronize(st));
      }
    }
    r.diag.reserve(sizeof(double) * std::max<int64_t>(1, r.rows));
    if (r.tiled)
      diag_of_tiled(r.rows, r.row0, p->n, static_cast<const float*>(r.K), r.diag.as<double>(), st);
    else
      diag_of_dense(r.rows, r.row0, r.K, r.ldk, p->dtype, r.diag.as<double>(), st);
  } else {
    fail(RLD_ERR_INVALID_ARGUMENT, "unknown source");
  }
  if (!r.kq_ready && r.K && r.path == RLD_PATH_STORED && r.dtype == RLD_FP64 && fp64_product_ozaki() && r.rows > 0) {
    // exact int8 slices of the stored float64 rows for the INT8 tensor-core product (kv_ozaki.cu)
    r.Kq.reserve((size_t)ozaki_bytes(r.rows, r.n, 128));
    r.ksigma.reserve(sizeof(double) * r.rows);
    ozaki_slice(static_cast<const double*>(r.K), r.ldk, r.rows, r.n, 128, r.Kq.as<int8_t>(), r.ksigma.as<double>(),
                st);
    r.kq_ready = true;
  }
  if (r.tiled && r.K && r.rows > 0) {
    r.rowscale.reserve(sizeof(float) * r.rows);
    kv_rowscales(static_cast<const float*>(r.K), r.rows, r.n, r.rowscale.as<float>(), st);
  }
  if (r.kq_ready && r.kslices == 7 && !r.kr_ready && !r.permuted && crt_supported(r.n)) {
    // the CRT residue image for the wide (sketch) products, where it fits beside the slices
    const int64_t bytes = crt_bytes(r.rows, r.n);
    size_t fr = 0, tot = 0;
    if (!r.kq_ready && r.Kq.bytes > ((size_t)1 << 30)) {
    // a large slice image of an earlier problem (grow-only buffers) would starve this one's workspaces
    r.Kq.release();
    r.koff.release();
    r.knz.release();
  }
  RLD_CUDA(cudaStreamSynchronize(st));
    RLD_CUDA(cudaMemGetInfo(&fr, &tot));
    if ((int64_t)r.Kr.bytes >= bytes || (int64_t)fr > bytes + (int64_t)(tot / 16)) {
      r.Kr.reserve((size_t)bytes);
      crt_residues(r.Kq.as<int8_t>(), r.rows, r.n, r.Kr.as<int8_t>(), st);
      r.kr_ready = true;
    }
  }
  RLD_CUDA(cudaStreamSynchronize(st));
  r.ready = true;
}

// rows (m x rows_local, row stride ld) <- host/device rows (m x n, global stride n), local columns only
void load_rows(rld_handle* h, const double* src, int memory, int64_t m, double* dst) {
  const Resident& r = h->res;
  RLD_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * r.rows, src + r.row0, sizeof(double) * r.n,
                             sizeof(double) * r.rows, m,
                             memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
}

// m x rows_local (local rows layout) -> m x n full rows on every rank
// Row shards: rank g owns columns [g L, g L + rows_g) of every n-vector, L = ceil(n / G).
// The gather packs the local m x rows block into an m x L send buffer (zero pad),
// ncclAllGather's it into [G][m][L], and a relayout kernel writes the m x n rows
// layout every K x block product reads (the one per-iteration exchange).
void gather_rows(rld_handle* h, const double* local, int64_t m, double* full) {
  const Resident& r = h->res;
  if (h->world == 1) {
    if (local != full) copy_doubles(m * r.n, local, full, h->st);
    return;
  }
  const int64_t L = ceil_div(r.n, h->world);
  Work& wk = h->wk;
  wk.gsend.reserve(sizeof(double) * m * L);
  wk.grecv.reserve(sizeof(double) * m * L * h->world);
  double* snd = wk.gsend.as<double>();
  double* rcv = wk.grecv.as<double>();
  if (r.rows < L) RLD_CUDA(cudaMemsetAsync(snd, 0, sizeof(double) * m * L, h->st));
  if (r.rows > 0)
    RLD_CUDA(cudaMemcpy2DAsync(snd, sizeof(double) * L, local, sizeof(double) * r.rows, sizeof(double) * r.rows, m,
                               cudaMemcpyDeviceToDevice, h->st));
  h->comm->allgather(snd, rcv, m * L, h->st);
  relayout_gathered(rcv, h->world, m, L, r.n, full, h->st);
}

// m rows of length n into the resident point order, in place (no-op unless the points were
// reordered at prepare: one GPU only)
void to_resident_order(rld_handle* h, int64_t m, double* V, int64_t ld) {
  Resident& r = h->res;
  if (!r.permuted || m <= 0) return;
  h->wk.ptmp.reserve(sizeof(double) * m * r.n);
  permute_rows(m, r.n, r.perm.as<int>(), V, ld, h->wk.ptmp.as<double>(), r.n, false, h->st);
  RLD_CUDA(cudaMemcpy2DAsync(V, sizeof(double) * ld, h->wk.ptmp.ptr, sizeof(double) * r.n, sizeof(double) * r.n, m,
                             cudaMemcpyDeviceToDevice, h->st));
}

// Y (m x rows) = V (m x n full) K^T restricted to the local rows
// Y (m x rows) = V (m x n full) K^T restricted to the local rows.  tc_mode 1 =
// single-pass TF32 on the tensor cores (power-iteration sketch products only),
// 3 = 3xTF32 (everything whose value enters the estimate directly).
void kv(rld_handle* h, int64_t m, const double* Vfull, double* Y, int tc_mode = 3, int oz_diags = 7) {
  KvOperand op = h->res.op();
  op.tc_mode = tc_mode;
  op.oz_diags = oz_diags;
  kv_product(op, m, Vfull, op.n, Y, op.rows, h->wk.kv, h->st, nullptr);
}


// ---- float64 products of the estimate outside K x V, on the FP64 tensor cores (kv_dmma.cu).
// Both operands' rows must start 16-byte aligned (even leading dimensions: every BASELINE shape);
// otherwise -- odd n or an odd shard offset -- the same product runs on cuBLAS.
//
// nt_f64: C (q x p, ld ldc) = beta C + A B^T for A: p x n, B: q x n (rows layout); in column-major
// terms C = A^T B.  The Grams, projections and U^T W of the preconditioner and its apply.
void nt_f64(rld_handle* h, const double* A, int64_t lda, int64_t p, const double* B, int64_t ldb, int64_t q, int64_t n,
            double* C, int64_t ldc, double beta = 0.0) {
  if (n <= 0) {   // a rank without rows: its partial is zero
    if (beta == 0.0 && p > 0 && q > 0)
      RLD_CUDA(cudaMemset2DAsync(C, sizeof(double) * ldc, 0, sizeof(double) * p, q, h->st));
    return;
  }
  if (gemm_nt_f64_ok(A, lda, B, ldb)) {
    gemm_nt_f64(A, lda, p, B, ldb, q, n, C, ldc, beta, h->wk.gram_scratch, h->st);
    return;
  }
  if (lda < std::max<int64_t>(1, n) || ldb < std::max<int64_t>(1, n) || ldc < std::max<int64_t>(1, p))
    fail(RLD_ERR_INVALID_ARGUMENT, "nt_f64: p " + std::to_string(p) + " q " + std::to_string(q) + " n " + std::to_string(n) +
                                       " lda " + std::to_string(lda) + " ldb " + std::to_string(ldb) + " ldc " +
                                       std::to_string(ldc));
  RLD_CUBLAS(cublasDgemm(h->cublas, CUBLAS_OP_T, CUBLAS_OP_N, (int)p, (int)q, (int)n, &ONE, A, (int)lda, B, (int)ldb,
                         &beta, C, (int)ldc));
}

// ex_f64: C (q x N rows layout, ld ldc) = beta C + alpha S^T X for S: p x q column-major, X: p x N
// rows layout; in column-major terms C = X S.  Basis changes and low-rank expansions.
void ex_f64(rld_handle* h, const double* S, int64_t lds, int64_t p, int64_t q, const double* X, int64_t ldx, int64_t N,
            double* C, int64_t ldc, double alpha = 1.0, double beta = 0.0, bool tri_upper = false) {
  if (N <= 0 || q <= 0) return;   // a rank without rows
  if (gemm_nt_f64_ok(S, lds, X, ldx)) {
    gemm_expand_f64(S, lds, p, q, X, ldx, N, C, ldc, alpha, beta, h->st, tri_upper);
    return;
  }
  RLD_CUBLAS(cublasDgemm(h->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)q, (int)p, &alpha, X, (int)ldx, S, (int)lds,
                         &beta, C, (int)ldc));
}

// G (w x w, full) = Y^T Y for the rows x w column-major block (fixed-order split-k, deterministic).
void gram_blas(rld_handle* h, int64_t rows, int w, const double* Y, int64_t ldy, double* G) {
  nt_f64(h, Y, ldy, w, Y, ldy, w, rows, G, w);
}

// In-place row orthonormalisation of the w x n block Y (col-major n x w), two
// Cholesky-QR passes.  Replaces the row-wise CGS2 of src/linalg.py:159-180:
// both give the unique Q with positive-diagonal triangular factor.  CholQR2 is
// only accurate while cond(Y) stays below ~1e6 (it squares the condition
// number), so pass 1 flags RLD_FLAG_QR_WEAK when any projected norm R_ii falls
// below 1e-6 |Y_i| (or potrf fails); the caller then redoes the attempt with
// Householder QR, which also decides the reference's RankDeficient test.
// Intermediate power iterations use one pass (`passes` = 1): any triangular
// re-basis keeps the final Q = qr(K^q Omega) unchanged, so only the last
// iteration needs the second pass for orthogonality.
// Upper Cholesky of the w x w fp64 matrix G (ld w): the one-cluster kernel for w <= 640
// (small_chol.cu), cuSOLVER potrf above that.  RLD_SMALL_CHOL=0 forces cuSOLVER.
// Returns true when R^-1 was written to `rinv` as well (only the one-cluster kernel does).
// Above 640: 2 x 2 block recursion on the same kernels (no cuSOLVER on the default path):
//   R11 = chol(G11) with X11 = R11^-1 (the cluster kernel, or this recursion), R12 = X11^T G12 (DMMA
//   nt), S = G22 - R12^T R12 (DMMA nt, symmetric), R22 = chol(S) with X22, and when R^-1 is wanted
//   X12 = -X11 R12 X22 (two DMMA expands).  The leading block is a multiple of 32 columns (half of
//   n), so every sub-factorisation is itself <= 640 or recursed.  info as potrf: first failing pivot.
// G column-major (ld), upper part read and written; X (if not null) n x n, ld n, upper part.
void blocked_potrf_upper(rld_handle* h, int n, double* G, int64_t ld, int* info, double* X) {
  cudaStream_t st = h->st;
  const int n1 = (n / 2 + 31) / 32 * 32, n2 = n - n1;
  double *x11 = nullptr, *x22 = nullptr, *r12 = nullptr, *t = nullptr;
  int* inf = nullptr;
  RLD_CUDA(cudaMallocAsync(&x11, sizeof(double) * n1 * n1, st));
  RLD_CUDA(cudaMallocAsync(&r12, sizeof(double) * n1 * n2, st));
  RLD_CUDA(cudaMallocAsync(&t, sizeof(double) * std::max<int64_t>((int64_t)n2 * n2, (int64_t)n1 * n2), st));
  RLD_CUDA(cudaMallocAsync(&inf, sizeof(int) * 2, st));
  if (X) RLD_CUDA(cudaMallocAsync(&x22, sizeof(double) * n2 * n2, st));
  auto sub = [&](int m, double* A, int64_t lda, int* i, double* Xs) {
    if (!small_potrf_upper(m, A, (int)lda, i, st, Xs)) blocked_potrf_upper(h, m, A, lda, i, Xs);
  };
  sub(n1, G, ld, inf, x11);
  // R12 = X11^T G12  (n1 x n2), then into the upper right block of G
  nt_f64(h, x11, n1, n1, G + (int64_t)n1 * ld, ld, n2, n1, r12, n1);
  RLD_CUDA(cudaMemcpy2DAsync(G + (int64_t)n1 * ld, sizeof(double) * ld, r12, sizeof(double) * n1, sizeof(double) * n1,
                             n2, cudaMemcpyDeviceToDevice, st));
  // S = G22 - R12^T R12
  nt_f64(h, r12, n1, n2, r12, n1, n2, n1, t, n2);
  double* G22 = G + (int64_t)n1 * ld + n1;
  sub_block(n2, n2, t, n2, G22, ld, st);
  sub(n2, G22, ld, inf + 1, x22);
  combine_info(info, inf, inf + 1, n1, st);
  if (X) {
    // X = [[X11, -X11 R12 X22], [0, X22]]
    RLD_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * (size_t)n * n, st));
    RLD_CUDA(cudaMemcpy2DAsync(X, sizeof(double) * n, x11, sizeof(double) * n1, sizeof(double) * n1, n1,
                               cudaMemcpyDeviceToDevice, st));
    RLD_CUDA(cudaMemcpy2DAsync(X + (int64_t)n1 * n + n1, sizeof(double) * n, x22, sizeof(double) * n2,
                               sizeof(double) * n2, n2, cudaMemcpyDeviceToDevice, st));
    ex_f64(h, x22, n2, n2, n2, r12, n1, n1, t, n1);                    // T = R12 X22  (n1 x n2)
    ex_f64(h, t, n1, n1, n2, x11, n1, n1, X + (int64_t)n1 * n, n, -1.0);   // X12 = -X11 T
  }
  RLD_CUDA(cudaFreeAsync(x11, st));
  RLD_CUDA(cudaFreeAsync(r12, st));
  RLD_CUDA(cudaFreeAsync(t, st));
  RLD_CUDA(cudaFreeAsync(inf, st));
  if (x22) RLD_CUDA(cudaFreeAsync(x22, st));
}

bool potrf_upper(rld_handle* h, int w, double* G, int* info, double* rinv = nullptr) {
  static const bool small = [] {
    const char* e = getenv("RLD_SMALL_CHOL");
    return !(e && e[0] == '0');
  }();
  if (small && small_potrf_upper(w, G, w, info, h->st, rinv)) return rinv != nullptr;
  if (small && w > 640 && (w % 2) == 0) {   // the DMMA kernels need 16-byte aligned columns
    blocked_potrf_upper(h, w, G, w, info, rinv);
    return rinv != nullptr;
  }
  Work& wk = h->wk;
  int lwork = 0;
  RLD_CUSOLVER(cusolverDnDpotrf_bufferSize(h->solver, CUBLAS_FILL_MODE_UPPER, w, G, w, &lwork));
  wk.solver_work.reserve(sizeof(double) * std::max(lwork, 1));
  RLD_CUSOLVER(cusolverDnDpotrf(h->solver, CUBLAS_FILL_MODE_UPPER, w, G, w, wk.solver_work.as<double>(), lwork, info));
  return false;
}

void cholqr2(rld_handle* h, int64_t n, int w, double* Y, int* flags, int passes = 2) {
  Work& wk = h->wk;
  wk.G.reserve(sizeof(double) * w * w);
  wk.gdiag.reserve(sizeof(double) * w);
  wk.rinv.reserve(sizeof(double) * w * w);
  double* G = wk.G.as<double>();
  double* Ri = wk.rinv.as<double>();
  int* info = wk.ints.as<int>() + 1;
  for (int pass = 0; pass < passes; ++pass) {
    gram_blas(h, n, w, Y, n, G);
    allreduce_sum(h, G, (int64_t)w * w);
    if (pass == 0) diag_copy(w, G, wk.gdiag.as<double>(), h->st);
    const bool have_rinv = potrf_upper(h, w, G, info, Ri);
    if (pass == 0) cholqr_check(w, G, wk.gdiag.as<double>(), info, 1e-6, flags, h->st);
    if (have_rinv && n > 0) {   // Y <- Y R^-1 through a scratch copy (the expand kernel is out of place)
      wk.scratch2.reserve(sizeof(double) * n * w);
      copy_doubles(n * (int64_t)w, Y, wk.scratch2.as<double>(), h->st);
      ex_f64(h, Ri, w, w, w, wk.scratch2.as<double>(), n, n, Y, n, 1.0, 0.0, true);   // (R^-1 upper triangular)
    } else if (n > 0) {   // (a rank without rows has nothing to change)
      RLD_CUBLAS(cublasDtrsm(h->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                             (int)n, w, &ONE, G, w, Y, (int)n));
    }
  }
}

// One GPU: the same CholQR with the basis change as a DGEMM with an explicit R^-1 (a w x w
// triangular solve on the identity), written straight into `dst` (the full-rows buffer, so no
// gather copy): dst = src R^-1 (one pass) or dst = (src R1^-1) R2^-1 (two passes, through `src`).
// cuBLAS DTRSM on the n x w block was ~143 us at config 2 (n = 16384, w = 266).
void cholqr_gemm(rld_handle* h, int64_t n, int w, double* src, double* dst, int* flags, int passes) {
  Work& wk = h->wk;
  wk.G.reserve(sizeof(double) * w * w);
  wk.gdiag.reserve(sizeof(double) * w);
  wk.rinv.reserve(sizeof(double) * w * w);
  double* G = wk.G.as<double>();
  double* Ri = wk.rinv.as<double>();
  int* info = wk.ints.as<int>() + 1;
  double* cur = src;
  for (int pass = 0; pass < passes; ++pass) {
    double* out = (pass == passes - 1) ? dst : (cur == src ? dst : src);
    if (passes == 2 && pass == 0) out = dst;
    if (passes == 2 && pass == 1) out = src;
    gram_blas(h, n, w, cur, n, G);
    if (pass == 0) diag_copy(w, G, wk.gdiag.as<double>(), h->st);
    const bool have_rinv = potrf_upper(h, w, G, info, Ri);   // the cluster kernel also writes R^-1
    if (pass == 0) cholqr_check(w, G, wk.gdiag.as<double>(), info, 1e-6, flags, h->st);
    if (!have_rinv) {
      RLD_CUDA(cudaMemsetAsync(Ri, 0, sizeof(double) * w * w, h->st));
      add_identity(w, Ri, h->st);
      RLD_CUBLAS(cublasDtrsm(h->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, w,
                             w, &ONE, G, w, Ri, w));
    }
    ex_f64(h, Ri, w, w, w, cur, n, n, out, n, 1.0, 0.0, true);   // out = cur R^-1 (upper triangular: half the k loop)
    cur = out;
  }
  if (cur != dst) copy_doubles(n * (int64_t)w, cur, dst, h->st);
}

// Default on (RLD_CHOLQR_GEMM=0 restores the DTRSM path): with R^-1 from the cluster Cholesky
// kernel the config-2 estimate takes 18.8 vs 19.2 ms (with cuBLAS's triangular solve on the w x w
// identity instead it measured even, 19.33 vs 19.35 ms).
bool cholqr_gemm_enabled() {
  static const bool on = !(getenv("RLD_CHOLQR_GEMM") && getenv("RLD_CHOLQR_GEMM")[0] == '0');
  return on;
}

// Householder QR of Y (col-major n x w, local rows), Q with positive R diagonal -- the same Q
// CGS2 produces -- and the reference's rank test |R_ii| < rtol |Y_i| (src/linalg.py:177-178).
// Row shards (world > 1): TSQR -- local Householder QR Y_g = Q_g R_g, all-gather of the R_g,
// one replicated QR of the stacked [R_0; ...; R_{G-1}] = Q_s R, local Q = Q_g Q_s[g] -- so the
// rank test sees the global R, exactly as on one GPU (up to rounding).
void qr_householder(rld_handle* h, int64_t n, int w, double* Y, double rtol, int* flags) {
  Work& wk = h->wk;
  wk.gdiag.reserve(sizeof(double) * 2 * w);
  wk.G.reserve(sizeof(double) * std::max<int64_t>((int64_t)w * w, 2 * w));
  double* norms2 = wk.gdiag.as<double>();
  double* tau = wk.G.as<double>();
  double* sgn = norms2 + w;
  int* info = wk.ints.as<int>() + 1;
  rows_dot(w, n, Y, n, Y, n, norms2, wk.scratch, h->st, nullptr);
  int l1 = 0, l2 = 0;
  if (h->world == 1) {
    RLD_CUSOLVER(cusolverDnDgeqrf_bufferSize(h->solver, (int)n, w, Y, (int)n, &l1));
    RLD_CUSOLVER(cusolverDnDorgqr_bufferSize(h->solver, (int)n, w, w, Y, (int)n, tau, &l2));
    wk.solver_work.reserve(sizeof(double) * std::max(std::max(l1, l2), 1));
    RLD_CUSOLVER(cusolverDnDgeqrf(h->solver, (int)n, w, Y, (int)n, tau, wk.solver_work.as<double>(), l1, info));
    householder_check(w, Y, n, norms2, rtol, sgn, flags, h->st);
    RLD_CUSOLVER(cusolverDnDorgqr(h->solver, (int)n, w, w, Y, (int)n, tau, wk.solver_work.as<double>(), l2, info));
    scale_cols_colmajor(n, w, n, sgn, Y, h->st);
    return;
  }
  if (n < w) fail(RLD_ERR_NOT_SUPPORTED, "TSQR needs at least w = " + std::to_string(w) + " rows per shard");
  allreduce_sum(h, norms2, w);
  const int G = h->world;
  const int64_t gw = (int64_t)G * w, ww = (int64_t)w * w;
  wk.gsend.reserve(sizeof(double) * ww);
  wk.grecv.reserve(sizeof(double) * ww * G);
  wk.scratch2.reserve(sizeof(double) * std::max<int64_t>(gw * w, n * w));
  wk.qtile.reserve(sizeof(double) * gw * w);
  double* S = wk.qtile.as<double>();
  // local factor
  RLD_CUSOLVER(cusolverDnDgeqrf_bufferSize(h->solver, (int)n, w, Y, (int)n, &l1));
  RLD_CUSOLVER(cusolverDnDorgqr_bufferSize(h->solver, (int)n, w, w, Y, (int)n, tau, &l2));
  int l3 = 0, l4 = 0;
  RLD_CUSOLVER(cusolverDnDgeqrf_bufferSize(h->solver, (int)gw, w, S, (int)gw, &l3));
  RLD_CUSOLVER(cusolverDnDorgqr_bufferSize(h->solver, (int)gw, w, w, S, (int)gw, tau, &l4));
  wk.solver_work.reserve(sizeof(double) * std::max(std::max(std::max(l1, l2), std::max(l3, l4)), 1));
  double* work = wk.solver_work.as<double>();
  RLD_CUSOLVER(cusolverDnDgeqrf(h->solver, (int)n, w, Y, (int)n, tau, work, std::max(l1, l2), info));
  copy_upper(w, Y, n, wk.gsend.as<double>(), h->st);
  RLD_CUSOLVER(cusolverDnDorgqr(h->solver, (int)n, w, w, Y, (int)n, tau, work, std::max(l1, l2), info));
  // stacked R factors, replicated QR
  h->comm->allgather(wk.gsend.as<double>(), wk.grecv.as<double>(), ww, h->st);
  relayout_gathered(wk.grecv.as<double>(), G, w, w, gw, S, h->st);   // (G w) x w column-major
  RLD_CUSOLVER(cusolverDnDgeqrf(h->solver, (int)gw, w, S, (int)gw, tau, work, std::max(l3, l4), info));
  householder_check(w, S, gw, norms2, rtol, sgn, flags, h->st);
  RLD_CUSOLVER(cusolverDnDorgqr(h->solver, (int)gw, w, w, S, (int)gw, tau, work, std::max(l3, l4), info));
  // Q_local = Q_g Q_s[g], then the sign fix
  double* out = wk.scratch2.as<double>();
  ex_f64(h, S + (int64_t)h->rank * w, gw, w, w, Y, n, n, out, n);
  copy_doubles(n * (int64_t)w, out, Y, h->st);
  scale_cols_colmajor(n, w, n, sgn, Y, h->st);
}

void syevd(rld_handle* h, int k, double* A, double* evals) {
  Work& wk = h->wk;
  // tridiagonalisation + multisection + inverse iteration (tri_eig.cu) for k <= 288, then
  // Newton-Schulz orthogonalisation of T's eigenvectors, Z <- 1.5 Z - 0.5 Z (Z^T Z) (symmetric in
  // the columns; the defect E = Z^T Z - I goes to ~0.75 E^2 per step), and the back-transformation,
  // all on FP64 DGEMMs.  Inverse-iteration vectors are orthogonal to ~eps |T| / gap; the defect is
  // read back (one sync per eigensolve) to pick 1-4 steps, and when it exceeds 0.05 (eigenvalues
  // inside one unreduced block of T closer than that allows) the matrix, still untouched, goes to
  // DSYEVD instead.
  double *Z, *Q, *sp;
  if (tri_eigh(k, A, evals, wk.eig_scratch, &Z, &Q, &sp, h->st, h->st2, h->efork, h->ejoin)) {
    const size_t kk = (size_t)k * k;
    double* G = sp;
    double* Z2 = sp + kk;
    double* defect = sp + 2 * kk;
    nt_f64(h, Z, k, k, Z, k, k, k, G, k);   // G = Z^T Z
    orth_defect(k, G, defect, h->st);
    double hd = 0.0;
    RLD_CUDA(cudaMemcpyAsync(&hd, defect, sizeof(double), cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaStreamSynchronize(h->st));
    if (hd <= 0.05) {
      int steps = 0;
      for (double e = hd; e > 1e-15 && steps < 6; e = 0.75 * e * e + 2e-16) ++steps;
      const double HALF_NEG = -0.5, THREE_HALF = 1.5;
      double* cur = Z;
      double* nxt = Z2;
      for (int it = 0; it < steps; ++it) {
        if (it > 0) nt_f64(h, cur, k, k, cur, k, k, k, G, k);
        copy_doubles((int64_t)kk, cur, nxt, h->st);
        ex_f64(h, G, k, k, k, cur, k, k, nxt, k, HALF_NEG, THREE_HALF);   // nxt = 1.5 Z - 0.5 Z G
        std::swap(cur, nxt);
      }
      ex_f64(h, cur, k, k, k, Q, k, k, A, k);   // A = Q Z
      return;
    }
    if (getenv("RLD_TRI_EIG_DEBUG")) fprintf(stderr, "rld: tri_eigh fallback to DSYEVD (k = %d, defect %.2e)\n", k, hd);
  }
  int* info = wk.ints.as<int>() + 2;
  int lwork = 0;
  RLD_CUSOLVER(cusolverDnDsyevd_bufferSize(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, A, k,
                                           evals, &lwork));
  wk.solver_work.reserve(sizeof(double) * std::max(lwork, 1));
  RLD_CUSOLVER(cusolverDnDsyevd(h->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k, A, k, evals,
                                wk.solver_work.as<double>(), lwork, info));
}

struct PrecondOut {
  int k = 0;              // columns of U (kept ones are nonzero)
  int attempts = 1;
  bool householder = false;
};

// Product precision of the first q-1 power iterations.  The last iteration and
// B = Q K Q^T always run 3xTF32.  Single-pass TF32 in the power iterations
// moved the reduced BASELINE config-4 estimate (clustered points, l = n/4) by
// 2.7e-4 (all iterations) and 2.1e-4 (all but the last), beyond the 1e-4 fp32
// budget, so the default is 3xTF32 everywhere; RLD_SKETCH_MODE=1 opts in to
// single-pass TF32 for the early iterations.
// Slice-pair diagonals of the float64 int8-slice product in the first q-1 power iterations: 6
// (21 of the 28 pairs, dropped terms ~2^-50 of max|K| max|V| per sum term) -- those iterations only
// steer the subspace, which the last full-precision iteration re-forms.  The last iteration,
// B = Q K Q^T and every Lanczos product keep all 7 diagonals; with a CRT residue image the wide
// products run as modular GEMMs instead (full precision).  Measured on config 3 (Morton order,
// 8 x 7-bit slices) against the float64 golden value: all diagonals 5.5e-15, one fewer 4.7e-15, two
// fewer 5.6e-14.  RLD_FP64_SKETCH_DIAGS (1..7, read per call) overrides.
int sketch_oz_diags() {
  const char* e = getenv("RLD_FP64_SKETCH_DIAGS");
  const int v = e ? atoi(e) : 6;
  return v < 1 ? 1 : (v > 7 ? 7 : v);
}

int sketch_tc_mode() {
  static const int mode = [] {
    const char* e = getenv("RLD_SKETCH_MODE");
    return (e && e[0] == '1') ? 1 : 3;
  }();
  return mode;
}

// ints layout: [0] flags [1] potrf info [2] syevd info [3] kept [4] inner-chol info
// scal layout: [0] sum log base [1] 2 sum log diag(inner chol) [2] trace
// Low-rank factor A (n_local x ka, column-major in wk.A) of the randomized truncated SVD
// (src/precond.py:168-198, 264-267).  Returns ka = k.
int lowrank_randsvd(rld_handle* h, const rld_config* c, const rld_inputs* in, PrecondOut& out) {
  Resident& r = h->res;
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  const int64_t n = r.n, nl = r.rows;
  int* flags = wk.ints.as<int>();
  const int k = c->precond_rank;
  const int w = (int)std::min<int64_t>(k + c->oversample, n);
  wk.Y.reserve(sizeof(double) * n * w);       // full rows (gathered) sketch / Q
  wk.Z.reserve(sizeof(double) * nl * w);      // local product rows
  double* Y = wk.Y.as<double>();
  double* Z = wk.Z.as<double>();

  auto read_flags = [&]() {
    int hf = 0;
    RLD_CUDA(cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    return hf;
  };
  for (int attempt = 0; attempt < 2; ++attempt) {
    out.attempts = attempt + 1;
    const double* om = attempt == 0 ? in->omega0 : in->omega1;
    const uint64_t* okey = c->omega_key + 2 * attempt;   // stream (seed, (1, attempt))
    int hflags = 0;
    for (int householder = 0; householder < 2; ++householder) {
      if (om)
        RLD_CUDA(cudaMemcpyAsync(Y, om, sizeof(double) * w * n,
                                 in->memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
      else  // numpy-exact Gaussian sketch rows, generated on the device (src/precond.py:183)
        normal_rows(okey, w, n, 0, n, n, Y, wk.rng_scratch, wk.ints.as<int>() + 5, st);
      to_resident_order(h, w, Y, n);
      RLD_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), st));
      for (int it = 0; it < c->precond_iters; ++it) {
        const bool last = it + 1 == c->precond_iters;
        kv(h, w, Y, Z, last ? 3 : sketch_tc_mode(), last ? 7 : sketch_oz_diags());   // Y <- Y M (src/precond.py:186)
        if (householder) {
          qr_householder(h, nl, w, Z, c->orth_rtol, flags);
          gather_rows(h, Z, w, Y);
        } else if (h->world == 1 && cholqr_gemm_enabled()) {
          cholqr_gemm(h, nl, w, Z, Y, flags, last ? 2 : 1);   // Q <- orth(Y), straight into Y
        } else {
          cholqr2(h, nl, w, Z, flags, last ? 2 : 1);      // Q <- orth(Y)  (src/precond.py:187)
          gather_rows(h, Z, w, Y);
        }
      }
      hflags = read_flags();
      if (!householder && !(hflags & RLD_FLAG_QR_WEAK)) break;
      out.householder = true;
    }
    if (hflags & RLD_FLAG_RANK_DEFICIENT) {
      if (attempt == 1) fail(RLD_ERR_RANK_DEFICIENT, "row is numerically dependent (after retry)");
      continue;
    }
    break;
  }
  // B = Q M Q^T (src/precond.py:189); Q full rows in Y, local rows of Q at Y + row0
  kv(h, w, Y, Z);
  wk.C.reserve(sizeof(double) * std::max<int64_t>((int64_t)w * w, (int64_t)k * k));
  double* B = wk.C.as<double>();
  const double* Ql = Y + r.row0;  // col-major n x w, local rows start at row0
  nt_f64(h, Ql, n, w, Z, nl, w, nl, B, w);   // B = Q_l^T (K Q^T)_l
  allreduce_sum(h, B, (int64_t)w * w);
  wk.theta.reserve(sizeof(double) * w);
  syevd(h, w, B, wk.theta.as<double>());                  // src/precond.py:190
  wk.Vtop.reserve(sizeof(double) * w * std::max(k, 1));
  wk.theta_top.reserve(sizeof(double) * std::max(k, 1));
  top_eigvecs(w, k, B, wk.theta.as<double>(), wk.Vtop.as<double>(), wk.theta_top.as<double>(), st);
  // A = (Q^T U_top) sqrt(max(theta, 0))  (src/precond.py:191-193, 264)
  wk.A.reserve(sizeof(double) * nl * k);
  double* A = wk.A.as<double>();
  ex_f64(h, wk.Vtop.as<double>(), w, w, k, Ql, n, nl, A, nl);   // A = Q_l V_top
  return k;
}

// All-rank (value, index) of the first largest local-row entry of d (np.argmax rule) into pv[0..1]
void global_argmax(rld_handle* h, const double* d, double* pv) {
  Resident& r = h->res;
  Work& wk = h->wk;
  if (h->world == 1) {   // ties: the smallest original index, also when the points were reordered
    argmax_first(r.rows, d, r.row0, pv, wk.scratch, h->st, r.permuted ? r.perm.as<int>() : nullptr);
    return;
  }
  wk.gsend.reserve(sizeof(double) * 2);
  wk.grecv.reserve(sizeof(double) * 2 * h->world);
  const int* perm = r.permuted ? r.perm.as<int>() : nullptr;   // ties: the smallest ORIGINAL index
  argmax_first(r.rows, d, r.row0, wk.gsend.as<double>(), wk.scratch, h->st, perm ? perm + r.row0 : nullptr);
  h->comm->allgather(wk.gsend.as<double>(), wk.grecv.as<double>(), 2, h->st);
  pick_first_max(h->world, wk.grecv.as<double>(), pv, h->st, perm);   // ranks hold increasing row ranges
}

// Rank-k pivoted partial Cholesky with greedy largest-diagonal pivoting (src/precond.py:215-228):
// A = C (n_local x ka), ka < k when the residual diagonal runs out (d[p] <= 0).
int lowrank_pchol(rld_handle* h, const rld_config* c) {
  Resident& r = h->res;
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  const int64_t nl = r.rows;
  const int k = c->precond_rank;
  wk.A.reserve(sizeof(double) * std::max<int64_t>(1, nl) * std::max(k, 1));
  wk.Tg.reserve(sizeof(double) * std::max<int64_t>(2 * nl, k + 2));   // residual diagonal d + column buffer
  wk.coef.reserve(sizeof(double) * (k + 2));
  double* C = wk.A.as<double>();
  double* d = wk.Tg.as<double>();
  double* col = d + nl;
  double* crow = wk.coef.as<double>();
  double* pv = wk.scal.as<double>() + 4;   // (value, index) of the pivot
  copy_doubles(nl, r.diag.as<double>(), d, st);
  const KvOperand op = r.op();
  int ka = k;
  for (int j = 0; j < k; ++j) {
    global_argmax(h, d, pv);
    double hp[2];
    RLD_CUDA(cudaMemcpyAsync(hp, pv, sizeof hp, cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    if (!(hp[0] > 0.0)) {   // src/precond.py:221-223
      ka = j;
      break;
    }
    const int64_t p = (int64_t)hp[1];
    kernel_column(nl, r.row0, r.n, p, op.K, op.ldk, op.dtype, op.tiled, r.X.as<double>(), r.kp, col, st);
    if (j > 0) {   // col -= C[:, :j] C[p, :j]
      row_of_owner(nl, r.row0, pv, C, j, crow, st);
      allreduce_sum(h, crow, j);
      const double MONE = -1.0;
      RLD_CUBLAS(cublasDgemv(h->cublas, CUBLAS_OP_N, (int)nl, j, &MONE, C, (int)std::max<int64_t>(1, nl), crow, 1,
                             &ONE, col, 1));
    }
    pchol_update(nl, col, pv, C + (size_t)j * nl, d, st);
  }
  return ka;
}

// Top-k eigenpairs of the dense K in float64 (src/precond.py:260-263), one GPU.
int lowrank_truncsvd(rld_handle* h, const rld_config* c) {
  Resident& r = h->res;
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  if (h->world != 1) fail(RLD_ERR_NOT_SUPPORTED, "trunc-svd needs the dense K on one GPU");
  const int64_t n = r.n;
  const int k = c->precond_rank;
  DevBuf L, W;
  L.reserve(sizeof(double) * n * n);
  W.reserve(sizeof(double) * n);
  if (r.path == RLD_PATH_ON_THE_FLY || !r.K)
    build_kernel_rows<double>(r.X.as<double>(), n, r.kp, 0, n, L.as<double>(), n, st);
  else if (r.tiled)
    untile_to_f64(static_cast<const float*>(r.K), n, n, L.as<double>(), n, st);
  else
    convert_rows_2d(r.K, r.dtype, r.ldk, L.as<double>(), n, n, st);
  cusolverDnParams_t params;
  RLD_CUSOLVER(cusolverDnCreateParams(&params));
  size_t dws = 0, hws = 0;
  RLD_CUSOLVER(cusolverDnXsyevd_bufferSize(h->solver, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                           CUDA_R_64F, L.ptr, n, CUDA_R_64F, W.ptr, CUDA_R_64F, &dws, &hws));
  DevBuf dwork;
  dwork.reserve(std::max<size_t>(dws, 8));
  std::vector<char> hwork(std::max<size_t>(hws, 8));
  RLD_CUSOLVER(cusolverDnXsyevd(h->solver, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F,
                                L.ptr, n, CUDA_R_64F, W.ptr, CUDA_R_64F, dwork.ptr, dws, hwork.data(), hws,
                                wk.ints.as<int>() + 2));
  cusolverDnDestroyParams(params);
  wk.A.reserve(sizeof(double) * n * std::max(k, 1));
  wk.theta_top.reserve(sizeof(double) * std::max(k, 1));
  // A[:, r] = V[:, n-1-r] sqrt(max(theta, 0)) (descending order, src/precond.py:262-263)
  if (k > 0) top_eigvecs((int)n, k, L.as<double>(), W.as<double>(), wk.A.as<double>(), wk.theta_top.as<double>(), st);
  RLD_CUDA(cudaStreamSynchronize(st));   // L, W go out of scope
  return k;
}

// Dominant eigenpair by power iteration (src/precond.py:201-213, 249-251): A = sqrt(max(lam, floor)) v.
int lowrank_rankone(rld_handle* h, const rld_config* c) {
  Resident& r = h->res;
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  const int64_t n = r.n, nl = r.rows;
  const int max_iters = std::max(100, c->precond_iters * std::max(c->precond_rank, 1));
  wk.Y.reserve(sizeof(double) * std::max<int64_t>(n, 1));
  wk.A.reserve(sizeof(double) * std::max<int64_t>(nl, 1));
  wk.Tg.reserve(sizeof(double) * std::max<int64_t>(nl, 1));
  double* vfull = wk.Y.as<double>();
  double* v = wk.A.as<double>();     // local rows of v, and finally A
  double* w = wk.Tg.as<double>();
  double* dd = wk.scal.as<double>() + 4;   // [0] v.w  [1] w.w  [2] v.v
  normal_rows(c->precond_key, 1, n, 0, n, n, vfull, wk.rng_scratch, wk.ints.as<int>() + 5, st);   // rng.normal(n)
  to_resident_order(h, 1, vfull, n);
  rows_dot(1, n, vfull, n, vfull, n, dd + 2, wk.scratch, st, nullptr);
  scale_by(n, vfull, dd + 2, 0, st);                                   // v /= |v|
  copy_doubles(nl, vfull + r.row0, v, st);
  double lam = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    kv(h, 1, vfull, w);                                                // w = M v
    rows_dot(1, nl, v, nl, w, nl, dd, wk.scratch, st, nullptr);
    rows_dot(1, nl, w, nl, w, nl, dd + 1, wk.scratch, st, nullptr);
    allreduce_sum(h, dd, 2);
    copy_doubles(nl, w, v, st);
    scale_by(nl, v, dd + 1, 0, st);                                    // v = w / |w|
    gather_rows(h, v, 1, vfull);
    double hv = 0.0;
    RLD_CUDA(cudaMemcpyAsync(&hv, dd, sizeof hv, cudaMemcpyDeviceToHost, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    const bool done = lam != 0.0 && std::fabs(hv - lam) <= 1e-10 * std::fabs(hv);
    lam = hv;
    if (done) break;
  }
  fill_doubles(1, lam, dd, st);
  scale_by(nl, v, dd, 1, st);                                          // A = sqrt(max(lam, 1e-12)) v
  RLD_CUDA(cudaStreamSynchronize(st));
  return 1;
}

PrecondOut build_preconditioner(rld_handle* h, const rld_config* c, const rld_inputs* in) {
  Resident& r = h->res;
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  const int64_t nl = r.rows;
  int* flags = wk.ints.as<int>();
  double* scal = wk.scal.as<double>();
  wk.base.reserve(sizeof(double) * std::max<int64_t>(1, nl));
  wk.sqrt_base.reserve(sizeof(double) * std::max<int64_t>(1, nl));
  double* base = wk.base.as<double>();
  double* sqrt_base = wk.sqrt_base.as<double>();
  PrecondOut out;
  const int kind = c->precond_kind;

  if (kind == RLD_PRECOND_IDENTITY) {
    fill_doubles(nl, 1.0, base, st);
    fill_doubles(nl, 1.0, sqrt_base, st);
    fill_doubles(2, 0.0, scal, st);
    return out;
  }
  if (kind == RLD_PRECOND_DIAGONAL) {
    copy_doubles(nl, r.diag.as<double>(), base, st);
    sqrt_into(nl, base, sqrt_base, flags, st);
    sum_log(nl, base, scal, wk.scratch, st);
    allreduce_sum(h, scal, 1);
    fill_doubles(1, 0.0, scal + 1, st);
    return out;
  }
  int k = 0;
  bool scaled = false;
  switch (kind) {
    case RLD_PRECOND_RAND_SVD_SCALED: scaled = true; [[fallthrough]];
    case RLD_PRECOND_RAND_SVD: k = lowrank_randsvd(h, c, in, out); break;
    case RLD_PRECOND_PARTIAL_CHOLESKY_SCALED: scaled = true; [[fallthrough]];
    case RLD_PRECOND_PARTIAL_CHOLESKY: k = lowrank_pchol(h, c); break;
    case RLD_PRECOND_TRUNC_SVD_SCALED: scaled = true; [[fallthrough]];
    case RLD_PRECOND_TRUNC_SVD: k = lowrank_truncsvd(h, c); break;
    case RLD_PRECOND_RANK_ONE: k = lowrank_rankone(h, c); break;
    default: fail(RLD_ERR_NOT_SUPPORTED, "unknown preconditioner kind " + std::to_string(kind));
  }
  wk.A.reserve(sizeof(double) * std::max<int64_t>(1, nl) * std::max(k, 1));
  wk.Z.reserve(sizeof(double) * std::max<int64_t>(1, nl) * std::max(k, 1));
  double* A = wk.A.as<double>();
  double* Z = wk.Z.as<double>();
  // base: floored residual diagonal max(diag M - sum A^2, 1e-12) (src/precond.py:231-233) or the
  // scale of the "-scaled" kinds; At = A / sqrt(base) (src/precond.py:94-95)
  if (scaled)
    precond_base_scaled(nl, k, c->precond_scale, A, base, sqrt_base, st);
  else
    precond_base(nl, k, r.diag.as<double>(), c->diag_floor, A, base, sqrt_base, st);
  sum_log(nl, base, scal, wk.scratch, st);
  allreduce_sum(h, scal, 1);
  RLD_CUDA(cudaMemsetAsync(wk.ints.as<int>() + 3, 0, sizeof(int), st));
  if (k == 0) {   // P = diag(base)
    fill_doubles(1, 0.0, scal + 1, st);
    out.k = 0;
    return out;
  }
  // C = At^T At ; inner = I + C ; log det inner by Cholesky (src/precond.py:75-80)
  wk.C.reserve(sizeof(double) * k * k);
  double* C = wk.C.as<double>();
  gram_blas(h, nl, k, A, nl, C);
  allreduce_sum(h, C, (int64_t)k * k);
  wk.inner.reserve(sizeof(double) * k * k);
  double* inner = wk.inner.as<double>();
  copy_doubles((int64_t)k * k, C, inner, st);
  add_identity(k, inner, st);
  // log det of the inner factor on the side stream, overlapping the eigensolve of C below (both
  // only read C / inner); joined at the end of this function
  const bool side = k <= 640 && h->world == 1;
  {
    int* info = wk.ints.as<int>() + 4;
    if (side) {
      RLD_CUDA(cudaEventRecord(h->fork, st));
      RLD_CUDA(cudaStreamWaitEvent(h->st2, h->fork, 0));
      small_potrf_upper(k, inner, k, info, h->st2);   // only the diagonal of the factor is used
      chol_logdet(k, inner, info, scal + 1, flags, h->st2);
      RLD_CUDA(cudaEventRecord(h->join, h->st2));
    } else {
      potrf_upper(h, k, inner, info);
      chol_logdet(k, inner, info, scal + 1, flags, st);
    }
  }
  // factored square root (src/precond.py:90-100): eigh(At^T At), keep filter, U = At W / sqrt(lam)
  wk.lam.reserve(sizeof(double) * k);
  syevd(h, k, C, wk.lam.as<double>());
  wk.hgg.reserve(sizeof(double) * 3 * k);
  double* hv = wk.hgg.as<double>();
  sqrt_factors(k, c->keep_rtol, wk.lam.as<double>(), C, hv, hv + k, hv + 2 * k, wk.ints.as<int>() + 3, st);
  // U (n_local x k) into Z (no longer needed)
  ex_f64(h, C, k, k, k, A, nl, nl, Z, nl);   // U = A W lambda^-1/2
  if (side) RLD_CUDA(cudaStreamWaitEvent(st, h->join, 0));
  out.k = k;
  return out;
}

// build_preconditioner's argument checks (src/precond.py:47-55, 176-177, 241-242)
void validate_precond(const rld_config* c, int64_t n) {
  if (c->precond_rank < 0) fail(RLD_ERR_INVALID_ARGUMENT, "rank must be >= 0");
  if (c->precond_iters < 1) fail(RLD_ERR_INVALID_ARGUMENT, "num_iters must be >= 1");
  const int pk = c->precond_kind;
  if (pk != RLD_PRECOND_IDENTITY && pk != RLD_PRECOND_DIAGONAL && pk != RLD_PRECOND_RANK_ONE && c->precond_rank > n)
    fail(RLD_ERR_INVALID_ARGUMENT, "rank " + std::to_string(c->precond_rank) + " exceeds dimension " + std::to_string(n));
  const bool randsvd = pk == RLD_PRECOND_RAND_SVD || pk == RLD_PRECOND_RAND_SVD_SCALED;
  if (randsvd && c->precond_rank < 1)   // randomized_range_svd (src/precond.py:176-177)
    fail(RLD_ERR_INVALID_ARGUMENT, "rank must be in 1.." + std::to_string(n) + ", got " + std::to_string(c->precond_rank));
  if (!(c->precond_scale > 0) && (pk == RLD_PRECOND_RAND_SVD_SCALED || pk == RLD_PRECOND_PARTIAL_CHOLESKY_SCALED ||
                                  pk == RLD_PRECOND_TRUNC_SVD_SCALED))
    fail(RLD_ERR_INVALID_ARGUMENT, "scale must be positive");
}

// rld_precond_build: build_preconditioner(M, cfg, rng) on its own (src/precond.py:236-267), the
// factors staying in the handle for rld_precond_apply; log det P and the kept rank read back.
void precond_build(rld_handle* h, const rld_config* c, const rld_inputs* in, rld_precond_info* out) {
  NvtxRange nv("rld:precond_build");
  Resident& r = h->res;
  if (!r.ready) fail(RLD_ERR_INVALID_ARGUMENT, "no resident problem (call rld_prepare)");
  if (!c || !out) fail(RLD_ERR_INVALID_ARGUMENT, "config / info is NULL");
  rld_inputs none{};
  if (!in) in = &none;
  validate_precond(c, r.n);
  Work& wk = h->wk;
  wk.ints.reserve(sizeof(int) * 16);
  wk.scal.reserve(sizeof(double) * 16);
  RLD_CUDA(cudaMemsetAsync(wk.ints.ptr, 0, sizeof(int) * 8, h->st));
  g_launches = 0;
  const PrecondOut po = build_preconditioner(h, c, in);
  double hs[2];
  int hi[8];
  RLD_CUDA(cudaMemcpyAsync(hs, wk.scal.ptr, sizeof hs, cudaMemcpyDeviceToHost, h->st));
  RLD_CUDA(cudaMemcpyAsync(hi, wk.ints.ptr, sizeof hi, cudaMemcpyDeviceToHost, h->st));
  RLD_CUDA(cudaStreamSynchronize(h->st));
  int fl[1] = {hi[0]};
  allreduce_flags(h, fl, 1);
  if (fl[0] & RLD_FLAG_NOT_PD) fail(RLD_ERR_NOT_POSITIVE_DEFINITE, "Matrix is not positive definite (inner Cholesky)");
  if (fl[0] & 8) fail(RLD_ERR_INVALID_ARGUMENT, "base diagonal must be strictly positive");
  h->precond_k = po.k;
  out->log_det = hs[0] + hs[1];
  out->rank = po.k;
  out->rank_kept = po.k > 0 ? hi[3] : 0;
  out->attempts = po.attempts;
  out->qr_fallback = po.householder ? 1 : 0;
  out->kernel_launches = g_launches;
}

// rld_precond_apply: Y = op(V) for m rows V (m x n, device) with the factors of the last
// preconditioner build: N^-1 (solve_sqrt, src/precond.py:102-108), N^-T (solve_sqrt_t,
// src/precond.py:110-115) or P^-1 = N^-T N^-1.  One GPU.
void precond_apply(rld_handle* h, int32_t op, int64_t m, const double* V, double* Y) {
  if (h->precond_k < 0) fail(RLD_ERR_INVALID_ARGUMENT, "no preconditioner built (call rld_precond_build)");
  if (h->world != 1) fail(RLD_ERR_NOT_SUPPORTED, "rld_precond_apply is single-GPU");
  if (m < 1 || !V || !Y) fail(RLD_ERR_INVALID_ARGUMENT, "bad precond_apply arguments");
  if (op < RLD_SOLVE_SQRT || op > RLD_SOLVE) fail(RLD_ERR_INVALID_ARGUMENT, "unknown precond op");
  Work& wk = h->wk;
  cudaStream_t st = h->st;
  const int64_t n = h->res.n;
  const int k = h->precond_k;
  const double* U = wk.Z.as<double>();
  const double* hv = wk.hgg.as<double>();
  const double* sqrt_base = wk.sqrt_base.as<double>();
  DevBuf& T = wk.Tg;
  T.reserve(sizeof(double) * std::max<int64_t>(1, (int64_t)k * m));
  const bool perm = h->res.permuted;   // operands in the caller's order, factors in the resident order
  double* const Yout = Y;
  if (perm) {
    wk.ptmp2.reserve(sizeof(double) * m * n);
    Y = wk.ptmp2.as<double>();
    permute_rows(m, n, h->res.perm.as<int>(), V, n, Y, n, false, st);
  } else {
    copy_doubles(m * n, V, Y, st);
  }
  // N^-1 z = w + U (g o U^T w), w = z / sqrt(base);  N^-T x = (x + U (g o U^T x)) / sqrt(base);
  // P^-1 u = (w + U (h o U^T w)) / sqrt(base), w = u / sqrt(base)
  if (op != RLD_SOLVE_SQRT_T) scale_rows_colmajor(n, m, n, sqrt_base, true, Y, st);
  if (k > 0) {
    nt_f64(h, U, n, k, Y, n, m, n, T.as<double>(), k);
    scale_rows_colmajor(k, m, k, op == RLD_SOLVE ? hv : hv + k, false, T.as<double>(), st);
    ex_f64(h, T.as<double>(), k, k, m, U, n, n, Y, n, 1.0, 1.0);
  }
  if (op != RLD_SOLVE_SQRT) scale_rows_colmajor(n, m, n, sqrt_base, true, Y, st);
  if (perm) permute_rows(m, n, h->res.perm.as<int>(), Y, n, Yout, n, true, st);
  RLD_CUDA(cudaStreamSynchronize(st));
}

void run_estimate(rld_handle* h, const rld_config* c, const rld_inputs* in, rld_result* res) {
  NvtxRange nv("rld:estimate");
  Resident& r = h->res;
  if (!r.ready) fail(RLD_ERR_INVALID_ARGUMENT, "no resident problem (call rld_prepare or rld_logdet)");
  if (!c) fail(RLD_ERR_INVALID_ARGUMENT, "config is NULL");
  if (!res) fail(RLD_ERR_INVALID_ARGUMENT, "result is NULL");
  rld_inputs none{};
  if (!in) in = &none;
  if (c->estimator != RLD_ESTIMATOR_RSTAR && c->estimator != RLD_ESTIMATOR_SLQ)
    fail(RLD_ERR_INVALID_ARGUMENT, "unknown estimator " + std::to_string(c->estimator));
  const bool slq = c->estimator == RLD_ESTIMATOR_SLQ;
  rld_config cs = *c;
  if (slq) cs.precond_kind = RLD_PRECOND_IDENTITY;   // SLQ runs on K itself (src/estimators.py:106)
  c = &cs;
  const Partial pf = slq ? Partial{0.0, 0, {}, {}} : partial_fraction(c->order);
  if (c->num_probes < 1 || c->lanczos_iters < 1) fail(RLD_ERR_INVALID_ARGUMENT, "num_probes and lanczos_iters must be >= 1");
  if (c->precond_rank < 0) fail(RLD_ERR_INVALID_ARGUMENT, "rank must be >= 0");
  if (c->precond_iters < 1) fail(RLD_ERR_INVALID_ARGUMENT, "num_iters must be >= 1");
  if (c->probe_kind != RLD_RADEMACHER && c->probe_kind != RLD_GAUSSIAN && c->probe_kind != RLD_NORMAL_ORTHOGONAL)
    fail(RLD_ERR_INVALID_ARGUMENT, "unknown probe kind");
  const int64_t n = r.n, nl = r.rows;
  const int64_t s = c->num_probes;
  const int t = (int)std::min<int64_t>(c->lanczos_iters, n);   // src/estimators.py:62
  validate_precond(c, n);
  cudaStream_t st = h->st;
  Work& wk = h->wk;
  wk.ints.reserve(sizeof(int) * (8 + 2 * s));
  wk.scal.reserve(sizeof(double) * (8 + 4 * s + 2 * s * t + 16));
  RLD_CUDA(cudaMemsetAsync(wk.ints.ptr, 0, sizeof(int) * 8, st));
  g_launches = 0;
  RLD_CUDA(cudaEventRecord(h->ev[0], st));

  // ---- preconditioner
  nvtxRangePushA("rld:preconditioner (sketch, QR, eigensolves, factors)");
  const PrecondOut po = build_preconditioner(h, c, in);
  h->precond_k = po.k;
  RLD_CUDA(cudaEventRecord(h->ev[1], st));
  const int k = po.k;
  const double* U = wk.Z.as<double>();
  const double* hv = wk.hgg.as<double>();
  const double* sqrt_base = wk.sqrt_base.as<double>();

  nvtxRangePop();
  // ---- probes (src/estimators.py:64)
  nvtxRangePushA("rld:probes + Lanczos");
  wk.probes.reserve(sizeof(double) * s * nl);
  double* Zp = wk.probes.as<double>();
  // sharded with the points in Morton order: a rank's rows are scattered through the caller's order,
  // so the probes are generated (or loaded) at full length and this rank's rows gathered from them
  const bool gather_local = h->world > 1 && r.permuted;
  double* Zfull = nullptr;
  if (gather_local) {
    wk.ptmp2.reserve(sizeof(double) * s * n);
    Zfull = wk.ptmp2.as<double>();
  }
  auto local_rows = [&](int64_t m, const double* full, double* out) {
    permute_rows(m, nl, r.perm.as<int>() + r.row0, full, n, out, nl, false, st);
  };
  if (in->probes && gather_local) {
    RLD_CUDA(cudaMemcpyAsync(Zfull, in->probes, sizeof(double) * s * n,
                             in->memory == RLD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    local_rows(s, Zfull, Zp);
  } else if (in->probes) {
    load_rows(h, in->probes, in->memory, s, Zp);
    to_resident_order(h, s, Zp, nl);
  } else if (c->probe_kind == RLD_RADEMACHER && gather_local) {
    rademacher_rows(c->probe_key, s, n, 0, n, n, Zfull, st);
    local_rows(s, Zfull, Zp);
  } else if (c->probe_kind == RLD_RADEMACHER) {
    rademacher_rows(c->probe_key, s, n, r.row0, nl, nl, Zp, st);
    to_resident_order(h, s, Zp, nl);
  } else if (c->probe_kind == RLD_NORMAL_ORTHOGONAL) {
    // src/probes.py:15-22, 36-44: block i of min(s_left, n) rows from stream (seed, (2, i)):
    // Gaussian rows, orthonormalised (CholQR = the CGS2 Q), scaled by chi(n) radii drawn from
    // the same stream right after the rows (host continuation, rng_host.cu)
    wk.endw.reserve(sizeof(int64_t));
    wk.radii.reserve(sizeof(double) * s);
    int64_t done = 0;
    for (int b = 0; done < s; ++b) {
      if (b >= RLD_MAX_PROBE_BLOCKS) fail(RLD_ERR_NOT_SUPPORTED, "normal-orthogonal probes need s <= 4 n");
      const int64_t sb = std::min<int64_t>(s - done, n);
      double* blk = Zp + done * nl;
      const uint64_t* key = c->probe_block_keys + 2 * b;
      if (gather_local) {
        normal_rows(key, sb, n, 0, n, n, Zfull, wk.rng_scratch, wk.ints.as<int>() + 5, st, wk.endw.as<int64_t>());
        local_rows(sb, Zfull, blk);
      } else {
        normal_rows(key, sb, n, r.row0, nl, nl, blk, wk.rng_scratch, wk.ints.as<int>() + 5, st, wk.endw.as<int64_t>());
        to_resident_order(h, sb, blk, nl);
      }
      cholqr2(h, nl, (int)sb, blk, wk.ints.as<int>(), 2);
      int64_t ew = 0;
      RLD_CUDA(cudaMemcpyAsync(&ew, wk.endw.ptr, sizeof ew, cudaMemcpyDeviceToHost, st));
      RLD_CUDA(cudaStreamSynchronize(st));
      std::vector<double> rad((size_t)sb);
      chi_radii_host(key, (uint64_t)ew, n, sb, rad.data());
      RLD_CUDA(cudaMemcpyAsync(wk.radii.ptr, rad.data(), sizeof(double) * sb, cudaMemcpyHostToDevice, st));
      scale_cols_colmajor(nl, sb, nl, wk.radii.as<double>(), blk, st);
      RLD_CUDA(cudaStreamSynchronize(st));   // rad goes out of scope
      done += sb;
    }
  } else if (gather_local) {
    normal_rows(c->probe_key, s, n, 0, n, n, Zfull, wk.rng_scratch, wk.ints.as<int>() + 5, st);
    local_rows(s, Zfull, Zp);
  } else {  // numpy-exact Gaussian probes on the device (src/probes.py:33-34)
    normal_rows(c->probe_key, s, n, r.row0, nl, nl, Zp, wk.rng_scratch, wk.ints.as<int>() + 5, st);
    to_resident_order(h, s, Zp, nl);
  }

  // ---- Lanczos state
  for (DevBuf* b : {&wk.x, &wk.p, &wk.pp, &wk.u, &wk.w, &wk.KX}) b->reserve(sizeof(double) * s * nl);
  wk.T.reserve(sizeof(double) * std::max(k, 1) * s);
  wk.Tg.reserve(sizeof(double) * std::max(k, 1) * s);
  double* x = wk.x.as<double>();
  double* p = wk.p.as<double>();
  double* pp = wk.pp.as<double>();
  double* u = wk.u.as<double>();
  double* wv = wk.w.as<double>();
  double* KX = wk.KX.as<double>();
  double* T = wk.T.as<double>();
  double* Tg = wk.Tg.as<double>();
  double* scal = wk.scal.as<double>();
  double* norms = scal + 8;
  double* dots = norms + s;
  double* alpha = dots + s;
  double* beta = alpha + s * t;
  double* beta_ref = beta + s * t;
  double* per_probe = beta_ref + s;
  double* consts = per_probe + s;      // offset, poles[5], residues[5]
  int* ints = wk.ints.as<int>();
  int* flags = ints;
  int* live = ints + 8;
  int* size = live + s;
  {
    std::vector<int> hl(2 * s);
    for (int64_t i = 0; i < s; ++i) { hl[i] = 1; hl[s + i] = t; }
    RLD_CUDA(cudaMemcpyAsync(live, hl.data(), sizeof(int) * 2 * s, cudaMemcpyHostToDevice, st));
    double hc[11] = {pf.offset};
    for (int q = 0; q < pf.npoles; ++q) { hc[1 + q] = pf.poles[q]; hc[6 + q] = pf.residues[q]; }
    RLD_CUDA(cudaMemcpyAsync(consts, hc, sizeof hc, cudaMemcpyHostToDevice, st));
    RLD_CUDA(cudaStreamSynchronize(st));  // host staging buffers go out of scope
  }
  fill_doubles(2 * s * t, 0.0, alpha, st);

  // q0 = v / |v|; x0 = N^-T q0; p0 = N q0
  rows_dot(s, nl, Zp, nl, Zp, nl, dots, wk.scratch, st, nullptr);
  allreduce_sum(h, dots, s);
  normalize_rows(s, nl, Zp, dots, norms, wv, st);       // q0 in wv
  copy_doubles(s * nl, wv, x, st);
  copy_doubles(s * nl, wv, p, st);
  if (k > 0) {
    nt_f64(h, U, nl, k, wv, nl, s, nl, T, k);                    // T = U^T q0
    allreduce_sum(h, T, (int64_t)k * s);
    copy_doubles((int64_t)k * s, T, Tg, st);
    scale_rows_colmajor(k, s, k, hv + k, false, Tg, st);       // g
    scale_rows_colmajor(k, s, k, hv + 2 * k, false, T, st);    // gamma
    ex_f64(h, Tg, k, k, s, U, nl, nl, x, nl, 1.0, 1.0);        // x += U (g o T)
    ex_f64(h, T, k, k, s, U, nl, nl, p, nl, 1.0, 1.0);         // p += U (gamma o T)
  }
  scale_rows_colmajor(nl, s, nl, sqrt_base, true, x, st);
  scale_rows_colmajor(nl, s, nl, sqrt_base, false, p, st);

  wk.Y.reserve(sizeof(double) * s * n);
  double* xfull = wk.Y.as<double>();
  // SLQ keeps the Lanczos basis for the full reorthogonalisation of src/lanczos.py:60-62:
  // Qb[j] = q_j rows (s x nl); probe c's basis is the nl x (j+1) column-major block at
  // Qb + c nl with leading dimension s nl
  // r* with any preconditioner but the hot path's rand-svd keeps both bases (x_j in Qb, p_j in
  // Pb) for the reference's full reorthogonalisation: weak or "-scaled" preconditioners leave
  // N^-1 K N^-T ill-conditioned, where the three-term recurrence loses orthogonality (fp32 K:
  // 2.7e-3 relative at config 1 with the diagonal P).  rand-svd does not need it.
  const bool reorth = !slq && c->precond_kind != RLD_PRECOND_RAND_SVD;
  double* Qb = nullptr;
  double* Pb = nullptr;
  double* coef = nullptr;
  if (slq || reorth) {
    wk.qbasis.reserve(sizeof(double) * (size_t)t * s * nl);
    wk.coef.reserve(sizeof(double) * (size_t)s * t);
    Qb = wk.qbasis.as<double>();
    coef = wk.coef.as<double>();
  }
  if (reorth) {
    wk.pbasis.reserve(sizeof(double) * (size_t)t * s * nl);
    Pb = wk.pbasis.as<double>();
  }
  int products = 0;
  for (int j = 0; j < t; ++j) {
    if (slq || reorth) copy_doubles(s * nl, x, Qb + (size_t)j * s * nl, st);
    if (reorth) copy_doubles(s * nl, p, Pb + (size_t)j * s * nl, st);
    const double* xin = x;                                // one GPU: the local rows are the full rows
    if (h->world > 1) {
      gather_rows(h, x, s, xfull);
      xin = xfull;
    }
    kv(h, s, xin, KX);                                    // K x_j
    ++products;
    rows_dot(s, nl, x, nl, KX, nl, dots, wk.scratch, st, nullptr);
    allreduce_sum(h, dots, s);
    lanczos_alpha(s, j, t, dots, live, alpha, st);        // alpha_j = q_j . A q_j
    if (j == t - 1) break;
    if (slq) {
      // w = K q_j; two passes w -= Q_j (Q_j^T w) over q_0..q_j (src/lanczos.py:58-62)
      copy_doubles(s * nl, KX, u, st);
      const double MONE = -1.0;
      for (int pass = 0; pass < 2; ++pass) {
        RLD_CUBLAS(cublasDgemvStridedBatched(h->cublas, CUBLAS_OP_T, (int)nl, j + 1, &ONE, Qb, (int)(s * nl), nl, u,
                                             1, nl, &ZERO, coef, 1, t, (int)s));
        if (h->world > 1) allreduce_sum(h, coef, s * t);
        RLD_CUBLAS(cublasDgemvStridedBatched(h->cublas, CUBLAS_OP_N, (int)nl, j + 1, &MONE, Qb, (int)(s * nl), nl,
                                             coef, 1, t, &ONE, u, 1, nl, (int)s));
      }
      rows_dot(s, nl, u, nl, u, nl, dots, wk.scratch, st, nullptr);
      allreduce_sum(h, dots, s);
      lanczos_beta(s, j, t, c->breakdown_rtol, dots, alpha, beta, beta_ref, live, size, st);
      lanczos_advance(s, nl, j, t, beta, live, u, u, p, pp, x, st);
      continue;
    }
    lanczos_residual(s, nl, j, t, KX, alpha, beta, p, pp, sqrt_base, u, wv, st, !reorth);
    if (k > 0) {
      nt_f64(h, U, nl, k, wv, nl, s, nl, T, k);                 // T = U^T w
      allreduce_sum(h, T, (int64_t)k * s);
      scale_rows_colmajor(k, s, k, hv, false, T, st);         // h = 1/(1+lam) - 1
      ex_f64(h, T, k, k, s, U, nl, nl, wv, nl, 1.0, 1.0);     // w += U (h o T)
    }
    scale_rows_colmajor(nl, s, nl, sqrt_base, true, wv, st);  // z = P^-1 u
    if (reorth) {
      // full two-pass reorthogonalisation of src/lanczos.py:60-62 in the two-sequence form:
      // with q_i = N^T x_i = N^-1 p_i and w = A q_j (u = N w, z = N^-T w), q_i.w = p_i.z, so
      // u -= sum_i (p_i.z) p_i and z -= sum_i (p_i.z) x_i keep u = N w and z = N^-T w
      const double MONE = -1.0;
      for (int pass = 0; pass < 2; ++pass) {
        RLD_CUBLAS(cublasDgemvStridedBatched(h->cublas, CUBLAS_OP_T, (int)nl, j + 1, &ONE, Pb, (int)(s * nl), nl, wv,
                                             1, nl, &ZERO, coef, 1, t, (int)s));
        if (h->world > 1) allreduce_sum(h, coef, s * t);
        RLD_CUBLAS(cublasDgemvStridedBatched(h->cublas, CUBLAS_OP_N, (int)nl, j + 1, &MONE, Pb, (int)(s * nl), nl,
                                             coef, 1, t, &ONE, u, 1, nl, (int)s));
        RLD_CUBLAS(cublasDgemvStridedBatched(h->cublas, CUBLAS_OP_N, (int)nl, j + 1, &MONE, Qb, (int)(s * nl), nl,
                                             coef, 1, t, &ONE, wv, 1, nl, (int)s));
      }
    }
    rows_dot(s, nl, u, nl, wv, nl, dots, wk.scratch, st, nullptr);
    allreduce_sum(h, dots, s);
    lanczos_beta(s, j, t, c->breakdown_rtol, dots, alpha, beta, beta_ref, live, size, st);
    lanczos_advance(s, nl, j, t, beta, live, u, wv, p, pp, x, st);
  }
  RLD_CUDA(cudaEventRecord(h->ev[2], st));
  nvtxRangePop();
  NvtxRange nv_solves("rld:shifted solves + Hutchinson");
  if (slq)   // Gauss quadrature of log on each probe's T (src/estimators.py:110-116)
    slq_epilogue(s, t, alpha, beta, size, norms, 1e-300, per_probe, scal + 2, ints + 6, flags, st);
  else
    thomas_hutchinson(s, t, alpha, beta, size, norms, pf.npoles, pf.offset, consts + 1, consts + 6, per_probe,
                      scal + 2, flags, st);
  RLD_CUDA(cudaEventRecord(h->ev[3], st));

  double hs[3];
  int hi[8];
  RLD_CUDA(cudaMemcpyAsync(hs, scal, sizeof hs, cudaMemcpyDeviceToHost, st));
  RLD_CUDA(cudaMemcpyAsync(hi, ints, sizeof hi, cudaMemcpyDeviceToHost, st));
  if (res->per_probe)
    RLD_CUDA(cudaMemcpyAsync(res->per_probe, per_probe, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
  RLD_CUDA(cudaStreamSynchronize(st));
  {
    int fl[2] = {hi[0], hi[5]};
    allreduce_flags(h, fl, 2);
    hi[0] = fl[0];
    hi[5] = fl[1];
  }
  if (hi[0] & RLD_FLAG_NOT_PD) fail(RLD_ERR_NOT_POSITIVE_DEFINITE, "Matrix is not positive definite (inner Cholesky)");
  if (hi[0] & RLD_FLAG_SINGULAR) fail(RLD_ERR_SINGULAR_SHIFTED_SYSTEM, "zero pivot in a shifted tridiagonal solve");
  if (hi[0] & 8) fail(RLD_ERR_INVALID_ARGUMENT, "base diagonal must be strictly positive");
  if (hi[5]) fail(RLD_ERR_CUDA, "device Gaussian stream generator overflow (flags " + std::to_string(hi[5]) + ")");
  if (hi[0] & RLD_FLAG_EIG_NOCONV) fail(RLD_ERR_CUDA, "tridiagonal eigensolver did not converge (SLQ)");
  res->clamped_eigs = slq ? hi[6] : 0;
  res->logdet_P = hs[0] + hs[1];
  res->trace_term = hs[2];
  res->value = res->logdet_P + res->trace_term;
  res->attempts = po.attempts;
  res->qr_fallback = po.householder ? 1 : 0;
  res->rank_kept = po.k > 0 ? hi[3] : 0;
  res->kv_products = products + (c->precond_kind == RLD_PRECOND_RAND_SVD || c->precond_kind == RLD_PRECOND_RAND_SVD_SCALED
                                     ? (c->precond_iters + 1) * po.attempts : 0);
  res->kernel_launches = g_launches;
  float ms[3] = {0, 0, 0};
  RLD_CUDA(cudaEventElapsedTime(&ms[0], h->ev[0], h->ev[1]));
  RLD_CUDA(cudaEventElapsedTime(&ms[1], h->ev[1], h->ev[2]));
  RLD_CUDA(cudaEventElapsedTime(&ms[2], h->ev[2], h->ev[3]));
  for (double& v : res->phase_ms) v = 0.0;
  res->phase_ms[1] = ms[0];
  res->phase_ms[4] = ms[1];
  res->phase_ms[5] = ms[2];
  res->phase_ms[7] = (double)ms[0] + ms[1] + ms[2];
  res->wall_time = res->phase_ms[7] * 1e-3;
}

template <typename F>
int guarded(rld_handle* h, F&& f) {
  try {
    if (h) set_device(h);
    f();
    if (h) h->last_error.clear();
    return RLD_OK;
  } catch (const Error& e) {
    if (h) h->last_error = e.msg;
    if (h && h->comm) h->comm->abort(e.msg);   // the other ranks fail instead of waiting on this one
    return e.code;
  } catch (const std::bad_alloc&) {
    if (h) h->last_error = "host allocation failed";
    return RLD_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    if (h) h->last_error = e.what();
    return RLD_ERR_CUDA;
  }
}

}  // namespace
}  // namespace rld

using namespace rld;

extern "C" {

int rld_abi_version(void) { return RLD_ABI_VERSION; }

int rld_nccl_unique_id(void* out) {
  if (!out) return RLD_ERR_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RLD_ERR_NCCL;
  memcpy(out, &id, sizeof id);
  return RLD_OK;
}

int rld_create(const rld_device_set* ds, rld_handle** out) {
  if (!out) return RLD_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  rld_handle* h = new (std::nothrow) rld_handle();
  if (!h) return RLD_ERR_OUT_OF_MEMORY;
  if (ds) {
    h->device = ds->device;
    h->rank = ds->rank;
    h->world = ds->world_size < 1 ? 1 : ds->world_size;
  }
  int rc = guarded(h, [&] {
    if (h->rank < 0 || h->rank >= h->world) fail(RLD_ERR_INVALID_ARGUMENT, "rank out of range");
    RLD_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    RLD_CUBLAS(cublasCreate(&h->cublas));
    RLD_CUBLAS(cublasSetStream(h->cublas, h->st));
    h->wk.kv.blas = h->cublas;
    RLD_CUSOLVER(cusolverDnCreate(&h->solver));
    RLD_CUSOLVER(cusolverDnSetStream(h->solver, h->st));
    for (auto& e : h->ev) RLD_CUDA(cudaEventCreate(&e));
    RLD_CUDA(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
    RLD_CUDA(cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming));
    RLD_CUDA(cudaEventCreateWithFlags(&h->join, cudaEventDisableTiming));
    RLD_CUDA(cudaEventCreateWithFlags(&h->efork, cudaEventDisableTiming));
    RLD_CUDA(cudaEventCreateWithFlags(&h->ejoin, cudaEventDisableTiming));
    if (h->world > 1) {
      if (ds->comm_kind == RLD_COMM_THREADS) {
        if (!ds->group) fail(RLD_ERR_INVALID_ARGUMENT, "group required for RLD_COMM_THREADS");
        h->comm = make_thread_comm(ds->group, h->rank);
        if (h->comm->world != h->world) fail(RLD_ERR_INVALID_ARGUMENT, "group size differs from world_size");
      } else if (ds->comm_kind == RLD_COMM_NCCL) {
        if (!ds->nccl_id) fail(RLD_ERR_INVALID_ARGUMENT, "nccl_id required for world_size > 1");
        h->comm = make_nccl_comm(ds->nccl_id, h->rank, h->world);
      } else {
        fail(RLD_ERR_INVALID_ARGUMENT, "unknown comm_kind");
      }
    }
  });
  if (rc != RLD_OK) {
    rld_destroy(h);
    return rc;
  }
  h->counted = true;
  rld::g_live_handles.fetch_add(1);
  *out = h;
  return RLD_OK;
}

void rld_destroy(rld_handle* h) {
  if (!h) return;
  if (h->counted) rld::g_live_handles.fetch_sub(1);
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  h->res.Kbuf.release();
  h->comm.reset();
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->st2) cudaStreamSynchronize(h->st2), cudaStreamDestroy(h->st2);
  if (h->fork) cudaEventDestroy(h->fork);
  if (h->join) cudaEventDestroy(h->join);
  if (h->efork) cudaEventDestroy(h->efork);
  if (h->ejoin) cudaEventDestroy(h->ejoin);
  if (h->solver) cusolverDnDestroy(h->solver);
  if (h->cublas) cublasDestroy(h->cublas);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

const char* rld_last_error(const rld_handle* h) { return h ? h->last_error.c_str() : "null handle"; }

void* rld_stream(rld_handle* h) { return h ? (void*)h->st : nullptr; }

int rld_prepare(rld_handle* h, const rld_problem* problem) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] { prepare(h, problem); });
}

int rld_logdet_resident(rld_handle* h, const rld_config* cfg, const rld_inputs* inputs, rld_result* result) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] { run_estimate(h, cfg, inputs, result); });
}

int rld_logdet(rld_handle* h, const rld_problem* problem, const rld_config* cfg, const rld_inputs* inputs,
               rld_result* result) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    prepare(h, problem);
    run_estimate(h, cfg, inputs, result);
  });
}

int rld_build_covariance(rld_handle* h, const rld_problem* p, void* out, int32_t out_memory) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!p || p->source != RLD_SOURCE_POINTS) fail(RLD_ERR_INVALID_ARGUMENT, "build_covariance needs points");
    if (!out) fail(RLD_ERR_INVALID_ARGUMENT, "out is NULL");
    if (h->world != 1) fail(RLD_ERR_NOT_SUPPORTED, "build_covariance is single-GPU");
    rld_problem q = *p;
    q.path = RLD_PATH_ON_THE_FLY;  // upload points only, in the caller's order
    prepare(h, &q, true);
    Resident& r = h->res;
    const size_t es = p->dtype == RLD_FP64 ? 8 : 4;
    if (out_memory == RLD_DEVICE) {
      if (p->dtype == RLD_FP64)
        build_kernel_rows<double>(r.X.as<double>(), r.n, r.kp, 0, r.n, static_cast<double*>(out), r.n, h->st);
      else
        build_kernel_rows<float>(r.X.as<double>(), r.n, r.kp, 0, r.n, static_cast<float*>(out), r.n, h->st);
    } else {
      const int64_t chunk = std::max<int64_t>(1, (int64_t)((512ull << 20) / (es * r.n)));
      DevBuf& stage = h->wk.scratch2;
      stage.reserve(es * chunk * r.n);
      for (int64_t r0 = 0; r0 < r.n; r0 += chunk) {
        const int64_t nr = std::min(chunk, r.n - r0);
        if (p->dtype == RLD_FP64)
          build_kernel_rows<double>(r.X.as<double>(), r.n, r.kp, r0, nr, stage.as<double>(), r.n, h->st);
        else
          build_kernel_rows<float>(r.X.as<double>(), r.n, r.kp, r0, nr, stage.as<float>(), r.n, h->st);
        RLD_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + es * r0 * r.n, stage.ptr, es * nr * r.n,
                                 cudaMemcpyDeviceToHost, h->st));
      }
    }
    RLD_CUDA(cudaStreamSynchronize(h->st));
  });
}

int rld_precond_build(rld_handle* h, const rld_config* cfg, const rld_inputs* inputs, rld_precond_info* info) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] { precond_build(h, cfg, inputs, info); });
}

int rld_precond_apply(rld_handle* h, int32_t op, int64_t m, const double* V, double* Y) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] { precond_apply(h, op, m, V, Y); });
}

int rld_slice_stats(rld_handle* h, int64_t* stats) {
  if (!h || !stats) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    const Resident& r = h->res;
    for (int i = 0; i < 4; ++i) stats[i] = 0;
    if (!r.ready || !r.kq_ready) return;
    const int64_t nb = ceil_div(r.rows, 128) * ceil_div(r.n, 32);
    stats[0] = nb;
    stats[3] = r.kr_ready ? 1 : 0;
    const int S = r.kslices, extra = S == 7 ? 0 : 1;   // float32 K: 3 slices against 4 of V
    if (!r.knz_ready) {   // no metadata: every block reads all 7 slices, 28 pairs
      stats[1] = (int64_t)S * nb;
      stats[2] = (int64_t)(S * (S + 1) / 2 + extra * S) * nb;
      return;
    }
    std::vector<int> nz((size_t)nb);
    RLD_CUDA(cudaMemcpyAsync(nz.data(), r.knz.ptr, sizeof(int) * nb, cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaStreamSynchronize(h->st));
    for (int v : nz) {
      stats[1] += v;
      stats[2] += (int64_t)v * (v + 1) / 2 + extra * v;
    }
  });
}

int rld_kv_apply(rld_handle* h, int64_t m, const double* V, double* Y) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!h->res.ready) fail(RLD_ERR_INVALID_ARGUMENT, "no resident problem");
    if (m < 1 || !V || !Y) fail(RLD_ERR_INVALID_ARGUMENT, "bad kv_apply arguments");
    Resident& r = h->res;
    if (r.permuted && h->world > 1) {
      // sharded: the product's rows come out in the resident order; gather them, undo the order and
      // hand back this rank's rows [row0, row0 + rows) of the caller's order
      h->wk.ptmp.reserve(sizeof(double) * m * r.n);
      h->wk.ptmp2.reserve(sizeof(double) * m * r.n);
      permute_rows(m, r.n, r.perm.as<int>(), V, r.n, h->wk.ptmp.as<double>(), r.n, false, h->st);
      h->wk.KX.reserve(sizeof(double) * m * std::max<int64_t>(r.rows, 1));
      kv(h, m, h->wk.ptmp.as<double>(), h->wk.KX.as<double>());
      gather_rows(h, h->wk.KX.as<double>(), m, h->wk.ptmp2.as<double>());
      permute_rows(m, r.n, r.perm.as<int>(), h->wk.ptmp2.as<double>(), r.n, h->wk.ptmp.as<double>(), r.n, true, h->st);
      if (r.rows > 0)
        RLD_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * r.rows, h->wk.ptmp.as<double>() + r.row0, sizeof(double) * r.n,
                                   sizeof(double) * r.rows, m, cudaMemcpyDeviceToDevice, h->st));
    } else if (r.permuted) {   // operands in the caller's order, K in the resident (Morton) order
      h->wk.ptmp.reserve(sizeof(double) * m * r.n);
      h->wk.ptmp2.reserve(sizeof(double) * m * r.n);
      permute_rows(m, r.n, r.perm.as<int>(), V, r.n, h->wk.ptmp.as<double>(), r.n, false, h->st);
      kv(h, m, h->wk.ptmp.as<double>(), h->wk.ptmp2.as<double>());
      permute_rows(m, r.n, r.perm.as<int>(), h->wk.ptmp2.as<double>(), r.n, Y, r.n, true, h->st);
    } else {
      kv(h, m, V, Y);   // stream-ordered on rld_stream(h)
    }
  });
}

int rld_dense_cholesky(rld_handle* h, int32_t n, double* G, int32_t* info) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (n < 1 || !G || !info) fail(RLD_ERR_INVALID_ARGUMENT, "bad dense_cholesky arguments");
    h->wk.ints.reserve(sizeof(int) * 8);
    int* dinfo = h->wk.ints.as<int>() + 1;
    potrf_upper(h, n, G, dinfo);
    RLD_CUDA(cudaMemcpyAsync(info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaStreamSynchronize(h->st));
  });
}

int rld_dense_eigh(rld_handle* h, int32_t n, double* A, double* w) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (n < 1 || !A || !w) fail(RLD_ERR_INVALID_ARGUMENT, "bad dense_eigh arguments");
    h->wk.ints.reserve(sizeof(int) * 8);
    syevd(h, n, A, w);
    RLD_CUDA(cudaStreamSynchronize(h->st));
  });
}

int rld_normal(rld_handle* h, const uint64_t key[2], int64_t rows, int64_t n, double* out) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!key || !out || rows < 0 || n < 0) fail(RLD_ERR_INVALID_ARGUMENT, "bad normal arguments");
    h->wk.ints.reserve(sizeof(int) * 8);
    int* f = h->wk.ints.as<int>() + 5;
    RLD_CUDA(cudaMemsetAsync(f, 0, sizeof(int), h->st));
    normal_rows(key, rows, n, 0, n, n, out, h->wk.rng_scratch, f, h->st);
    int hf = 0;
    RLD_CUDA(cudaMemcpyAsync(&hf, f, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaStreamSynchronize(h->st));
    if (hf) fail(RLD_ERR_CUDA, "device Gaussian stream generator overflow (flags " + std::to_string(hf) + ")");
  });
}

int rld_rademacher(rld_handle* h, const uint64_t key[2], int64_t rows, int64_t n, double* out) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!key || !out || rows < 0 || n < 0) fail(RLD_ERR_INVALID_ARGUMENT, "bad rademacher arguments");
    rademacher_rows(key, rows, n, 0, n, n, out, h->st);
    RLD_CUDA(cudaStreamSynchronize(h->st));
  });
}

int rld_exact_logdet(rld_handle* h, double* value) {
  if (!h) return RLD_ERR_INVALID_ARGUMENT;
  return guarded(h, [&] {
    Resident& r = h->res;
    if (!r.ready) fail(RLD_ERR_INVALID_ARGUMENT, "no resident problem");
    if (!value) fail(RLD_ERR_INVALID_ARGUMENT, "value is NULL");
    if (h->world != 1) fail(RLD_ERR_NOT_SUPPORTED, "exact_logdet is single-GPU");
    const int64_t n = r.n;
    DevBuf L;
    L.reserve(sizeof(double) * n * n);
    if (r.path == RLD_PATH_ON_THE_FLY || !r.K) {
      build_kernel_rows<double>(r.X.as<double>(), n, r.kp, 0, n, L.as<double>(), n, h->st);
    } else {
      if (r.tiled)
        untile_to_f64(static_cast<const float*>(r.K), n, n, L.as<double>(), n, h->st);
      else
        convert_rows_2d(r.K, r.dtype, r.ldk, L.as<double>(), n, n, h->st);
    }
    cusolverDnParams_t params;
    RLD_CUSOLVER(cusolverDnCreateParams(&params));
    size_t dws = 0, hws = 0;
    RLD_CUSOLVER(cusolverDnXpotrf_bufferSize(h->solver, params, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, L.ptr, n,
                                             CUDA_R_64F, &dws, &hws));
    DevBuf dwork;
    dwork.reserve(std::max<size_t>(dws, 8));
    std::vector<char> hwork(std::max<size_t>(hws, 8));
    h->wk.ints.reserve(sizeof(int) * 8);
    int* info = h->wk.ints.as<int>();
    RLD_CUSOLVER(cusolverDnXpotrf(h->solver, params, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, L.ptr, n, CUDA_R_64F,
                                  dwork.ptr, dws, hwork.data(), hws, info + 1));
    cusolverDnDestroyParams(params);
    RLD_CUDA(cudaMemsetAsync(info, 0, sizeof(int), h->st));
    // 2 sum log diag L with the diagonal stride n + 1
    h->wk.scal.reserve(sizeof(double) * 8);
    strided_sum_log(n, L.as<double>(), n + 1, h->wk.scal.as<double>(), h->wk.scratch, h->st);
    double sv = 0;
    int hinfo = 0;
    RLD_CUDA(cudaMemcpyAsync(&sv, h->wk.scal.ptr, sizeof sv, cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaMemcpyAsync(&hinfo, info + 1, sizeof hinfo, cudaMemcpyDeviceToHost, h->st));
    RLD_CUDA(cudaStreamSynchronize(h->st));
    if (hinfo != 0) fail(RLD_ERR_NOT_POSITIVE_DEFINITE, "Matrix is not positive definite");
    *value = 2.0 * sv;
  });
}

}  // extern "C"
