// K x block products on the CUDA cores (float64 DFMA / float32 FFMA).
//
// Y[c, i] = sum_j K[row0 + i, j] * V[c, j]: the batched form of the
// reference's per-probe `M @ x` (src/estimators.py:72) and of the sketch
// product `Y @ M` (src/precond.py:186, 189).  K comes either from a stored
// row block (HBM stream) or is generated tile by tile from the points held in
// shared memory (on-the-fly path).
//
// Classic register-tiled NT GEMM: CTA tile BM x BN over (rows of K) x (vectors),
// BK-deep k-steps double-buffered in shared memory, TM x TN outputs per thread.
// The k range is split across CTAs so that small-m products still fill the
// 148 SMs; partial sums land in a [split][m][rows] float64 buffer that a second
// kernel reduces in fixed split order (deterministic, no atomics).
#include <cstdlib>

#include "rld_internal.cuh"
#include "rld_device.cuh"

namespace rld {

namespace {

template <typename T, int BM, int BN, int BK, int TM, int TN, bool OTF>
struct KvTile {
  static constexpr int THREADS = (BM / TM) * (BN / TN);
};

template <typename TK, typename T, int BM, int BN, int BK, int TM, int TN, bool OTF>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
kv_simt_kernel(const TK* __restrict__ K, int64_t ldk, const double* __restrict__ X, KernelParams kp,
               int64_t row0, int64_t rows, int64_t n, const T* __restrict__ V, int64_t ldv, int64_t m,
               int64_t kchunk, double* __restrict__ out, int64_t ldo, int64_t split_stride) {
  constexpr int THREADS = (BM / TM) * (BN / TN);
  constexpr int PA = BM + 4, PB = BN + 4;
  __shared__ T As[2][BK][PA];
  __shared__ T Bs[2][BK][PB];
  __shared__ double Xr[OTF ? BM * RLD_MAX_DIM : 1];

  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN);   // vector (column) group
  const int ty = tid / (BN / TN);   // row group
  const int64_t i0 = (int64_t)blockIdx.y * BM;
  const int64_t c0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min64(n, kbeg + kchunk);

  // on-the-fly: stage this CTA's row points once
  float a2f = 0.f, gscale = 0.f, s5f = 0.f;
  if constexpr (OTF) {
    const int d = kp.d;
    for (int e = tid; e < BM * d; e += THREADS) {
      int64_t r = i0 + e / d;
      Xr[e] = (r < rows) ? X[(row0 + r) * d + (e % d)] : 0.0;
    }
    a2f = (float)kp.a2;
    gscale = (float)(kp.inv_2l2 * 1.4426950408889634);
    s5f = (float)kp.s5_over_l;
    __syncthreads();
  }

  constexpr int A_PER = (BM * BK) / THREADS;
  constexpr int B_PER = (BN * BK) / THREADS;
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "tile/threads");
  T ra[A_PER], rb[B_PER];

  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = tid + e * THREADS;
      const int r = idx / BK, kk = idx % BK;
      const int64_t gi = i0 + r, gj = k0 + kk;
      T v = T(0);
      if (gi < rows && gj < kend) {
        if constexpr (OTF) {
          const int d = kp.d;
          const int64_t gr = row0 + gi;
          if (gr == gj) {
            v = (T)kp.diag;
          } else {
            if constexpr (sizeof(T) == 8) {
              double r2 = 0.0;
              for (int q = 0; q < d; ++q) {
                double df = Xr[r * d + q] - X[gj * d + q];
                r2 = fma(df, df, r2);
              }
              v = (T)kernel_value_f64(kp, r2);
            } else {
              float r2 = 0.f;
              for (int q = 0; q < d; ++q) {
                float df = (float)Xr[r * d + q] - (float)X[gj * d + q];
                r2 = fmaf(df, df, r2);
              }
              v = (T)kernel_value_f32(kp.family, a2f, gscale, s5f, r2);
            }
          }
        } else {
          v = (T)K[gi * ldk + gj];
        }
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = tid + e * THREADS;
      const int c = idx / BK, kk = idx % BK;
      const int64_t gc = c0 + c, gj = k0 + kk;
      rb[e] = (gc < m && gj < kend) ? V[gc * ldv + gj] : T(0);
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = tid + e * THREADS;
      As[buf][idx % BK][idx / BK] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = tid + e * THREADS;
      Bs[buf][idx % BK][idx / BK] = rb[e];
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = T(0);

  if (kbeg < kend) {
    load_tile(kbeg);
    store_tile(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
      const bool more = k0 + BK < kend;
      if (more) load_tile(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T av[TM], bv[TN];
#pragma unroll
        for (int a = 0; a < TM; ++a) av[a] = As[buf][kk][ty * TM + a];
#pragma unroll
        for (int b = 0; b < TN; ++b) bv[b] = Bs[buf][kk][tx * TN + b];
#pragma unroll
        for (int a = 0; a < TM; ++a)
#pragma unroll
          for (int b = 0; b < TN; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
      if (more) {
        store_tile(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }

  double* o = out + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int b = 0; b < TN; ++b) {
    const int64_t gc = c0 + tx * TN + b;
    if (gc >= m) continue;
#pragma unroll
    for (int a = 0; a < TM; ++a) {
      const int64_t gi = i0 + ty * TM + a;
      if (gi < rows) o[gc * ldo + gi] = (double)acc[a][b];
    }
  }
}

__global__ void split_reduce_kernel(const double* __restrict__ part, int splits, int64_t split_stride,
                                    int64_t m, int64_t rows, double* __restrict__ Y, int64_t ldy) {
  const int64_t total = m * rows;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, i = e % rows;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * split_stride + c * rows + i];
    Y[c * ldy + i] = s;
  }
}

__global__ void cast_rows_kernel(const double* __restrict__ src, int64_t lds, float* __restrict__ dst,
                                 int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n, j = e % n;
    dst[e] = (float)src[c * lds + j];
  }
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    RLD_CUDA(cudaGetDevice(&dev));
    RLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

template <typename TK, typename T, int BM, int BN, int BK, int TM, int TN, bool OTF>
void launch_kv(const KvOperand& op, int64_t m, const T* V, int64_t ldv, double* Y, int64_t ldy,
               KvWorkspace& ws, cudaStream_t st, int* launches) {
  constexpr int THREADS = (BM / TM) * (BN / TN);
  const int64_t rows = op.rows, n = op.n;
  const int64_t tiles = ceil_div(rows, BM) * ceil_div(m, BN);
  const int64_t want = (int64_t)num_sms() * 4;
  int64_t splits = std::max<int64_t>(1, ceil_div(want, tiles));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, n / (BK * 16)));
  int64_t kchunk = ceil_div(ceil_div(n, splits), BK) * BK;
  splits = ceil_div(n, kchunk);
  dim3 grid((unsigned)ceil_div(m, BN), (unsigned)ceil_div(rows, BM), (unsigned)splits);
  const TK* K = static_cast<const TK*>(op.K);
  if (splits == 1) {
    kv_simt_kernel<TK, T, BM, BN, BK, TM, TN, OTF><<<grid, THREADS, 0, st>>>(
        K, op.ldk, op.X, op.kp, op.row0, rows, n, V, ldv, m, kchunk, Y, ldy, 0);
    RLD_LAUNCH_CHECK();
    if (launches) *launches += 1;
    return;
  }
  const int64_t split_stride = m * rows;
  ws.partial.reserve(sizeof(double) * split_stride * splits);
  kv_simt_kernel<TK, T, BM, BN, BK, TM, TN, OTF><<<grid, THREADS, 0, st>>>(
      K, op.ldk, op.X, op.kp, op.row0, rows, n, V, ldv, m, kchunk, ws.partial.as<double>(), rows,
      split_stride);
  RLD_LAUNCH_CHECK();
  const int64_t total = m * rows;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8);
  split_reduce_kernel<<<blocks, 256, 0, st>>>(ws.partial.as<double>(), (int)splits, split_stride, m, rows, Y,
                                               ldy);
  RLD_LAUNCH_CHECK();
  if (launches) *launches += 2;
}

}  // namespace

void kv_product(const KvOperand& op, int64_t m, const double* V, int64_t ldv, double* Y, int64_t ldy,
                KvWorkspace& ws, cudaStream_t st, int* launches, bool presplit) {
  if (m <= 0 || op.rows <= 0) return;
  const bool otf = (op.K == nullptr);
  if (op.dtype == RLD_FP64) {
    // Stored float64 K: Y = V K^T on the FP64 tensor cores (kv_dmma.cu: TMA-fed DMMA, fixed-order
    // split-k).  Operand rows must start 16-byte aligned: V is re-pitched into the workspace when
    // it is not; a K aliased from a caller's odd-pitched matrix takes this file's DFMA kernel.
    static const bool simt = getenv("RLD_FP64_SIMT") && getenv("RLD_FP64_SIMT")[0] == '1';
    const double* K = static_cast<const double*>(op.K);
    if (!simt && op.kr && m >= CRT_MIN_M) {   // wide: modular int8 GEMMs + CRT (kv_crt.cu)
      kv_product_crt(op.kr, op.ksigma, op.rows, op.n, V, ldv, m, Y, ldy, ws, st);
      return;
    }
    if (!simt && op.kq) {   // exact int8 slices of K on the INT8 tensor cores (kv_ozaki.cu)
      kv_product_ozaki(op.kq, op.ksigma, op.rows, op.n, V, ldv, m, Y, ldy, ws, st, op.oz_diags, op.knz, op.kslices);
      return;
    }
    if (!otf && !simt && gemm_nt_f64_ok(K, op.ldk, K, op.ldk)) {
      const double* Vp = V;
      int64_t ldvp = ldv;
      if (!gemm_nt_f64_ok(V, ldv, V, ldv)) {
        ldvp = (op.n + 1) / 2 * 2;
        ws.vcast.reserve(sizeof(double) * m * ldvp);
        RLD_CUDA(cudaMemcpy2DAsync(ws.vcast.ptr, sizeof(double) * ldvp, V, sizeof(double) * ldv,
                                   sizeof(double) * op.n, m, cudaMemcpyDeviceToDevice, st));
        Vp = ws.vcast.as<double>();
      }
      gemm_nt_f64(K, op.ldk, op.rows, Vp, ldvp, m, op.n, Y, ldy, 0.0, ws.partial, st);
      return;
    }
    if (otf)
      launch_kv<double, double, 64, 32, 16, 4, 4, true>(op, m, V, ldv, Y, ldy, ws, st, launches);
    else
      launch_kv<double, double, 64, 32, 16, 4, 4, false>(op, m, V, ldv, Y, ldy, ws, st, launches);
    return;
  }
  if (op.kq) {   // float32 K held as 3 int8 slices (Morton-ordered points, kv_ozaki.cu)
    kv_product_ozaki(op.kq, op.ksigma, op.rows, op.n, V, ldv, m, Y, ldy, ws, st, 0, op.knz, op.kslices, op.koff);
    return;
  }
  if (kv_tc_supported(op) && (op.tiled || !getenv("RLD_NO_TC"))) {
    kv_product_tc(op, op.tc_mode, m, V, ldv, Y, ldy, ws, st, presplit);
    return;
  }
  if (op.tiled) fail(RLD_ERR_NOT_SUPPORTED, "tiled fp32 K needs the tensor-core product");
  // float32 arithmetic: cast the float64 operand rows once
  ws.vcast.reserve(sizeof(float) * m * op.n);
  float* Vf = ws.vcast.as<float>();
  {
    const int64_t total = m * op.n;
    int blocks = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8);
    cast_rows_kernel<<<blocks, 256, 0, st>>>(V, ldv, Vf, m, op.n);
    RLD_LAUNCH_CHECK();
    if (launches) *launches += 1;
  }
  if (otf)
    launch_kv<float, float, 64, 32, 32, 4, 4, true>(op, m, Vf, op.n, Y, ldy, ws, st, launches);
  else
    launch_kv<float, float, 64, 32, 32, 4, 4, false>(op, m, Vf, op.n, Y, ldy, ws, st, launches);
}

}  // namespace rld
