// numpy-exact Gaussian rows on the device.
//
// The reference draws its sketch Omega and Gaussian probes with
// Generator(Philox(SeedSequence(seed, spawn_key=path))).standard_normal(shape)
// (src/linalg.py:81-82, src/precond.py:183, src/probes.py:33-34).  numpy's
// standard_normal is a 256-layer ziggurat: each attempt starts at one 64-bit
// Philox word; the fast path (99.3 %) accepts it outright, the wedge path reads
// one more word and may reject, the tail (layer 0) loops on pairs of words.  The
// stream position of draw k is therefore data-dependent.  Parallel form:
//
//   pass 1 (zig_chunk_kernel): per chunk of C words, every word's attempt length
//     L(q) and accept bit are computed (Philox is counter-addressable).  Only
//     "slow" words (L > 1, ~0.7 %) can break the one-word-per-draw pattern, so a
//     single thread walks the chunk's slow words in order, once per possible
//     entry offset e < EMAX (how far the previous chunk's last attempt reached
//     into this one), giving exit offset and accepted count per e;
//   pass 2 (zig_link_kernel): one CTA chains the chunks -- entry offset and output
//     base of every chunk (fixed order, deterministic);
//   pass 3 (zig_emit_kernel): per chunk, the attempt starts are marked, a block
//     prefix sum ranks the accepted ones, and each draw is written in place.
//
// exp / log1p in the slow paths are CUDA's; the GPU test compares against numpy
// bit-for-bit and reports any last-bit differences in tail draws.
#include "rld_device.cuh"
#include "rld_internal.cuh"
#include "rld_kernels.cuh"
#include "ziggurat_tables.h"

namespace rld {

namespace {

constexpr int ZC = 4096;        // words per chunk
constexpr int ZT = 256;         // threads per chunk CTA (16 words each)
constexpr int ZM = 64;          // margin words past the chunk (attempts that overhang)
constexpr int EMAX = 16;        // entry offsets tracked per chunk
constexpr int MAXSLOW = 512;    // slow words per chunk (expected ~30)

__device__ __forceinline__ double u01(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

// attempt starting at word q: returns length (words consumed) and whether it accepts;
// `words` holds the chunk's words from offset `base` (q - base < ZC + ZM guaranteed by caller)
struct Attempt {
  int len;
  bool acc;
  double value;
};

// Ziggurat tables in shared memory: the layer index is random per lane, and __constant__ reads
// with 32 different addresses serialise (the emit kernel spent 40 % of its stalls there).
struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};

__device__ __forceinline__ void load_zig_tables(ZigTables& z) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    z.ki[i] = rld_zig_ki[i];
    z.wi[i] = rld_zig_wi[i];
    z.fi[i] = rld_zig_fi[i];
  }
}

__device__ Attempt attempt_at(const uint64_t* words, int qi, int limit, bool want_value, const ZigTables& z) {
  Attempt a{1, true, 0.0};
  uint64_t r = words[qi];
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const int sign = (int)(r & 1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = (double)rabs * z.wi[idx];
  if (sign) x = -x;
  if (rabs < z.ki[idx]) {
    a.value = x;
    return a;
  }
  if (idx == 0) {
    int k = qi + 1;
    for (;;) {
      if (k + 1 >= limit) {  // tail loop ran past the margin (probability ~1e-30)
        a.len = -1;
        return a;
      }
      const double xx = -RLD_ZIG_INV_R * log1p(-u01(words[k]));
      const double yy = -log1p(-u01(words[k + 1]));
      k += 2;
      if (yy + yy > xx * xx) {
        a.len = k - qi;
        a.value = ((rabs >> 8) & 1) ? -(RLD_ZIG_R + xx) : (RLD_ZIG_R + xx);
        return a;
      }
    }
  }
  if (qi + 1 >= limit) {
    a.len = -1;
    return a;
  }
  a.len = 2;
  a.acc = ((z.fi[idx - 1] - z.fi[idx]) * u01(words[qi + 1]) + z.fi[idx]) < exp(-0.5 * x * x);
  a.value = x;
  (void)want_value;
  return a;
}

// Fill sm_words[0 .. ZC + ZM) with stream words chunk*ZC + i, and build the ordered
// list of slow words (attempt length != 1 or rejecting) with their lengths / accept bits.
__device__ void load_chunk(int64_t chunk, uint64_t k0, uint64_t k1, uint64_t* sm_words, int* sm_slow_pos,
                           short* sm_slow_len, unsigned char* sm_slow_acc, int* sm_nslow, int* sm_cnt, int* flags,
                           const ZigTables& z) {
  const int t = threadIdx.x;
  const uint64_t q0 = (uint64_t)chunk * ZC;
  // 16 words per thread = 4 Philox blocks; margin words by the first ZM/4 threads
  {
    const uint64_t qb = q0 + (uint64_t)t * 16;
#pragma unroll
    for (int b4 = 0; b4 < 4; ++b4) {
      const uint64_t blk = ((qb + 4 * b4) >> 2) + 1;
      U64x4 c;
      c.v[0] = blk;
      c.v[1] = 0;
      c.v[2] = 0;
      c.v[3] = 0;
      const U64x4 o = philox4x64_10(c, k0, k1);
#pragma unroll
      for (int l = 0; l < 4; ++l) sm_words[t * 16 + 4 * b4 + l] = o.v[l];
    }
    if (t < ZM / 4) {
      const uint64_t blk = ((q0 + ZC + 4 * t) >> 2) + 1;
      U64x4 c;
      c.v[0] = blk;
      c.v[1] = 0;
      c.v[2] = 0;
      c.v[3] = 0;
      const U64x4 o = philox4x64_10(c, k0, k1);
#pragma unroll
      for (int l = 0; l < 4; ++l) sm_words[ZC + 4 * t + l] = o.v[l];
    }
  }
  __syncthreads();
  // slow words of this thread's 16, compacted in order
  int pos[16];
  short len[16];
  unsigned char acc[16];
  int ns = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int qi = t * 16 + i;
    const uint64_t r = sm_words[qi];
    const int idx = (int)(r & 0xff);
    const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
    if (rabs >= z.ki[idx]) {
      const Attempt a = attempt_at(sm_words, qi, ZC + ZM, false, z);
      if (a.len < 0) atomicOr(flags, 1);
      pos[ns] = qi;
      len[ns] = (short)(a.len < 0 ? 1 : a.len);
      acc[ns] = a.acc ? 1 : 0;
      ++ns;
    }
  }
  // exclusive scan of ns over the block (ordered by thread = ordered by position)
  sm_cnt[t] = ns;
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int i = 0; i < ZT; ++i) {
      const int c = sm_cnt[i];
      sm_cnt[i] = run;
      run += c;
    }
    *sm_nslow = run;
  }
  __syncthreads();
  const int off = sm_cnt[t];
  for (int i = 0; i < ns; ++i) {
    if (off + i < MAXSLOW) {
      sm_slow_pos[off + i] = pos[i];
      sm_slow_len[off + i] = len[i];
      sm_slow_acc[off + i] = acc[i];
    } else {
      atomicOr(flags, 2);
    }
  }
  __syncthreads();
}

struct ChunkSmem {
  ZigTables zig;
  uint64_t words[ZC + ZM];
  int slow_pos[MAXSLOW];
  short slow_len[MAXSLOW];
  unsigned char slow_acc[MAXSLOW];
  int cnt[ZT];
  int nslow;
  unsigned int start_mask[ZC / 32];
};

// pass 1: exit offset and accepted count of every chunk for entry offsets 0..EMAX-1
__global__ void __launch_bounds__(ZT) zig_chunk_kernel(uint64_t k0, uint64_t k1, int* __restrict__ exits,
                                                       int* __restrict__ naccs, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  ChunkSmem& sm = *reinterpret_cast<ChunkSmem*>(zsm_raw);
  const int64_t chunk = blockIdx.x;
  load_zig_tables(sm.zig);
  load_chunk(chunk, k0, k1, sm.words, sm.slow_pos, sm.slow_len, sm.slow_acc, &sm.nslow, sm.cnt, flags, sm.zig);
  const int ns = min(sm.nslow, MAXSLOW);
  if (threadIdx.x < EMAX) {
    const int e = threadIdx.x;
    int cursor = e, covered = 0, rejected = 0;
    for (int i = 0; i < ns; ++i) {
      const int pq = sm.slow_pos[i];
      if (pq < cursor) continue;  // inside an earlier attempt
      const int L = sm.slow_len[i];
      cursor = pq + L;
      covered += min(L - 1, ZC - 1 - pq);
      rejected += sm.slow_acc[i] ? 0 : 1;
    }
    const int starts = (ZC - e) - covered;
    exits[chunk * EMAX + e] = cursor > ZC ? cursor - ZC : 0;
    naccs[chunk * EMAX + e] = starts - rejected;
  }
}

// pass 2: entry offset and first output index of every chunk (one CTA, fixed order)
constexpr int ZL = 128;   // threads of the link kernel

__global__ void __launch_bounds__(ZL) zig_link_kernel(int64_t nchunks, int64_t count, const int* __restrict__ exits,
                                                      const int* __restrict__ naccs, int* __restrict__ entry,
                                                      int64_t* __restrict__ base, int* __restrict__ flags) {
  __shared__ int s_exit[ZL][EMAX];
  __shared__ long long s_cnt[ZL][EMAX];
  __shared__ int s_entry[ZL];
  __shared__ long long s_base[ZL];
  const int t = threadIdx.x;
  const int64_t per = ceil_div(nchunks, ZL);
  const int64_t c0 = min64((int64_t)t * per, nchunks), c1 = min64(c0 + per, nchunks);
  // composed map of this run: entry e -> (exit, accepted count)
  for (int e = 0; e < EMAX; ++e) {
    int cur = e;
    long long cnt = 0;
    bool bad = false;
    for (int64_t c = c0; c < c1; ++c) {
      if (cur >= EMAX) {
        bad = true;
        cur = 0;
      }
      cnt += naccs[c * EMAX + cur];
      cur = exits[c * EMAX + cur];
    }
    if (bad) cur = EMAX;  // marks an overflow; only fatal if this entry is the one used
    s_exit[t][e] = cur;
    s_cnt[t][e] = cnt;
  }
  __syncthreads();
  if (t == 0) {
    int cur = 0;
    long long b = 0;
    for (int i = 0; i < ZL; ++i) {
      s_entry[i] = cur;
      s_base[i] = b;
      if (cur >= EMAX) {
        atomicOr(flags, 4);
        cur = 0;
      }
      b += s_cnt[i][cur];
      cur = s_exit[i][cur];
    }
    if (b < count) atomicOr(flags, 8);   // not enough words for `count` draws
  }
  __syncthreads();
  int cur = s_entry[t];
  long long b = s_base[t];
  for (int64_t c = c0; c < c1; ++c) {
    if (cur >= EMAX) {
      atomicOr(flags, 4);
      cur = 0;
    }
    entry[c] = cur;
    base[c] = b;
    b += naccs[c * EMAX + cur];
    cur = exits[c * EMAX + cur];
  }
}

// pass 3: write draw `base + rank` for every accepted attempt start of the chunk
__global__ void __launch_bounds__(ZT) zig_emit_kernel(uint64_t k0, uint64_t k1, const int* __restrict__ entry,
                                                      const int64_t* __restrict__ base, int64_t count, int64_t ncols,
                                                      int64_t col0, int64_t ldo, int64_t nout_cols,
                                                      double* __restrict__ out, int* __restrict__ flags,
                                                      int64_t* __restrict__ end_word) {
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  ChunkSmem& sm = *reinterpret_cast<ChunkSmem*>(zsm_raw);
  const int64_t chunk = blockIdx.x;
  const int64_t b0 = base[chunk];
  if (b0 >= count) return;
  load_zig_tables(sm.zig);
  load_chunk(chunk, k0, k1, sm.words, sm.slow_pos, sm.slow_len, sm.slow_acc, &sm.nslow, sm.cnt, flags, sm.zig);
  const int t = threadIdx.x;
  const int e = entry[chunk];
  // start mask: every word >= e, minus words covered by slow attempts
  for (int i = t; i < ZC / 32; i += ZT) {
    const int lo = i * 32;
    unsigned int m = 0xffffffffu;
    if (e > lo) m = (e >= lo + 32) ? 0u : (0xffffffffu << (e - lo));
    sm.start_mask[i] = m;
  }
  __syncthreads();
  if (t == 0) {
    const int ns = min(sm.nslow, MAXSLOW);
    int cursor = e;
    for (int i = 0; i < ns; ++i) {
      const int pq = sm.slow_pos[i];
      if (pq < cursor) continue;
      const int L = sm.slow_len[i];
      cursor = pq + L;
      for (int w = pq + 1; w < min(pq + L, ZC); ++w) sm.start_mask[w >> 5] &= ~(1u << (w & 31));
      if (!sm.slow_acc[i]) sm.start_mask[pq >> 5] &= ~(1u << (pq & 31));  // rejected: no draw
    }
  }
  __syncthreads();
  // this thread's 16 words: accepted starts, block prefix sum
  const unsigned int mword = sm.start_mask[(t * 16) >> 5];
  const unsigned int mine = (mword >> ((t * 16) & 31)) & 0xffffu;
  sm.cnt[t] = __popc(mine);
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int i = 0; i < ZT; ++i) {
      const int c = sm.cnt[i];
      sm.cnt[i] = run;
      run += c;
    }
  }
  __syncthreads();
  int64_t k = b0 + sm.cnt[t];
  for (int i = 0; i < 16; ++i) {
    if (!((mine >> i) & 1)) continue;
    if (k >= count) break;
    const Attempt a = attempt_at(sm.words, t * 16 + i, ZC + ZM, true, sm.zig);
    const int64_t r = k / ncols, jj = k % ncols;
    if (jj >= col0 && jj < col0 + nout_cols) out[r * ldo + (jj - col0)] = a.value;
    if (end_word && k == count - 1) *end_word = chunk * ZC + t * 16 + i + a.len;   // stream word after the last draw
    ++k;
  }
}

}  // namespace

// rows x n standard normals of numpy stream `key`, columns [col0, col0 + ncols_out) of
// each row written to out (row stride ld).  Scratch is grown as needed.
void normal_rows(const uint64_t key[2], int64_t rows, int64_t n, int64_t col0, int64_t ncols_out, int64_t ld,
                 double* out, DevBuf& scratch, int* dflags, cudaStream_t st, int64_t* end_word) {
  const int64_t count = rows * n;
  if (count <= 0) return;
  // words: ~1.007 per draw on average; generous margin, checked below
  const int64_t nchunks = ceil_div(count + count / 32 + 4096, ZC);
  const size_t need = (size_t)nchunks * EMAX * sizeof(int) * 2 + (size_t)nchunks * (sizeof(int) + sizeof(int64_t));
  scratch.reserve(need);
  int* exits = scratch.as<int>();
  int* naccs = exits + nchunks * EMAX;
  int* entry = naccs + nchunks * EMAX;
  int64_t* base = reinterpret_cast<int64_t*>(entry + nchunks + (nchunks & 1));
  const size_t smem = sizeof(ChunkSmem);
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [&] {
    RLD_CUDA(cudaFuncSetAttribute(zig_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RLD_CUDA(cudaFuncSetAttribute(zig_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  zig_chunk_kernel<<<(unsigned)nchunks, ZT, smem, st>>>(key[0], key[1], exits, naccs, dflags);
  RLD_LAUNCH_CHECK();
  zig_link_kernel<<<1, ZL, 0, st>>>(nchunks, count, exits, naccs, entry, base, dflags);
  RLD_LAUNCH_CHECK();
  zig_emit_kernel<<<(unsigned)nchunks, ZT, smem, st>>>(key[0], key[1], entry, base, count, n, col0, ld, ncols_out,
                                                        out, dflags, end_word);
  RLD_LAUNCH_CHECK();
}

}  // namespace rld
