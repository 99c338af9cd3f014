// Work schedule and step iterators shared by the tensor-core K x block kernels
// (kv_tc.cu: tf32 stored / on the fly; kv_otf.cu: fp16 on the fly), plus packed
// FP32x2 and MUFU helpers and the host-side TMA / device-attribute helpers.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <algorithm>

namespace rld {

constexpr int GROUP = 4;            // k-steps accumulated in TMEM before the register flush

// Work schedule of one CTA (G CTAs per column pass).  Phase 1: R = tiles / G full
// rounds -- CTA c takes tile c + r G over all k-steps, so every CTA sweeps the B
// operand (V) in the same k order at about the same time and L2 serves the reuse
// (with per-CTA stream-K ranges the CTAs sat at unrelated k offsets and re-read B
// from HBM once per tile: ~8.8 TB per config-5 product).  Phase 2: the remaining
// tiles' (tile, k-step) space is cut into G equal contiguous ranges ("stream-K"),
// whose per-CTA partial tiles kv_tc_reduce adds in fixed order.
struct Sched {
  int ks, G, R;          // k-steps per tile, CTAs per pass, full rounds
  int group = GROUP;     // k-steps per TMEM accumulation group (register flush after each)
  int64_t tail_total;    // (tiles - R G) * ks
  __host__ __device__ int64_t tail_beg(int64_t c) const { return c * tail_total / G; }
  __host__ __device__ int64_t tail_end(int64_t c) const { return (c + 1) * tail_total / G; }
};

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fast_sqrt(float x) {   // MUFU; sqrt(0) = 0
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed FP32x2 helpers (sm_100 FADD2 / FMUL2 / FFMA2), lanes = (lo 32 bits, hi 32 bits)
__device__ __forceinline__ uint64_t pk(float a, float b) {
  return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ float pk_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float pk_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__host__ __device__ __forceinline__ int64_t cta_of_step(int64_t x, int64_t total, int64_t G) {
  // the CTA whose range [c*total/G, (c+1)*total/G) contains step x
  return ((x + 1) * G - 1) / total;
}

// Walks a CTA's steps with running 32-bit counters (no divisions in the loops:
// the pipeline warps run this once per k-step, inside their critical loops, and
// each role pays only for the counters it uses: GRP = group boundaries (MMA),
// BR = a second ring (the converters walk the A-source ring in (s, ph) and the
// B / TMEM-buffer ring in (sb, phb))).
template <bool GRP, bool BR>
struct StepIter {
  int v, vend;           // step index (== pipeline slot j) and end: [0, R ks) phase 1, then the tail range
  int ks, kstep, tile, s, S, G, R, round, group;
  int tail_next, tail_k0;   // where the tail range starts (tile, k-step)
  uint32_t ph;
  int gpos = 0;          // GRP: position in the accumulation group
  int sb = 0, SB = 1;    // BR: second ring
  uint32_t phb = 0;
  __device__ __forceinline__ StepIter(const Sched& sc, int64_t cta, int S_, int SB_ = 1)
      : v(0), ks(sc.ks), kstep(0), s(0), S(S_), G(sc.G), R(sc.R), round(0), group(sc.group), ph(0), SB(SB_) {
    const int64_t tb = sc.tail_beg(cta), te = sc.tail_end(cta);
    vend = R * ks + (int)(te - tb);
    tail_next = R * G + (int)(tb / ks);
    tail_k0 = (int)(tb - (int64_t)(tb / ks) * ks);
    if (R > 0) {
      tile = (int)cta;
    } else {
      tile = tail_next;
      kstep = tail_k0;
    }
  }
  __device__ __forceinline__ bool valid() const { return v < vend; }
  __device__ __forceinline__ bool in_tail() const { return round >= R; }
  __device__ __forceinline__ bool group_start() const { return gpos == 0; }
  __device__ __forceinline__ bool seg_end() const { return v + 1 == vend || kstep + 1 == ks; }
  __device__ __forceinline__ bool group_end() const { return seg_end() || gpos + 1 == group; }
  __device__ __forceinline__ void next() {
    if (GRP) gpos = group_end() ? 0 : gpos + 1;
    ++v;
    if (++kstep == ks) {
      kstep = 0;
      if (round < R) {
        if (++round < R) {
          tile += G;
        } else {   // phase 1 done: continue in the tail range
          tile = tail_next;
          kstep = tail_k0;
        }
      } else {
        ++tile;
      }
    }
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
    if (BR && ++sb == SB) {
      sb = 0;
      phb ^= 1;
    }
  }
};

// Segment (tile, first step, steps) iteration for the drain warps: one call per
// segment instead of one StepIter advance per k-step.
struct SegIter {
  int64_t cta;
  const Sched* sc;
  int r;                 // phase-1 round, then R for the tail
  int64_t x, xe;         // tail-space position and end
  __device__ __forceinline__ SegIter(const Sched& s, int64_t c) : cta(c), sc(&s), r(0) {
    x = s.tail_beg(c);
    xe = s.tail_end(c);
  }
  // next segment: tile, its length in k-steps and its partial-sum slot; false when done
  __device__ __forceinline__ bool next(int& tile, int& len, int& seg) {
    int k0;
    return next(tile, len, seg, k0);
  }
  // ... and the segment's first k-step
  __device__ __forceinline__ bool next(int& tile, int& len, int& seg, int& k0) {
    if (r < sc->R) {
      tile = (int)cta + r * sc->G;
      len = sc->ks;
      seg = 0;
      k0 = 0;
      ++r;
      return true;
    }
    if (x >= xe) return false;
    const int64_t u = x / sc->ks;
    const int64_t x0 = u * sc->ks;
    tile = sc->R * sc->G + (int)u;
    len = (int)(std::min<int64_t>(xe, x0 + sc->ks) - x);
    seg = (int)(cta - cta_of_step(x0, sc->tail_total, sc->G));
    k0 = (int)(x - x0);
    x += len;
    return true;
  }
};


typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn();
int sm_count();
int max_smem_optin();

}  // namespace rld
