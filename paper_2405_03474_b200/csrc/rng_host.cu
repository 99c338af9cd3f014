// Host port of numpy's Generator draws that follow the device-generated Gaussian rows
// in the same stream: the chi radii of normal-orthogonal probes (src/probes.py:15-22,
// Rng.chi = sqrt(Generator.chisquare(df)), src/linalg.py:87-88).
//
// numpy (2.3) draws chisquare(df) as 2 * standard_gamma(df / 2) with the
// Marsaglia-Tsang method for shape >= 1 (one ziggurat normal and one next_double per
// attempt); the ziggurat is the one the device port (rng.cu) reproduces, over the same
// Philox4x64-10 stream.  The device reports how many 64-bit words its Gaussian rows
// consumed, so the host continues the stream at exactly that word.
#include <cmath>
#include <cstdint>

#define RLD_ZIG_QUAL static const
#include "ziggurat_tables.h"
#include "rld_internal.cuh"

namespace rld {

namespace {

struct HostPhilox {   // numpy's Philox4x64-10 bit generator, positioned at a word index
  uint64_t k0, k1;
  uint64_t word;      // index of the next 64-bit word
  uint64_t buf[4];
  uint64_t buf_blk = ~0ull;

  static void mulhilo(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
    const unsigned __int128 p = (unsigned __int128)a * b;
    lo = (uint64_t)p;
    hi = (uint64_t)(p >> 64);
  }
  void block(uint64_t blk) {   // counter value blk (numpy pre-increments: word q is in block q/4 + 1)
    uint64_t c0 = blk, c1 = 0, c2 = 0, c3 = 0, a0 = k0, a1 = k1;
    for (int r = 0; r < 10; ++r) {
      if (r) {
        a0 += 0x9E3779B97F4A7C15ULL;
        a1 += 0xBB67AE8584CAA73BULL;
      }
      uint64_t lo0, hi0, lo1, hi1;
      mulhilo(0xD2E7470EE14C6C93ULL, c0, lo0, hi0);
      mulhilo(0xCA5A826395121157ULL, c2, lo1, hi1);
      const uint64_t n0 = hi1 ^ c1 ^ a0, n1 = lo1, n2 = hi0 ^ c3 ^ a1, n3 = lo0;
      c0 = n0;
      c1 = n1;
      c2 = n2;
      c3 = n3;
    }
    buf[0] = c0;
    buf[1] = c1;
    buf[2] = c2;
    buf[3] = c3;
    buf_blk = blk;
  }
  uint64_t next() {
    const uint64_t blk = (word >> 2) + 1;
    if (blk != buf_blk) block(blk);
    return buf[(word++) & 3];
  }
  double next_double() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }

  double standard_normal() {   // numpy random_standard_normal (ziggurat)
    for (;;) {
      uint64_t r = next();
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const int sign = (int)(r & 1);
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = (double)rabs * rld_zig_wi[idx];
      if (sign) x = -x;
      if (rabs < rld_zig_ki[idx]) return x;
      if (idx == 0) {
        for (;;) {
          const double xx = -RLD_ZIG_INV_R * std::log1p(-next_double());
          const double yy = -std::log1p(-next_double());
          if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(RLD_ZIG_R + xx) : (RLD_ZIG_R + xx);
        }
      }
      if (((rld_zig_fi[idx - 1] - rld_zig_fi[idx]) * next_double() + rld_zig_fi[idx]) < std::exp(-0.5 * x * x))
        return x;
    }
  }

  double standard_gamma(double shape) {   // numpy random_standard_gamma, shape > 1 branch
    const double b = shape - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * b);
    for (;;) {
      double X, V;
      do {
        X = standard_normal();
        V = 1.0 + c * X;
      } while (V <= 0.0);
      V = V * V * V;
      const double U = next_double();
      if (U < 1.0 - 0.0331 * (X * X) * (X * X)) return b * V;
      if (std::log(U) < 0.5 * X * X + b * (1.0 - V + std::log(V))) return b * V;
    }
  }
};

}  // namespace

void chi_radii_host(const uint64_t key[2], uint64_t word0, int64_t df, int64_t count, double* out) {
  if (df < 3) fail(RLD_ERR_NOT_SUPPORTED, "normal-orthogonal probes need n >= 3 (chi radii with df < 3)");
  HostPhilox g{key[0], key[1], word0, {0, 0, 0, 0}};
  for (int64_t i = 0; i < count; ++i) out[i] = std::sqrt(2.0 * g.standard_gamma(0.5 * (double)df));
}

}  // namespace rld

extern "C" int rld_chi_radii(const uint64_t key[2], uint64_t word0, int64_t df, int64_t count, double* out) {
  if (!key || !out || count < 0) return RLD_ERR_INVALID_ARGUMENT;
  try {
    rld::chi_radii_host(key, word0, df, count, out);
  } catch (const rld::Error& e) {
    return e.code;
  }
  return RLD_OK;
}
