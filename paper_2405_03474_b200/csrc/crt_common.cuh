// Moduli of the CRT float64 product (kv_crt.cu), shared with the slicing kernels of kv_ozaki.cu
// that emit K's residue image straight from the points.
#pragma once

namespace rld {

constexpr int CRT_L = 15;           // moduli used
constexpr int OZ_NSLICES = 7;       // int8 digits (base 256) per float64 entry in the slice image (kv_ozaki.cu)
constexpr int CRT_SLICES = 6;       // K' = sum_{s<6} d_s 256^{5-s}: the first 6 exact slices (48 bits)

__host__ __device__ constexpr int crt_mod(int l) {
  // pairwise coprime, largest first: 2^8, 3.5.17, 11.23, 251, 13.19, 241, 239, 233, 229, 227, 223, 7.31, 211, 199, 197
  return l == 0 ? 256 : l == 1 ? 255 : l == 2 ? 253 : l == 3 ? 251 : l == 4 ? 247 : l == 5 ? 241 : l == 6 ? 239
       : l == 7 ? 233 : l == 8 ? 229 : l == 9 ? 227 : l == 10 ? 223 : l == 11 ? 217 : l == 12 ? 211 : l == 13 ? 199
       : 197;
}

// symmetric representative of 2^e mod p (|.| <= p / 2), for the 16-bit-chunk residue split
__host__ __device__ constexpr int crt_pow2_sym(int e, int p) {
  int r = 1;
  for (int i = 0; i < e; ++i) r = (r * 2) % p;
  return r > p / 2 ? r - p : r;
}

// symmetric residue of an int32 x modulo p (odd p: [-(p-1)/2, (p-1)/2]; p = 256: [-128, 127])
__device__ __forceinline__ int sym_mod(int x, int p) {
  int r = x % p;
  if (r > (p - 1) / 2) r -= p;
  if (r < -(p / 2)) r += p;
  return r;
}

}  // namespace rld
