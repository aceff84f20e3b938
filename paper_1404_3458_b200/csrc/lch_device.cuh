// Device helpers: bit-sliced GF(2^R) arithmetic and a 32x32 bit transpose.
//
// Bit-sliced ("BS") representation used by every transform kernel: a value
// of R 32-bit words, word b = bit-plane b of 32 symbols that belong to 32
// different codewords (batch lanes).  Field addition is a plane-wise XOR
// (field.py:1-13: element index == representation); multiplication by a
// warp-uniform constant f is evaluated by a Horner scheme over the 2-bit
// digits of f, using only XORs of whole planes:
//     f*v = (((d_top * v) x^2 + d_.. * v) x^2 + ...) ,  d * v in {0, v, xv, v+xv}
// where x*v is a plane rotation plus XORs at the taps of the reduction
// polynomial.  All 32 symbols of a word share the factor, so one thread
// multiplies 32 symbols with ~R/2 * (R + taps) XORs.
#pragma once

#include <cstdint>

namespace lch {

template <int R, uint32_t POLY>
struct GF {
  static_assert(R == 8 || R == 16, "R must be 8 or 16");
  static constexpr uint32_t TAPS = POLY & ((1u << R) - 1u);
  static constexpr int ND = R / 2;  // 2-bit digits of a factor

  // o = x * a  (multiplication by the field generator x, polynomial basis)
  __device__ __forceinline__ static void mulx(const uint32_t (&a)[R], uint32_t (&o)[R]) {
#pragma unroll
    for (int b = 0; b < R; ++b) {
      uint32_t t = (b > 0) ? a[b - 1] : 0u;
      if ((TAPS >> b) & 1u) t ^= a[R - 1];
      o[b] = t;
    }
  }

  __device__ __forceinline__ static void xor_into(uint32_t (&a)[R], const uint32_t (&b)[R]) {
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] ^= b[i];
  }

  // acc = f * v for a warp-uniform f != 0.
  __device__ __forceinline__ static void mul(uint32_t (&acc)[R], const uint32_t (&v)[R],
                                             uint32_t f) {
    uint32_t xv[R], vx[R];
    mulx(v, xv);
#pragma unroll
    for (int b = 0; b < R; ++b) vx[b] = v[b] ^ xv[b];
    {
      const uint32_t d = (f >> (2 * (ND - 1))) & 3u;
      if (d == 0u) {
#pragma unroll
        for (int b = 0; b < R; ++b) acc[b] = 0u;
      } else if (d == 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) acc[b] = v[b];
      } else if (d == 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) acc[b] = xv[b];
      } else {
#pragma unroll
        for (int b = 0; b < R; ++b) acc[b] = vx[b];
      }
    }
#pragma unroll
    for (int t = ND - 2; t >= 0; --t) {
      uint32_t tmp[R];
      mulx(acc, tmp);
      mulx(tmp, acc);
      const uint32_t d = (f >> (2 * t)) & 3u;
      if (d == 1u) {
        xor_into(acc, v);
      } else if (d == 2u) {
        xor_into(acc, xv);
      } else if (d == 3u) {
        xor_into(acc, vx);
      }
    }
  }

  // acc = f_lane * v where the factor differs per lane (not warp-uniform):
  // branch-free, 1-bit digits selected by lane masks.
  __device__ __forceinline__ static void mul_lane(uint32_t (&acc)[R], const uint32_t (&v)[R],
                                                  uint32_t f) {
#pragma unroll
    for (int b = 0; b < R; ++b) acc[b] = 0u;
#pragma unroll
    for (int t = R - 1; t >= 0; --t) {
      uint32_t tmp[R];
      mulx(acc, tmp);
      const uint32_t msk = 0u - ((f >> t) & 1u);
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = tmp[b] ^ (v[b] & msk);
    }
  }

  // acc = a * b for two bit-sliced operands (per-symbol factors).
  __device__ __forceinline__ static void mul_bs(uint32_t (&acc)[R], const uint32_t (&a)[R],
                                                const uint32_t (&b)[R]) {
    // Horner over the planes of b (MSB first): acc = x*acc + a & b_t
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0u;
#pragma unroll
    for (int t = R - 1; t >= 0; --t) {
      uint32_t tmp[R];
      mulx(acc, tmp);
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = tmp[i] ^ (a[i] & b[t]);
    }
  }
};

// 32x32 bit-matrix transpose in registers: bit c of a[r] <-> bit r of a[c].
// Stages 16 and 8 are byte permutes; 4, 2, 1 are masked swaps.
__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t x = a[k], y = a[k + 16];
    a[k] = __byte_perm(x, y, 0x5410);
    a[k + 16] = __byte_perm(x, y, 0x7632);
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 8) continue;
    const uint32_t x = a[k], y = a[k + 8];
    a[k] = __byte_perm(x, y, 0x6240);
    a[k + 8] = __byte_perm(x, y, 0x7351);
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 4) continue;
    const uint32_t t = ((a[k] >> 4) ^ a[k + 4]) & 0x0F0F0F0Fu;
    a[k + 4] ^= t;
    a[k] ^= t << 4;
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 2) continue;
    const uint32_t t = ((a[k] >> 2) ^ a[k + 2]) & 0x33333333u;
    a[k + 2] ^= t;
    a[k] ^= t << 2;
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k & 1) continue;
    const uint32_t t = ((a[k] >> 1) ^ a[k + 1]) & 0x55555555u;
    a[k + 1] ^= t;
    a[k] ^= t << 1;
  }
}

}  // namespace lch
