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

  // x^2 as a plane map: plane b of x^2*a is the XOR of a[s] over the bits s
  // of s2(b) (compile-time constants once the plane loops are unrolled).
  __host__ __device__ static constexpr uint32_t s1(int b) {
    return (b > 0 ? (1u << (b - 1)) : 0u) ^ (((TAPS >> b) & 1u) ? (1u << (R - 1)) : 0u);
  }
  __host__ __device__ static constexpr uint32_t s2(int b) {
    uint32_t m = 0, x = s1(b);
    for (int s = 0; s < R; ++s)
      if ((x >> s) & 1u) m ^= s1(s);
    return m;
  }
  __host__ __device__ static constexpr int nbits(uint32_t m) {
    int c = 0;
    for (; m; m &= m - 1u) ++c;
    return c;
  }
  __host__ __device__ static constexpr int lowbit(uint32_t m) {
    int i = 0;
    while (i < 31 && !((m >> i) & 1u)) ++i;
    return i;
  }
  __device__ __forceinline__ static uint32_t lop3_xor(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
  }
  // Plane masks of the digit term d * v: d = 1 -> v, 2 -> x v, 3 -> (1 + x) v.
  __host__ __device__ static constexpr uint32_t dmask(int d, int b) {
    return d == 0 ? 0u : d == 1 ? (1u << b) : d == 2 ? s1(b) : (s1(b) ^ (1u << b));
  }

  // acc <- (SQ ? x^2 * acc : 0) + D * v.  Every output plane is the XOR of at
  // most 5 planes (<= 2 LOP3s); the digit term's planes come first so each
  // LOP3 is unique to its digit branch and the compiler cannot hoist the
  // reduction taps out of the branches (which would cost an extra XOR).
  template <bool SQ, int D>
  __device__ __forceinline__ static void step(uint32_t (&acc)[R], const uint32_t (&v)[R]) {
    uint32_t o[R];
#pragma unroll
    for (int b = 0; b < R; ++b) {
      const uint32_t am = SQ ? s2(b) : 0u, vm = dmask(D, b);
      uint32_t t[6];
      int n = 0;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if ((vm >> i) & 1u) t[n++] = v[i];
#pragma unroll
      for (int i = 0; i < R; ++i)
        if ((am >> i) & 1u) t[n++] = acc[i];
      uint32_t x = n ? t[0] : 0u;
      int i = 1;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (n - i >= 2) {
          x = lop3_xor(x, t[i], t[i + 1]);
          i += 2;
        } else if (n - i == 1) {
          x ^= t[i];
          i += 1;
        }
      }
      o[b] = x;
    }
#pragma unroll
    for (int b = 0; b < R; ++b) acc[b] = o[b];
  }

  template <bool SQ>
  __device__ __forceinline__ static void digit(uint32_t (&acc)[R], const uint32_t (&v)[R],
                                               uint32_t f, int t) {
    const uint32_t hi = f & (2u << (2 * t)), lo = f & (1u << (2 * t));
    if (hi) {
      if (lo)
        step<SQ, 3>(acc, v);
      else
        step<SQ, 2>(acc, v);
    } else {
      if (lo)
        step<SQ, 1>(acc, v);
      else
        step<SQ, 0>(acc, v);
    }
  }

  // acc = f * v for a warp-uniform f: Horner over the 2-bit digits of f,
  // d * v in {0, v, x v, (1 + x) v}; digits tested bit by bit.
  __device__ __forceinline__ static void mul(uint32_t (&acc)[R], const uint32_t (&v)[R],
                                             uint32_t f) {
    digit<false>(acc, v, f, ND - 1);
#pragma unroll
    for (int t = ND - 2; t >= 0; --t) digit<true>(acc, v, f, t);
  }

  // Two independent vectors sharing one warp-uniform factor: one digit
  // dispatch per step drives both (twice the independent work per branch).
  template <bool SQ>
  __device__ __forceinline__ static void digit2(uint32_t (&a0)[R], uint32_t (&a1)[R],
                                                const uint32_t (&v0)[R], const uint32_t (&v1)[R],
                                                uint32_t f, int t) {
    const uint32_t hi = f & (2u << (2 * t)), lo = f & (1u << (2 * t));
    if (hi) {
      if (lo) {
        step<SQ, 3>(a0, v0);
        step<SQ, 3>(a1, v1);
      } else {
        step<SQ, 2>(a0, v0);
        step<SQ, 2>(a1, v1);
      }
    } else {
      if (lo) {
        step<SQ, 1>(a0, v0);
        step<SQ, 1>(a1, v1);
      } else {
        step<SQ, 0>(a0, v0);
        step<SQ, 0>(a1, v1);
      }
    }
  }
  __device__ __forceinline__ static void mul2(uint32_t (&a0)[R], uint32_t (&a1)[R],
                                              const uint32_t (&v0)[R], const uint32_t (&v1)[R],
                                              uint32_t f) {
    digit2<false>(a0, a1, v0, v1, f, ND - 1);
#pragma unroll
    for (int t = ND - 2; t >= 0; --t) digit2<true>(a0, a1, v0, v1, f, t);
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
