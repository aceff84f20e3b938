// Device helpers: bit-sliced GF(2^R) arithmetic and a 32x32 bit transpose.
//
// Bit-sliced ("BS") representation used by every transform kernel: a value
// of R 32-bit words, word b = bit-plane b of 32 symbols that belong to 32
// different codewords (batch lanes).  Field addition is a plane-wise XOR
// (field.py:1-13: element index == representation); multiplication by a
// warp-uniform constant f is evaluated by a Horner scheme over the 2-bit
// digits of f, using only XORs of whole planes:
//     f*v = sum_t d_t * (x^(2t) v),  d * p in {0, p, xp, p+xp}
// where x*p is a plane rotation plus XORs at the taps of the reduction
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

  // x ^ XOR_{s in m} p[s] (m a compile-time plane set once the callers'
  // plane loops are unrolled): terms paired into 3-input LOP3s.
  __device__ __forceinline__ static uint32_t xor_into_set(uint32_t x, const uint32_t (&p)[R],
                                                          uint32_t m) {
    uint32_t pend = 0u;
    bool has = false;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      if ((m >> s) & 1u) {
        if (has) {
          x = lop3_xor(x, pend, p[s]);
          has = false;
        } else {
          pend = p[s];
          has = true;
        }
      }
    }
    return has ? (x ^ pend) : x;
  }
  // XOR_{s in m} p[s]
  __device__ __forceinline__ static uint32_t xor_set(const uint32_t (&p)[R], uint32_t m) {
    if (m == 0u) return 0u;
    const int s0 = lowbit(m);
    return xor_into_set(p[s0], p, m & (m - 1u));
  }

  // u += f * v for a warp-uniform f.  f v = sum_t d_t (x^(2t) v) over the
  // 2-bit digits d_t of f, least significant first: p = x^(2t) v advances
  // unconditionally (plane renames plus the reduction taps) and only
  // u += d_t p (d p in {p, x p, (1 + x) p}) sits under the warp-uniform digit
  // branch, updating u in place, so the branch paths join without register
  // moves.  ~R/2 * (R + taps) XORs per 32 symbols.
  __device__ __forceinline__ static void mul_acc(uint32_t (&u)[R], const uint32_t (&v)[R],
                                                 uint32_t f) {
    uint32_t p[R];
#pragma unroll
    for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
    for (int t = 0; t < ND; ++t) {
      const uint32_t d = (f >> (2 * t)) & 3u;
      if (d == 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
      } else if (d == 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = xor_into_set(u[b], p, dmask(2, b));
      } else if (d == 3u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = xor_into_set(u[b], p, dmask(3, b));
      }
      if (t + 1 < ND) {
        uint32_t q[R];
#pragma unroll
        for (int b = 0; b < R; ++b) q[b] = xor_set(p, s2(b));
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = q[b];
      }
    }
  }

  // Measured alternatives (build with -DLCH_MUL_LAZY / -DLCH_MUL_LAZY2 /
  // -DLCH_MUL_2BIT; all bit-exact, none faster than mul_acc_1 in the pass
  // kernel: 1.41 / 1.48 / 1.47 ms vs 1.41 ms per RS(2^16,2^15) encode of 4096).
  // Lazy-reduction multiply: u + f v accumulated as an unreduced polynomial
  // of degree <= 2R-2 (planes R..2R-2 in h[]), so the set bits of f only
  // XOR shifted copies of v (no per-bit x*p updates and no dependency chain
  // through them); one reduction of h[] by the taps at the end.
  __device__ __forceinline__ static void lazy_reduce(uint32_t (&u)[R], uint32_t (&h)[R - 1]) {
    // x^i = x^(i-R) * TAPS for i >= R, top plane first (targets above R cascade)
#pragma unroll
    for (int i = 2 * R - 2; i >= R; --i) {
      const uint32_t x = h[i - R];
#pragma unroll
      for (int s = 0; s < R; ++s) {
        if (!((TAPS >> s) & 1u)) continue;
        const int t = i - R + s;
        if (t < R)
          u[t < R ? t : 0] ^= x;
        else
          h[t >= R ? t - R : 0] ^= x;
      }
    }
  }
  __device__ __forceinline__ static void mul_acc_lazy(uint32_t (&u)[R], const uint32_t (&v)[R],
                                                      uint32_t f) {
    uint32_t h[R - 1];
#pragma unroll
    for (int i = 0; i < R - 1; ++i) h[i] = 0u;
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if ((f >> t) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          const int i = t + b;
          if (i < R)
            u[i < R ? i : 0] ^= v[b];
          else
            h[i >= R ? i - R : 0] ^= v[b];
        }
      }
    }
    lazy_reduce(u, h);
  }
  // 2-bit digits: d = 3 pairs the two shifted copies in one 3-input LOP3 per plane
  __device__ __forceinline__ static void mul_acc_lazy2(uint32_t (&u)[R], const uint32_t (&v)[R],
                                                       uint32_t f) {
    uint32_t h[R - 1];
#pragma unroll
    for (int i = 0; i < R - 1; ++i) h[i] = 0u;
    auto pl = [&](int i) -> uint32_t & { return i < R ? u[i < R ? i : 0] : h[i >= R ? i - R : 0]; };
#pragma unroll
    for (int t = 0; t < ND; ++t) {
      const uint32_t d = (f >> (2 * t)) & 3u;
      const int o = 2 * t;
      if (d == 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) pl(o + b) ^= v[b];
      } else if (d == 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) pl(o + 1 + b) ^= v[b];
      } else if (d == 3u) {
        pl(o) ^= v[0];
#pragma unroll
        for (int b = 1; b < R; ++b) pl(o + b) = lop3_xor(pl(o + b), v[b], v[b - 1]);
        pl(o + R) ^= v[R - 1];
      }
    }
    lazy_reduce(u, h);
  }

  // Nested 2-bit digits: per digit (bits t, t+1) two warp-uniform branches,
  // as many as the 1-bit form, but a digit with both bits set adds p + x p
  // in ONE 3-input LOP3 per plane (u ^= p ^ q): 3/4 * 16 body ops per digit
  // instead of 2 * 1/2 * 16.  p and q = x p are both computed every digit
  // (the same tap XORs the 1-bit form spends), so no body does extra work.
  __device__ __forceinline__ static void mul_acc_n2(uint32_t (&u)[R], const uint32_t (&v)[R],
                                                    uint32_t f) {
    uint32_t p[R];
#pragma unroll
    for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
    for (int t = 0; t < R; t += 2) {
      uint32_t q[R];
#pragma unroll
      for (int b = 0; b < R; ++b) q[b] = xor_set(p, s1(b));
      if ((f >> t) & 1u) {
        if ((f >> (t + 1)) & 1u) {
#pragma unroll
          for (int b = 0; b < R; ++b) u[b] = lop3_xor(u[b], p[b], q[b]);
        } else {
#pragma unroll
          for (int b = 0; b < R; ++b) u[b] ^= p[b];
        }
      } else if ((f >> (t + 1)) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= q[b];
      }
      if (t + 2 < R) {
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = xor_set(q, s1(b));
      }
    }
  }
  __device__ __forceinline__ static void mul_acc2_n2(uint32_t (&u0)[R], const uint32_t (&v0)[R],
                                                     uint32_t (&u1)[R], const uint32_t (&v1)[R],
                                                     uint32_t f) {
    uint32_t p0[R], p1[R];
#pragma unroll
    for (int b = 0; b < R; ++b) {
      p0[b] = v0[b];
      p1[b] = v1[b];
    }
#pragma unroll
    for (int t = 0; t < R; t += 2) {
      uint32_t q0[R], q1[R];
#pragma unroll
      for (int b = 0; b < R; ++b) {
        q0[b] = xor_set(p0, s1(b));
        q1[b] = xor_set(p1, s1(b));
      }
      if ((f >> t) & 1u) {
        if ((f >> (t + 1)) & 1u) {
#pragma unroll
          for (int b = 0; b < R; ++b) {
            u0[b] = lop3_xor(u0[b], p0[b], q0[b]);
            u1[b] = lop3_xor(u1[b], p1[b], q1[b]);
          }
        } else {
#pragma unroll
          for (int b = 0; b < R; ++b) {
            u0[b] ^= p0[b];
            u1[b] ^= p1[b];
          }
        }
      } else if ((f >> (t + 1)) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] ^= q0[b];
          u1[b] ^= q1[b];
        }
      }
      if (t + 2 < R) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          p0[b] = xor_set(q0, s1(b));
          p1[b] = xor_set(q1, s1(b));
        }
      }
    }
  }

  // Compact forms of mul_acc_n2 / mul_acc2_n2: a rolled loop over 4 bits of f
  // per iteration (two nested 2-bit digits), so a multiply is ~100
  // instructions of code instead of ~450 (instruction-cache footprint of the
  // pass kernel); p = x^t v is the only loop-carried state.
  __device__ __forceinline__ static void digit_acc(uint32_t (&u)[R], const uint32_t (&p)[R],
                                                   const uint32_t (&q)[R], uint32_t d) {
    if (d & 1u) {
      if (d & 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = lop3_xor(u[b], p[b], q[b]);
      } else {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
      }
    } else if (d & 2u) {
#pragma unroll
      for (int b = 0; b < R; ++b) u[b] ^= q[b];
    }
  }
  __device__ __forceinline__ static void mul_acc_l(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) {
    uint32_t p[R];
#pragma unroll
    for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll 1
    for (int t = 0; t < R; t += 4) {
      uint32_t q[R], p2[R], q2[R];
#pragma unroll
      for (int b = 0; b < R; ++b) q[b] = xor_set(p, s1(b));
      digit_acc(u, p, q, (f >> t) & 3u);
#pragma unroll
      for (int b = 0; b < R; ++b) p2[b] = xor_set(q, s1(b));
#pragma unroll
      for (int b = 0; b < R; ++b) q2[b] = xor_set(p2, s1(b));
      digit_acc(u, p2, q2, (f >> (t + 2)) & 3u);
#pragma unroll
      for (int b = 0; b < R; ++b) p[b] = xor_set(q2, s1(b));
    }
  }
  __device__ __forceinline__ static void digit_acc2(uint32_t (&u0)[R], const uint32_t (&p0)[R],
                                                    const uint32_t (&q0)[R], uint32_t (&u1)[R],
                                                    const uint32_t (&p1)[R], const uint32_t (&q1)[R],
                                                    uint32_t d) {
    if (d & 1u) {
      if (d & 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] = lop3_xor(u0[b], p0[b], q0[b]);
          u1[b] = lop3_xor(u1[b], p1[b], q1[b]);
        }
      } else {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] ^= p0[b];
          u1[b] ^= p1[b];
        }
      }
    } else if (d & 2u) {
#pragma unroll
      for (int b = 0; b < R; ++b) {
        u0[b] ^= q0[b];
        u1[b] ^= q1[b];
      }
    }
  }
  __device__ __forceinline__ static void mul_acc2_l(uint32_t (&u0)[R], const uint32_t (&v0)[R],
                                                    uint32_t (&u1)[R], const uint32_t (&v1)[R],
                                                    uint32_t f) {
    uint32_t p0[R], p1[R];
#pragma unroll
    for (int b = 0; b < R; ++b) {
      p0[b] = v0[b];
      p1[b] = v1[b];
    }
#pragma unroll 1
    for (int t = 0; t < R; t += 2) {
      uint32_t q0[R], q1[R];
#pragma unroll
      for (int b = 0; b < R; ++b) {
        q0[b] = xor_set(p0, s1(b));
        q1[b] = xor_set(p1, s1(b));
      }
      digit_acc2(u0, p0, q0, u1, p1, q1, (f >> t) & 3u);
#pragma unroll
      for (int b = 0; b < R; ++b) {
        p0[b] = xor_set(q0, s1(b));
        p1[b] = xor_set(q1, s1(b));
      }
    }
  }

#ifndef LCH_MUL_2BIT
  // 1-bit digits: one warp-uniform branch per bit of f (fewer taken
  // branches than the 2-bit digits below: measured 4-5% faster passes)
  __device__ __forceinline__ static void mul_acc_1(uint32_t (&u)[R], const uint32_t (&v)[R],
                                                   uint32_t f) {
    uint32_t p[R];
#pragma unroll
    for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      // x * p for the next bit is computed ahead of this bit's branch, so
      // its tap XORs are ready by the time the next body reads them
      uint32_t q[R];
      if (t + 1 < R) {
#pragma unroll
        for (int b = 0; b < R; ++b) q[b] = xor_set(p, s1(b));
      }
      if ((f >> t) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
      }
      if (t + 1 < R) {
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = q[b];
      }
    }
  }
  __device__ __forceinline__ static void mul_acc2_1(uint32_t (&u0)[R], const uint32_t (&v0)[R],
                                                    uint32_t (&u1)[R], const uint32_t (&v1)[R],
                                                    uint32_t f) {
    uint32_t p0[R], p1[R];
#pragma unroll
    for (int b = 0; b < R; ++b) {
      p0[b] = v0[b];
      p1[b] = v1[b];
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if ((f >> t) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] ^= p0[b];
          u1[b] ^= p1[b];
        }
      }
      if (t + 1 < R) {
        uint32_t q0[R], q1[R];
#pragma unroll
        for (int b = 0; b < R; ++b) {
          q0[b] = xor_set(p0, s1(b));
          q1[b] = xor_set(p1, s1(b));
        }
#pragma unroll
        for (int b = 0; b < R; ++b) {
          p0[b] = q0[b];
          p1[b] = q1[b];
        }
      }
    }
  }
#endif

  // u0 += f * v0 and u1 += f * v1 under one digit dispatch (twice the
  // independent work per warp-uniform branch).
  __device__ __forceinline__ static void mul_acc2(uint32_t (&u0)[R], const uint32_t (&v0)[R],
                                                  uint32_t (&u1)[R], const uint32_t (&v1)[R],
                                                  uint32_t f) {
    uint32_t p0[R], p1[R];
#pragma unroll
    for (int b = 0; b < R; ++b) {
      p0[b] = v0[b];
      p1[b] = v1[b];
    }
#pragma unroll
    for (int t = 0; t < ND; ++t) {
      const uint32_t d = (f >> (2 * t)) & 3u;
      if (d == 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] ^= p0[b];
          u1[b] ^= p1[b];
        }
      } else if (d == 2u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] = xor_into_set(u0[b], p0, dmask(2, b));
          u1[b] = xor_into_set(u1[b], p1, dmask(2, b));
        }
      } else if (d == 3u) {
#pragma unroll
        for (int b = 0; b < R; ++b) {
          u0[b] = xor_into_set(u0[b], p0, dmask(3, b));
          u1[b] = xor_into_set(u1[b], p1, dmask(3, b));
        }
      }
      if (t + 1 < ND) {
        uint32_t q0[R], q1[R];
#pragma unroll
        for (int b = 0; b < R; ++b) {
          q0[b] = xor_set(p0, s2(b));
          q1[b] = xor_set(p1, s2(b));
        }
#pragma unroll
        for (int b = 0; b < R; ++b) {
          p0[b] = q0[b];
          p1[b] = q1[b];
        }
      }
    }
  }

  // acc = f * v
  __device__ __forceinline__ static void mul(uint32_t (&acc)[R], const uint32_t (&v)[R],
                                             uint32_t f) {
#pragma unroll
    for (int b = 0; b < R; ++b) acc[b] = 0u;
    mul_acc_n2(acc, v, f);
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

// The same multiplies for a reduction polynomial known only at run time (any
// primitive polynomial, field.py:28-53): taps in a warp-uniform register, so
// x * p costs one masked XOR per plane instead of one XOR per tap.
template <int R>
struct GFrt {
  uint32_t taps;  // POLY & (2^R - 1)
  __device__ __forceinline__ void step(const uint32_t (&p)[R], uint32_t (&q)[R]) const {
    const uint32_t top = p[R - 1];
#pragma unroll
    for (int b = 0; b < R; ++b) q[b] = (b ? p[b > 0 ? b - 1 : 0] : 0u) ^ (top & (0u - ((taps >> b) & 1u)));
  }
  __device__ __forceinline__ void mul_acc(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) const {
    uint32_t p[R];
#pragma unroll
    for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if ((f >> t) & 1u) {
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
      }
      if (t + 1 < R) {
        uint32_t q[R];
        step(p, q);
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = q[b];
      }
    }
  }
  __device__ __forceinline__ void mul_acc2(uint32_t (&u0)[R], const uint32_t (&v0)[R], uint32_t (&u1)[R],
                                           const uint32_t (&v1)[R], uint32_t f) const {
    mul_acc(u0, v0, f);
    mul_acc(u1, v1, f);
  }
  __device__ __forceinline__ void mul(uint32_t (&acc)[R], const uint32_t (&v)[R], uint32_t f) const {
#pragma unroll
    for (int b = 0; b < R; ++b) acc[b] = 0u;
    mul_acc(acc, v, f);
  }
};

// Product of two GF(2^16) symbols (polynomial basis, x^16 + x^12 + x^3 + x + 1,
// field.py:100-129) without tables.  gf16_clmul: the carry-less 16x16
// product from 9 integer multiplies of bit-interleaved thirds (the bits of a
// and b spaced 3 apart, so a partial coefficient is at most 6 < 8 and the
// parity bits of one residue class never collide); gf16_fold: reduction by
// the taps in four folds of the high half (or two byte-table lookups where a
// kernel keeps gf16_red tables in shared memory).
__device__ __forceinline__ uint32_t gf16_clmul(uint32_t a, uint32_t b) {
  const uint32_t a0 = a & 0x9249u, a1 = a & 0x2492u, a2 = a & 0x4924u;
  const uint32_t b0 = b & 0x9249u, b1 = b & 0x2492u, b2 = b & 0x4924u;
  const uint32_t z0 = (a0 * b0) ^ (a1 * b2) ^ (a2 * b1);
  const uint32_t z1 = (a0 * b1) ^ (a1 * b0) ^ (a2 * b2);
  const uint32_t z2 = (a0 * b2) ^ (a1 * b1) ^ (a2 * b0);
  return (z0 & 0x49249249u) | (z1 & 0x92492492u) | (z2 & 0x24924924u);
}
__host__ __device__ __forceinline__ uint32_t gf16_fold(uint32_t z) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // degree 30 -> 26 -> 22 -> 18 -> 14
    const uint32_t h = z >> 16;
    z = (z & 0xFFFFu) ^ h ^ (h << 1) ^ (h << 3) ^ (h << 12);
  }
  return z;
}
__device__ __forceinline__ uint32_t gf16_mul(uint32_t a, uint32_t b) { return gf16_fold(gf16_clmul(a, b)); }
// gf16_red: red[x] = (x << 16) mod p for x < 256, red[256 + x] = (x << 24) mod p
// for x < 128, so clmul(a, b) mod p = low ^ red[byte 2] ^ red[256 + byte 3].
__device__ __forceinline__ uint32_t gf16_mul_t(uint32_t a, uint32_t b, const uint32_t *red) {
  const uint32_t z = gf16_clmul(a, b);
  return (z & 0xFFFFu) ^ red[(z >> 16) & 0xFFu] ^ red[256 + (z >> 24)];
}

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
