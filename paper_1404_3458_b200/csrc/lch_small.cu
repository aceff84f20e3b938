// Small-codeword codec for GF(2^8) (config 1, SURVEY §2 "r=8 small-codeword
// variants"): one CTA per codeword, the whole codeword (n = 256 symbols) and
// the field/basis tables in shared memory, multiplies by log/exp lookups.  A
// batch of 64 codewords is one launch per encode or decode instead of the
// ~10 bit-sliced passes the batched path needs, which are launch-latency
// bound at this size.  Every step follows the reference line by line:
//   encode  rs.py:85-96      (transform.py:143-175 inverse, :102-140 forward)
//   decode  rs.py:99-149     (walsh.py:42-115 locator, derivative.py:46-77)
#include <cuda_runtime.h>

#include <cstdint>

#include "lch_kernels.h"

namespace lch {

namespace {

constexpr int SN = 256;  // n for r = 8, threads per CTA
constexpr uint32_t SM_ORD = 255;

struct SmallTables {
  uint16_t log[SN], exp[SN], w_hat[SN], b_prod[SN], b_inv[SN];
  uint32_t fwht_log[SN];
};

__device__ __forceinline__ uint32_t smul(const SmallTables &t, uint32_t a, uint32_t b) {
  if (!a || !b) return 0u;
  uint32_t s = uint32_t(t.log[a]) + t.log[b];
  s = s >= SM_ORD ? s - SM_ORD : s;
  return t.exp[s];
}

__device__ __forceinline__ void load_tables(SmallTables &t, const Small8Params &p) {
  const int i = threadIdx.x;
  t.log[i] = p.log[i];
  t.exp[i] = i < int(SM_ORD) ? p.exp[i] : p.exp[0];
  t.w_hat[i] = i < p.max_h - 1 ? p.w_hat[i] : 0;
  t.b_prod[i] = i < p.max_h ? p.b_prod[i] : 1;
  t.b_inv[i] = i < p.max_h ? p.b_prod_inv[i] : 1;
  t.fwht_log[i] = p.fwht_log[i];
}

// w_hat level i starts at max_h - (max_h >> i) (basis.py:63-69)
__device__ __forceinline__ uint32_t factor(const SmallTables &t, int max_h, int i, int j) {
  return t.w_hat[max_h - (max_h >> i) + (j >> (i + 1))];
}

// inverse, shift 0, h = 2^lg (transform.py:149-169)
__device__ __forceinline__ void inverse_s(uint32_t *a, const SmallTables &t, int max_h, int lg) {
  const int q = threadIdx.x, half_n = 1 << (lg - 1);
  for (int i = 0; i < lg; ++i) {
    if (q < half_n) {
      const int half = 1 << i;
      const int j = ((q >> i) << (i + 1)) | (q & (half - 1));
      const uint32_t v = a[j] ^ a[j + half];
      a[j + half] = v;
      a[j] ^= smul(t, v, factor(t, max_h, i, j));
    }
    __syncthreads();
  }
}

// forward with level constants hs[i] = W^_i(shift) (transform.py:108-133)
__device__ __forceinline__ void forward_s(uint32_t *a, const SmallTables &t, int max_h, int lg,
                                          const uint8_t *hs) {
  const int q = threadIdx.x, half_n = 1 << (lg - 1);
  for (int i = lg - 1; i >= 0; --i) {
    if (q < half_n) {
      const int half = 1 << i;
      const int j = ((q >> i) << (i + 1)) | (q & (half - 1));
      const uint32_t u = a[j] ^ smul(t, a[j + half], factor(t, max_h, i, j) ^ (hs ? hs[i] : 0u));
      a[j] = u;
      a[j + half] ^= u;
    }
    __syncthreads();
  }
}

// in-place Walsh-Hadamard transform mod 255 over 256 canonical residues (walsh.py:52-60)
__device__ __forceinline__ void fwht_s(uint32_t *x) {
  const int q = threadIdx.x;
  for (int h = 1; h < SN; h <<= 1) {
    if (q < SN / 2) {
      const int j = ((q / h) * 2 * h) + (q % h);
      const uint32_t a = x[j], b = x[j + h];
      const uint32_t s = a + b;
      x[j] = s >= SM_ORD ? s - SM_ORD : s;
      x[j + h] = a >= b ? a - b : a + SM_ORD - b;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SN) small8_kernel(const __grid_constant__ Small8Params p) {
  __shared__ SmallTables t;
  __shared__ uint32_t a[SN], c[SN], x[SN];
  const int q = threadIdx.x;
  const int64_t b = blockIdx.x;
  load_tables(t, p);
  if (p.mode == 0) {
    // rs.py:91 coefficients, then one forward per parity block at shift blk * k
    const int k = p.k;
    if (q < k) c[q] = p.in[b * p.in_stride + q];
    __syncthreads();
    if (p.lg_k > 0) inverse_s(c, t, p.max_h, p.lg_k);
    for (int blk = 1; blk < SN / k; ++blk) {
      if (q < k) a[q] = c[q];
      __syncthreads();
      if (p.lg_k > 0) forward_s(a, t, p.max_h, p.lg_k, p.hs + blk * 8);
      if (q < k) p.out[b * p.out_stride + (blk - 1) * k + q] = uint16_t(a[q]);
      __syncthreads();
    }
    return;
  }
  // decode
  const uint32_t *bits = p.bits + b * p.bits_stride;
  const uint32_t rx = p.in[b * p.in_stride + q];
  const uint32_t rx8 = rx & 0xFFu;  // symbols are the low r bits (as in the bit-sliced path)
  const bool er = (bits[q >> 5] >> (q & 31)) & 1u;
  // walsh.py:97-105: R^w = FWHT(FWHT(indicator) * FWHT(log)) mod 255
  x[q] = er ? 1u : 0u;
  __syncthreads();
  fwht_s(x);
  x[q] = (x[q] * t.fwht_log[q]) % SM_ORD;
  __syncthreads();
  fwht_s(x);
  const uint32_t lx = x[q];  // log of Pi_bar (survivor) or Pi' (erased)
  // rs.py:130-134 phi = received * Pi_bar on survivors
  a[q] = (er || !rx8) ? 0u : t.exp[(uint32_t(t.log[rx8]) + lx) % SM_ORD];
  __syncthreads();
  inverse_s(a, t, p.max_h, 8);  // rs.py:136
  // derivative.py:56-76: y_i = B_i d_i, out_j = B_j^-1 XOR_{l: j_l = 0} y_{j|2^l}
  c[q] = smul(t, t.b_prod[q], a[q]);
  __syncthreads();
  uint32_t acc = 0;
  for (int l = 0; l < 8; ++l)
    if (!((q >> l) & 1)) acc ^= c[q | (1 << l)];
  a[q] = smul(t, t.b_inv[q], acc);
  __syncthreads();
  forward_s(a, t, p.max_h, 8, nullptr);  // rs.py:138
  // rs.py:140-148
  if (q < p.k) {
    uint32_t o = rx;
    if (er) {
      const uint32_t d = a[q];
      o = d ? t.exp[(uint32_t(t.log[d]) + SM_ORD - lx) % SM_ORD] : 0u;
    }
    p.out[b * p.out_stride + q] = uint16_t(o);
  }
}

}  // namespace

cudaError_t launch_small8(const Small8Params &p, cudaStream_t s) {
  small8_kernel<<<unsigned(p.batch), SN, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace lch
