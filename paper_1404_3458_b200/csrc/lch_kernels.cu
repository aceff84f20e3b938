// sm_100a kernels for the LCH transform codec.
//
// pass_kernel: one CTA owns a tile of 2^tpb positions x 1024 batch lanes (one
// 32-bit word per bit-plane per thread lane, 32 codewords per word) and runs a
// short program of butterfly levels / per-position scalings on it in shared
// memory.  Every lane of a warp processes the SAME positions for different
// codewords, so butterfly factors (transform.py:112,123: w_hat[i][c>>(i+1)] ^
// W^_i(shift)) are warp-uniform and the Horner multiply branches uniformly.
// Input/output is either the raw uint16 batch (transposed to/from bit planes
// in registers) or the bit-sliced intermediate buffer (straight 2 KB block
// copies, laid out exactly like the shared-memory tile).
#include "lch_device.cuh"
#include "lch_kernels.h"

namespace lch {

namespace {

// Per-position block of the BS layout: 32 lanes x R plane-words, stored as
// R/4 16-byte chunks per lane with a lane-dependent chunk swizzle so that
// 128-bit shared-memory accesses by 8 consecutive lanes hit distinct banks.
template <int R>
struct Blk {
  static constexpr int CH = R / 4;
  static constexpr int SWS = (CH == 4) ? 1 : 2;
  static constexpr int U4 = 8 * R;  // uint4 per position block
  __device__ __forceinline__ static int chunk(int lane, int c) {
    return lane * CH + (c ^ ((lane >> SWS) & (CH - 1)));
  }
  __device__ __forceinline__ static void load(const uint4 *blk, int lane, uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint4 x = blk[chunk(lane, c)];
      v[4 * c + 0] = x.x;
      v[4 * c + 1] = x.y;
      v[4 * c + 2] = x.z;
      v[4 * c + 3] = x.w;
    }
  }
  __device__ __forceinline__ static void load_g(const uint4 *blk, int lane, uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint4 x = __ldg(blk + chunk(lane, c));
      v[4 * c + 0] = x.x;
      v[4 * c + 1] = x.y;
      v[4 * c + 2] = x.z;
      v[4 * c + 3] = x.w;
    }
  }
  __device__ __forceinline__ static void store(uint4 *blk, int lane, const uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      blk[chunk(lane, c)] = make_uint4(v[4 * c + 0], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
};

__device__ __forceinline__ void cp_async16(void *smem_ptr, const void *gptr) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_ptr));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gptr));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::);
}

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int R>
__device__ __forceinline__ void load_tile_bs(const PassParams &p, uint4 *smem,
                                             const uint32_t *tpos, int g, uint32_t base,
                                             int TP) {
  constexpr int U4 = Blk<R>::U4;
  const uint4 *src = p.bs_in + ((size_t(g) << p.lgH) * U4);
  for (int idx = threadIdx.x; idx < TP * U4; idx += NT) {
    const int q = idx / U4, c = idx - q * U4;
    cp_async16(smem + idx, src + size_t(base | tpos[q]) * U4 + c);
  }
  cp_async_wait_all();
}

template <int R>
__device__ __forceinline__ void store_tile_bs(const PassParams &p, const uint4 *smem,
                                              const uint32_t *tpos, int g, uint32_t base,
                                              int TP) {
  constexpr int U4 = Blk<R>::U4;
  uint4 *dst = p.bs_out + ((size_t(g) << p.lgH) * U4);
  for (int idx = threadIdx.x; idx < TP * U4; idx += NT) {
    const int q = idx / U4, c = idx - q * U4;
    dst[size_t(base | tpos[q]) * U4 + c] = smem[idx];
  }
}

// Raw (row-major uint16) -> bit-sliced tile.  Requires the tile to be the
// contiguous run [base, base + TP).  Lane w, bit L of a plane word = codeword
// g*1024 + 32L + w of the group.
template <int R>
__device__ __forceinline__ void load_tile_raw(const PassParams &p, uint4 *smem, int g,
                                              uint32_t base, int TP) {
  uint32_t *rs = reinterpret_cast<uint32_t *>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int WPR = TP >> 1;  // 32-bit words (position pairs) per row
  const int64_t row0 = int64_t(g) * GROUP;
  const RawIO &io = p.raw_in;
  if (io.vec && TP >= 8) {
    const int lcpr = p.tpb - 3;  // log2 of 16-byte chunks per row
    for (int idx = tid; idx < (GROUP << lcpr); idx += NT) {
      const int r = idx >> lcpr, c = idx & ((1 << lcpr) - 1);
      const int64_t b = row0 + r;
      uint4 val = make_uint4(0u, 0u, 0u, 0u);
      if (b < p.batch)
        val = ldg_stream(reinterpret_cast<const uint4 *>(io.ptr + b * io.row_stride + base) + c);
      const int sw = (r >> 1) & (WPR - 1);
      uint32_t *row = rs + r * WPR;
      row[(4 * c + 0) ^ sw] = val.x;
      row[(4 * c + 1) ^ sw] = val.y;
      row[(4 * c + 2) ^ sw] = val.z;
      row[(4 * c + 3) ^ sw] = val.w;
    }
  } else {
    for (int idx = tid; idx < GROUP * WPR; idx += NT) {
      const int r = idx / WPR, cw = idx - r * WPR;
      const int64_t b = row0 + r;
      uint32_t w = 0;
      if (b < p.batch) {
        const uint16_t *s = io.ptr + b * io.row_stride + base + 2 * cw;
        w = uint32_t(s[0]) | (uint32_t(s[1]) << 16);
      }
      rs[r * WPR + (cw ^ ((r >> 1) & (WPR - 1)))] = w;
    }
  }
  __syncthreads();
  uint32_t keep[2][2][R];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int cw = warp + s * NWARP;
    if (cw < WPR) {
      uint32_t a[32];
#pragma unroll
      for (int L = 0; L < 32; ++L) {
        const int r = 32 * L + lane;
        a[L] = rs[r * WPR + (cw ^ ((r >> 1) & (WPR - 1)))];
      }
      transpose32(a);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        keep[s][0][k] = a[k];
        keep[s][1][k] = a[16 + k];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int cw = warp + s * NWARP;
    if (cw < WPR) {
      Blk<R>::store(smem + (2 * cw) * Blk<R>::U4, lane, keep[s][0]);
      Blk<R>::store(smem + (2 * cw + 1) * Blk<R>::U4, lane, keep[s][1]);
    }
  }
}

template <int R>
__device__ __forceinline__ void store_tile_raw(const PassParams &p, uint4 *smem, int g,
                                               uint32_t base, int TP) {
  uint32_t *rs = reinterpret_cast<uint32_t *>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int WPR = TP >> 1;
  const int64_t row0 = int64_t(g) * GROUP;
  const RawIO &io = p.raw_out;
  uint32_t keep[2][32];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int cw = warp + s * NWARP;
    if (cw < WPR) {
      uint32_t v0[R], v1[R];
      Blk<R>::load(smem + (2 * cw) * Blk<R>::U4, lane, v0);
      Blk<R>::load(smem + (2 * cw + 1) * Blk<R>::U4, lane, v1);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        keep[s][k] = (k < R) ? v0[k < R ? k : 0] : 0u;
        keep[s][16 + k] = (k < R) ? v1[k < R ? k : 0] : 0u;
      }
      transpose32(keep[s]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int cw = warp + s * NWARP;
    if (cw < WPR) {
#pragma unroll
      for (int L = 0; L < 32; ++L) {
        const int r = 32 * L + lane;
        rs[r * WPR + (cw ^ ((r >> 1) & (WPR - 1)))] = keep[s][L];
      }
    }
  }
  __syncthreads();
  if (io.vec && TP >= 8) {
    const int lcpr = p.tpb - 3;
    for (int idx = tid; idx < (GROUP << lcpr); idx += NT) {
      const int r = idx >> lcpr, c = idx & ((1 << lcpr) - 1);
      const int64_t b = row0 + r;
      if (b >= p.batch) continue;
      const int sw = (r >> 1) & (WPR - 1);
      const uint32_t *row = rs + r * WPR;
      uint4 val = make_uint4(row[(4 * c + 0) ^ sw], row[(4 * c + 1) ^ sw],
                             row[(4 * c + 2) ^ sw], row[(4 * c + 3) ^ sw]);
      const uint32_t pos0 = base + 8 * c;
      if (io.merge_src) {
        const uint32_t eb = (io.merge_bits[pos0 >> 5] >> (pos0 & 31)) & 0xFFu;
        if (eb != 0xFFu) {
          const uint4 src =
              __ldg(reinterpret_cast<const uint4 *>(io.merge_src + b * io.merge_stride + pos0));
          uint32_t *vv = &val.x;
          const uint32_t *ss = &src.x;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint32_t keep_lo = (eb >> (2 * h)) & 1u, keep_hi = (eb >> (2 * h + 1)) & 1u;
            const uint32_t msk = (keep_lo ? 0x0000FFFFu : 0u) | (keep_hi ? 0xFFFF0000u : 0u);
            vv[h] = (vv[h] & msk) | (ss[h] & ~msk);
          }
        }
      }
      *(reinterpret_cast<uint4 *>(io.ptr + b * io.row_stride + base) + c) = val;
    }
  } else {
    for (int idx = tid; idx < GROUP * WPR; idx += NT) {
      const int r = idx / WPR, cw = idx - r * WPR;
      const int64_t b = row0 + r;
      if (b >= p.batch) continue;
      const uint32_t w = rs[r * WPR + (cw ^ ((r >> 1) & (WPR - 1)))];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t pos = base + 2 * cw + h;
        uint16_t v = uint16_t(h ? (w >> 16) : (w & 0xFFFFu));
        if (io.merge_src && !((io.merge_bits[pos >> 5] >> (pos & 31)) & 1u))
          v = io.merge_src[b * io.merge_stride + pos];
        io.ptr[b * io.row_stride + pos] = v;
      }
    }
  }
}

}  // namespace

template <int R, uint32_t POLY>
__global__ void __launch_bounds__(NT, 2) pass_kernel(const __grid_constant__ PassParams p) {
  using F = GF<R, POLY>;
  constexpr int U4 = Blk<R>::U4;
  extern __shared__ uint4 smem[];
  __shared__ uint32_t tpos[1 << TPB_MAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int TP = 1 << p.tpb;
  const uint32_t t = blockIdx.x;
  const int g = blockIdx.y;

  uint32_t base = 0;
  for (int i = 0; i < p.nnb; ++i) base |= ((t >> i) & 1u) << p.nbit[i];
  if (tid < TP) {
    uint32_t o = 0;
    for (int m = 0; m < p.tpb; ++m) o |= ((uint32_t(tid) >> m) & 1u) << p.gbit[m];
    tpos[tid] = o;
  }
  __syncthreads();

  if (p.in_mode == IO_BS)
    load_tile_bs<R>(p, smem, tpos, g, base, TP);
  else
    load_tile_raw<R>(p, smem, g, base, TP);
  __syncthreads();

  for (int o = 0; o < p.nops; ++o) {
    const int kind = p.ops[o].kind;
    if (kind == OP_SCALE) {
      const uint16_t *tab = p.ops[o].table;
      for (int q = warp; q < TP; q += NWARP) {
        const uint32_t f = __ldg(tab + (base | tpos[q]));
        uint32_t v[R], acc[R];
        Blk<R>::load(smem + q * U4, lane, v);
        if (f) {
          F::mul(acc, v, f);
        } else {
#pragma unroll
          for (int b = 0; b < R; ++b) acc[b] = 0u;
        }
        Blk<R>::store(smem + q * U4, lane, acc);
      }
    } else {
      const int m = p.ops[o].m, lvl = p.ops[o].level;
      const uint32_t hs = p.ops[o].hs;
      const uint16_t *hat = p.w_hat + p.w_hat_off[lvl];
      for (int pp = warp; pp < (TP >> 1); pp += NWARP) {
        const int qu = ((pp >> m) << (m + 1)) | (pp & ((1 << m) - 1));
        const int qv = qu | (1 << m);
        const uint32_t pos_u = base | tpos[qu];
        const uint32_t f = __ldg(hat + (pos_u >> (lvl + 1))) ^ hs;
        uint32_t u[R], v[R];
        Blk<R>::load(smem + qu * U4, lane, u);
        Blk<R>::load(smem + qv * U4, lane, v);
        if (kind == OP_FWD) {
          // transform.py:126-133: u' = u + f v, v' = u' + v
          if (f) {
            uint32_t fv[R];
            F::mul(fv, v, f);
            F::xor_into(u, fv);
          }
          F::xor_into(v, u);
        } else {
          // transform.py:165-169: v' = u + v, u' = u + f v'
          F::xor_into(v, u);
          if (f) {
            uint32_t fv[R];
            F::mul(fv, v, f);
            F::xor_into(u, fv);
          }
        }
        Blk<R>::store(smem + qu * U4, lane, u);
        Blk<R>::store(smem + qv * U4, lane, v);
      }
    }
    __syncthreads();
  }

  if (p.out_mode == IO_BS)
    store_tile_bs<R>(p, smem, tpos, g, base, TP);
  else
    store_tile_raw<R>(p, smem, g, base, TP);
}

// T[pos] (+)= XOR over tile bits m with bit m of q clear of g[pos | 2^gbit[m]],
// for pos < 2^lgH_out: the gather step of derivative.py:60-70, split by bit
// groups so the full sum over all lg h bits takes ceil(lg h / tpb) passes.
template <int R>
__global__ void __launch_bounds__(NT, 2) gather_kernel(const __grid_constant__ GatherParams p) {
  constexpr int U4 = Blk<R>::U4;
  extern __shared__ uint4 smem[];
  __shared__ uint32_t tpos[1 << TPB_MAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int TP = 1 << p.tpb;
  const uint32_t t = blockIdx.x;
  const int g = blockIdx.y;
  uint32_t base = 0;
  for (int i = 0; i < p.nnb; ++i) base |= ((t >> i) & 1u) << p.nbit[i];
  const uint32_t hout = 1u << p.lgH_out;
  if (tid < TP) {
    uint32_t o = 0;
    for (int m = 0; m < p.tpb; ++m) o |= ((uint32_t(tid) >> m) & 1u) << p.gbit[m];
    tpos[tid] = o;
  }
  __syncthreads();
  if (base >= hout) {
    // all positions >= hout unless a tile bit reaches below hout's top; tile
    // positions only add bits, so base >= hout means the whole tile is out.
    return;
  }
  const uint4 *src = p.g + ((size_t(g) << p.lgH_in) * U4);
  for (int idx = tid; idx < TP * U4; idx += NT) {
    const int q = idx / U4, c = idx - q * U4;
    cp_async16(smem + idx, src + size_t(base | tpos[q]) * U4 + c);
  }
  cp_async_wait_all();
  __syncthreads();
  uint4 *tb = p.t + ((size_t(g) << p.lgH_out) * U4);
  for (int q = warp; q < TP; q += NWARP) {
    const uint32_t pos = base | tpos[q];
    if (pos >= hout) continue;
    uint32_t acc[R];
    if (p.acc_in) {
      Blk<R>::load_g(tb + size_t(pos) * U4, lane, acc);
    } else {
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0u;
    }
    for (int m = 0; m < p.tpb; ++m) {
      if ((q >> m) & 1) continue;
      uint32_t x[R];
      Blk<R>::load(smem + (q | (1 << m)) * U4, lane, x);
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] ^= x[b];
    }
    Blk<R>::store(tb + size_t(pos) * U4, lane, acc);
  }
}

// Walsh-Hadamard transform over Z_mod, bits [b0, b0 + tb) of each vector
// (walsh.py:42-61), with the locator's fused prologue/epilogue
// (walsh.py:97-114): indicator from a bitmask, pointwise product with
// FWHT(log), and exp[] of the result split into Pi_bar / Pi' rows.
__global__ void fwht_kernel(const __grid_constant__ FwhtParams p) {
  __shared__ uint32_t s[256];
  const int q = threadIdx.x;
  const int TB = 1 << p.tb;
  const int64_t nt = int64_t(1) << (p.lgn - p.tb);
  const int64_t vec = blockIdx.x / nt;
  const uint32_t t = uint32_t(blockIdx.x - vec * nt);
  const uint32_t lowmask = (1u << p.b0) - 1u;
  const uint32_t pos = (t & lowmask) | (uint32_t(q) << p.b0) | ((t >> p.b0) << (p.b0 + p.tb));
  const size_t n = size_t(1) << p.lgn;
  const size_t idx = size_t(vec) * n + pos;
  const size_t words = (n + 31) / 32;
  const uint64_t mod = p.mod;
  uint32_t x;
  if (p.bits)
    x = (p.bits[size_t(vec) * words + (pos >> 5)] >> (pos & 31)) & 1u;
  else
    x = p.data[idx];
  x = uint32_t(uint64_t(x) % mod);
  s[q] = x;
  __syncthreads();
  for (int h = 1; h < TB; h <<= 1) {
    if (!(q & h)) {
      const uint64_t a = s[q], b = s[q + h];
      const uint64_t sum = a + b;
      s[q] = uint32_t(sum >= mod ? sum - mod : sum);
      s[q + h] = uint32_t(a >= b ? a - b : a + mod - b);
    }
    __syncthreads();
  }
  x = s[q];
  if (p.post_mul) x = uint32_t((uint64_t(x) * p.post_mul[pos]) % mod);
  if (p.exp) {
    const uint16_t val = p.exp[x];
    if (p.loc_out) p.loc_out[idx] = val;
    if (p.log_out) p.log_out[idx] = uint16_t(x);
  } else {
    p.data[idx] = x;
  }
}

// decode rows from the locator logs: pi_row[j] = erased ? 0 : exp[x],
// pinv[j] = (erased && j < k) ? exp[(m - x) % m] : 0   (rs.py:130-148)
__global__ void decode_rows_kernel(const uint16_t *logs, const uint32_t *bits,
                                   const uint16_t *exp, uint32_t m, uint32_t n, uint32_t k,
                                   uint16_t *pi_row, uint16_t *pinv) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t x = logs[j];
    const bool erased = (bits[j >> 5] >> (j & 31)) & 1u;
    pi_row[j] = erased ? uint16_t(0) : exp[x];
    if (j < k) pinv[j] = erased ? exp[(m - x) % m] : uint16_t(0);
  }
}

__device__ __forceinline__ uint64_t mix64_d(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t key_d(uint64_t seed, uint64_t cw, uint64_t pos) {
  const uint64_t s = mix64_d(seed + 0x9E3779B97F4A7C15ull);
  return mix64_d(s + ((cw << 32) | pos) * 0x9E3779B97F4A7C15ull);
}

__global__ void gen_symbols_kernel(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                                   uint32_t mask, uint16_t *out, int64_t row_stride) {
  const int64_t total = batch * len;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / len, j = i - b * len;
    out[b * row_stride + j] = uint16_t(key_d(seed, cw0 + uint64_t(b), uint64_t(j)) & mask);
  }
}

__global__ void gen_keys_kernel(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                                int64_t *keys) {
  const int64_t total = batch * len;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / len, j = i - b * len;
    keys[i] = int64_t(key_d(seed, cw0 + uint64_t(b), uint64_t(j)) >> 1);
  }
}

__global__ void count_bits_kernel(const uint32_t *bits, int64_t npatterns, int words,
                                  int64_t *counts) {
  __shared__ int64_t red[256];
  const int64_t pidx = blockIdx.x;
  int64_t c = 0;
  for (int w = threadIdx.x; w < words; w += blockDim.x) c += __popc(bits[pidx * words + w]);
  red[threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[pidx] = red[0];
}

// ---------------------------------------------------------------------------

size_t pass_smem_bytes(int R, int tpb, bool raw) {
  const size_t tp = size_t(1) << tpb;
  size_t bs = tp * 8 * R * 16;
  size_t rw = raw ? size_t(GROUP) * tp * 2 : 0;
  return bs > rw ? bs : rw;
}

template <int R, uint32_t POLY>
cudaError_t launch_pass(const PassParams &p, int ngroups, cudaStream_t s) {
  const bool raw = p.in_mode == IO_RAW || p.out_mode == IO_RAW;
  const size_t smem = pass_smem_bytes(R, p.tpb, raw);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(pass_kernel<R, POLY>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(pass_smem_bytes(R, TPB_MAX, true)));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(1u << (p.lgH - p.tpb), ngroups);
  pass_kernel<R, POLY><<<grid, NT, smem, s>>>(p);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_gather(const GatherParams &p, int ngroups, cudaStream_t s) {
  const size_t smem = pass_smem_bytes(R, p.tpb, false);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gather_kernel<R>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(pass_smem_bytes(R, TPB_MAX, false)));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(1u << (p.lgH_in - p.tpb), ngroups);
  gather_kernel<R><<<grid, NT, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwht(const FwhtParams &p, cudaStream_t s) {
  const int64_t blocks = p.nvec * (int64_t(1) << (p.lgn - p.tb));
  fwht_kernel<<<unsigned(blocks), 1 << p.tb, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_decode_rows(const uint16_t *logs, const uint32_t *bits, const uint16_t *exp,
                               uint32_t m, uint32_t n, uint32_t k, uint16_t *pi_row,
                               uint16_t *pinv, cudaStream_t s) {
  decode_rows_kernel<<<(n + 255) / 256, 256, 0, s>>>(logs, bits, exp, m, n, k, pi_row, pinv);
  return cudaGetLastError();
}

cudaError_t launch_gen_symbols(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                               uint32_t mask, uint16_t *out, int64_t row_stride,
                               cudaStream_t s) {
  const int64_t total = batch * len;
  const int blocks = int(total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32);
  gen_symbols_kernel<<<blocks, 256, 0, s>>>(seed, cw0, batch, len, mask, out, row_stride);
  return cudaGetLastError();
}

cudaError_t launch_gen_keys(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                            int64_t *keys, cudaStream_t s) {
  const int64_t total = batch * len;
  const int blocks = int(total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32);
  gen_keys_kernel<<<blocks, 256, 0, s>>>(seed, cw0, batch, len, keys);
  return cudaGetLastError();
}

cudaError_t launch_count_bits(const uint32_t *bits, int64_t npatterns, int words,
                              int64_t *counts, cudaStream_t s) {
  count_bits_kernel<<<unsigned(npatterns), 256, 0, s>>>(bits, npatterns, words, counts);
  return cudaGetLastError();
}

template cudaError_t launch_pass<16, 0x1100Bu>(const PassParams &, int, cudaStream_t);
template cudaError_t launch_pass<8, 0x11Du>(const PassParams &, int, cudaStream_t);
template cudaError_t launch_gather<16>(const GatherParams &, int, cudaStream_t);
template cudaError_t launch_gather<8>(const GatherParams &, int, cudaStream_t);

}  // namespace lch
