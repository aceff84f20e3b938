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
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "lch_device.cuh"
#include "lch_kernels.h"

#ifdef LCH_PASS_DBG
#define PDBG(x) (p.dbg & (x))  // LCH_DBG_PASS bisection flags (experiment builds only)
#else
#define PDBG(x) 0
#endif

namespace lch {

namespace {

// Per-position block of the BS layout: 32 lanes x R plane-words, stored
// chunk-major: 16-byte chunk c (planes 4c..4c+3) of lane w at c * 32 + w, so a
// warp's 128-bit access to one chunk covers 512 contiguous bytes (shared
// memory: conflict-free; global memory: fully coalesced).
template <int R>
struct Blk {
  static constexpr int CH = R / 4;
  static constexpr int U4 = 8 * R;  // uint4 per position block
  __device__ __forceinline__ static int chunk(int lane, int c) { return c * 32 + lane; }
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
  // straight from registers to global memory (streaming stores)
  __device__ __forceinline__ static void store_g(uint4 *blk, int lane, const uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      __stcs(blk + chunk(lane, c), make_uint4(v[4 * c + 0], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
  }
};

// --- TMA (bulk async copy) + mbarrier helpers -------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_add_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// generic-proxy smem accesses before -> async-proxy (TMA) writes after
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tma_store_1d(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void cp_async16(void *smem_ptr, const void *gptr) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_ptr));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gptr));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::);
}


template <int R>
__device__ __forceinline__ void store_tile_bs(const PassParams &p, const uint4 *smem,
                                              const uint32_t *tpos, int g, uint32_t base,
                                              int TP) {
  if (PDBG(5)) return;
  constexpr int U4 = Blk<R>::U4;
  uint4 *dst = p.bs_out + ((size_t(g) << p.lgH) * U4);
  for (int idx = threadIdx.x; idx < TP * U4; idx += NT) {
    const int q = idx / U4, c = idx - q * U4;
    dst[size_t(base | tpos[q]) * U4 + c] = smem[idx];
  }
}



// Raw staging for row-major uint16 tiles (tile = contiguous run [base,
// base + TP) of 1024 rows): 32-bit words w(row, cw) = positions (2cw, 2cw+1),
// stored column-major, word column cw at [cw * 1024, cw * 1024 + 1024) with
// the row index XOR-swizzled by 8 * ((cw >> 2) & 3) (conflict-free for both the
// 4-column stores of a 16-byte row chunk and the transposing column reads).
// A column is exactly the 4 KB the two BS blocks of positions 2cw, 2cw+1
// occupy (R = 16), so one warp transposes a column in place; for R = 8 the
// BS tile lives past the staging area.  Lane w, bit L of a plane word =
// codeword g*1024 + 32L + w of the group.
__device__ __forceinline__ int stage_idx(int r, int cw) {
  return cw * GROUP + (r ^ (8 * ((cw >> 2) & 3)));
}

template <int R>
__host__ __device__ constexpr int bs_offset_u4() {
  return R == 16 ? 0 : GROUP * (1 << TPB_MAX) * 2 / 16;
}
// half-tile staging area for the bulk stores of the last round, after the tile
template <int R>
__host__ __device__ constexpr int stage_offset_u4() {
  return bs_offset_u4<R>() + (1 << TPB_MAX) * 8 * R;
}

// Raw element address (see RawIO); b = batch index, j = position.
__device__ __forceinline__ const uint16_t *raw_addr(const RawIO &io, int64_t b, int64_t j) {
  if (io.pkt) return io.ptr + ((b / io.pkt) * io.npos + (j - io.pos_lo)) * io.pkt + b % io.pkt;
  return io.ptr + b * io.row_stride + (j - io.pos_lo);
}

// Issue the loads of a tile: BS input asynchronously (TMA bulk copies, see
// below), raw input synchronously through registers into the staging layout.
template <int R, bool BS_ONLY, bool ROWONLY = false>
__device__ __forceinline__ void issue_tile(const PassParams &p, uint4 *smem, const uint32_t *tpos,
                                           int g, uint32_t base, int TP, uint64_t *bar) {
  if (BS_ONLY || p.in_mode == IO_BS) {
    // lane 0 of every warp issues the blocks q = warp, warp + 8, ...; thread 0
    // supplies the barrier's single arrival
    if ((threadIdx.x & 31) == 0) {
      constexpr int U4 = Blk<R>::U4;
      uint4 *bs = smem + bs_offset_u4<R>();
      const uint4 *src = p.bs_in + ((size_t(g) << p.lgH) * U4);
      const int w = threadIdx.x >> 5;
      fence_proxy_async();
      if (!(PDBG(9))) {
        int nq = 0;
        for (int q = w; q < TP; q += NWARP) ++nq;
        if (nq) mbar_add_tx(bar, unsigned(nq * U4 * 16));
        for (int q = w; q < TP; q += NWARP)
          tma_load_1d(bs + q * U4, src + size_t(base | tpos[q]) * U4, U4 * 16, bar);
      }
      if (w == 0) mbar_arrive(bar);
    }
    return;
  }
  if (PDBG(9)) return;
  if (R == 16 && p.raw_tma) {
    // one thread: 4 chunks x 4 row blocks of 256, 64 KB, zero-filled outside
    // the input (rows >= batch, positions outside [pos_lo, pos_hi))
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_expect_tx(bar, 64u * 1024u);
      const int c0 = int((int64_t(base) - p.raw_in.pos_lo) >> 3);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int rb = 0; rb < 4; ++rb)
          tma_load_3d(smem + c * 1024 + rb * 256, &p.tm_in, 0, c0 + c, g * GROUP + rb * 256, bar);
    }
    return;
  }
  if (R == 16 && p.raw_bulk) {
    // packet layout: 32 bulk copies of 2 KB (one per position, lane 0 of
    // each warp issues 4); a tile outside the window arrives without bytes
    // and is zeroed by finish_tile_raw_bulk
    const RawIO &io = p.raw_in;
    const bool in = int64_t(base) >= io.pos_lo && int64_t(base) < io.pos_hi;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
      fence_proxy_async();
      if (w == 0) {
        if (in)
          mbar_expect_tx(bar, 64u * 1024u);
        else
          mbar_arrive(bar);
      }
      if (in) {
        const int64_t row0 = int64_t(g) * GROUP;
        for (int q = 4 * w; q < 4 * w + 4; ++q)
          tma_load_1d(smem + q * 128, raw_addr(io, row0, int64_t(base) + q), 2048u, bar);
      }
    }
    return;
  }
  uint32_t *rs = reinterpret_cast<uint32_t *>(smem);
  const int WPR = TP >> 1;
  const int64_t row0 = int64_t(g) * GROUP;
  const RawIO &io = p.raw_in;
  const bool inwin = int64_t(base) >= io.pos_lo && int64_t(base) + TP <= io.pos_hi;
  if (int64_t(base) + TP <= io.pos_lo || int64_t(base) >= io.pos_hi) {
    // tile entirely outside the input window: zeros
    uint4 *z = smem;
    for (int idx = threadIdx.x; idx < WPR * (GROUP / 4); idx += NT) z[idx] = make_uint4(0u, 0u, 0u, 0u);
  } else if (!ROWONLY && io.pkt && inwin) {
    // packet-major: 1024 consecutive symbols per position; a thread takes 8
    // rows of one word column (positions 2cw, 2cw+1) and interleaves them
    for (int idx = threadIdx.x; idx < WPR * (GROUP / 8); idx += NT) {
      const int cw = idx / (GROUP / 8), r8 = idx - cw * (GROUP / 8);
      const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(raw_addr(io, row0 + 8 * r8, base + 2 * cw)));
      const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(raw_addr(io, row0 + 8 * r8, base + 2 * cw + 1)));
      uint4 lo, hi;
      lo.x = __byte_perm(a.x, b.x, 0x5410); lo.y = __byte_perm(a.x, b.x, 0x7632);
      lo.z = __byte_perm(a.y, b.y, 0x5410); lo.w = __byte_perm(a.y, b.y, 0x7632);
      hi.x = __byte_perm(a.z, b.z, 0x5410); hi.y = __byte_perm(a.z, b.z, 0x7632);
      hi.z = __byte_perm(a.w, b.w, 0x5410); hi.w = __byte_perm(a.w, b.w, 0x7632);
      uint4 *dst = reinterpret_cast<uint4 *>(rs + stage_idx(8 * r8, cw));
      dst[0] = lo;
      dst[1] = hi;
    }
  } else if (!io.pkt && io.vec && TP >= 8 && inwin) {
    const int lcpr = p.tpb - 3;
    for (int idx = threadIdx.x; idx < (GROUP << lcpr); idx += NT) {
      const int r = idx >> lcpr, c = idx & ((1 << lcpr) - 1);
      const int64_t b = row0 + r;
      uint4 val = make_uint4(0u, 0u, 0u, 0u);
      if (b < p.batch) val = __ldcs(reinterpret_cast<const uint4 *>(raw_addr(io, b, base)) + c);
      rs[stage_idx(r, 4 * c + 0)] = val.x;
      rs[stage_idx(r, 4 * c + 1)] = val.y;
      rs[stage_idx(r, 4 * c + 2)] = val.z;
      rs[stage_idx(r, 4 * c + 3)] = val.w;
    }
  } else {  // small / partial tiles, unaligned rows: element loads
    for (int idx = threadIdx.x; idx < GROUP * WPR; idx += NT) {
      const int r = idx / WPR, cw = idx - r * WPR;
      const int64_t b = row0 + r;
      uint32_t w = 0;
      if (b < p.batch) {
        const int64_t j = int64_t(base) + 2 * cw;
        const uint32_t lo = (j >= io.pos_lo && j < io.pos_hi) ? *raw_addr(io, b, j) : 0u;
        const uint32_t hi = (j + 1 >= io.pos_lo && j + 1 < io.pos_hi) ? *raw_addr(io, b, j + 1) : 0u;
        w = lo | (hi << 16);
      }
      rs[stage_idx(r, cw)] = w;
    }
  }
}

// Raw staging -> bit-sliced tile, one word column per warp (in place).
template <int R>
__device__ __forceinline__ void finish_tile_raw(uint4 *smem, int TP) {
  const uint32_t *rs = reinterpret_cast<const uint32_t *>(smem);
  uint4 *bs = smem + bs_offset_u4<R>();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int WPR = TP >> 1;
  for (int cw = warp; cw < WPR; cw += NWARP) {
    uint32_t a[32];
#pragma unroll
    for (int L = 0; L < 32; ++L) a[L] = rs[stage_idx(32 * L + lane, cw)];
    __syncwarp();
    transpose32(a);
    uint32_t lo[R], hi[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      lo[k] = a[k];
      hi[k] = a[16 + k];
    }
    Blk<R>::store(bs + (2 * cw) * Blk<R>::U4, lane, lo);
    Blk<R>::store(bs + (2 * cw + 1) * Blk<R>::U4, lane, hi);
  }
}

// TMA-staged raw tile ([chunk c][row][16 B], c = positions 8c..8c+7) ->
// bit-sliced tile, in place: chunk c's 16 KB are exactly the BS blocks of
// positions 8c..8c+7.  Warps 2c, 2c+1 own chunk c; each reads two 32-bit
// words (4 positions) of every row, then both sync and write back.
template <int R>
__device__ __forceinline__ void finish_tile_raw_tma(uint4 *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = warp >> 1, wp = (warp & 1) * 2;
  const uint32_t *reg = reinterpret_cast<const uint32_t *>(smem) + c * 4096 + wp;
  uint32_t a[32], b[32];
#pragma unroll
  for (int L = 0; L < 32; ++L) {
    const uint2 v = *reinterpret_cast<const uint2 *>(reg + (32 * L + lane) * 4);
    a[L] = v.x;
    b[L] = v.y;
  }
  named_sync(1 + c, 64);
  transpose32(a);
  transpose32(b);
  uint32_t x[R];
  uint4 *bs = smem + (8 * c + 2 * wp) * Blk<R>::U4;
#pragma unroll
  for (int k = 0; k < R; ++k) x[k] = a[k];
  Blk<R>::store(bs, lane, x);
#pragma unroll
  for (int k = 0; k < R; ++k) x[k] = a[16 + k];
  Blk<R>::store(bs + Blk<R>::U4, lane, x);
#pragma unroll
  for (int k = 0; k < R; ++k) x[k] = b[k];
  Blk<R>::store(bs + 2 * Blk<R>::U4, lane, x);
#pragma unroll
  for (int k = 0; k < R; ++k) x[k] = b[16 + k];
  Blk<R>::store(bs + 3 * Blk<R>::U4, lane, x);
}

// The same conversion straight into the registers of a first round over tile
// bits (0, 1): after the transposes warp w holds the four consecutive
// positions 4w .. 4w+3 of its lane-word -- exactly that round's operands, so
// the tile skips one shared-memory round trip and one CTA barrier.  The
// round's results then overwrite the raw bytes in place; the pair barrier
// keeps warp 2c+1's reads ahead of warp 2c's stores (and vice versa).
template <int R>
__device__ __forceinline__ void raw_tma_tile_to_regs(const uint4 *smem, uint32_t (&x0)[R], uint32_t (&x1)[R],
                                                     uint32_t (&x2)[R], uint32_t (&x3)[R]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = warp >> 1, wp = (warp & 1) * 2;
  const uint32_t *reg = reinterpret_cast<const uint32_t *>(smem) + c * 4096 + wp;
  uint32_t a[32], b[32];
#pragma unroll
  for (int L = 0; L < 32; ++L) {
    const uint2 v = *reinterpret_cast<const uint2 *>(reg + (32 * L + lane) * 4);
    a[L] = v.x;
    b[L] = v.y;
  }
  named_sync(1 + c, 64);
  transpose32(a);
  transpose32(b);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    x0[k] = a[k];
    x1[k] = a[16 + k];
    x2[k] = b[k];
    x3[k] = b[16 + k];
  }
}

// Bulk-staged packet tile ([position][1024 lanes] of uint16) -> bit-sliced
// tile in place: warp w owns positions 4w .. 4w+3, two at a time (their 4 KB
// of rows become their 4 KB of BS blocks), so only warp-level syncs.
template <int R>
__device__ __forceinline__ void finish_tile_raw_bulk(uint4 *smem, bool in) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint16_t *sv = reinterpret_cast<const uint16_t *>(smem);
#pragma unroll 1
  for (int pp = 0; pp < 2; ++pp) {
    const int p0 = 4 * warp + 2 * pp;
    uint32_t a[32];
    if (in) {
#pragma unroll
      for (int L = 0; L < 32; ++L)
        a[L] = uint32_t(sv[p0 * GROUP + 32 * L + lane]) | (uint32_t(sv[(p0 + 1) * GROUP + 32 * L + lane]) << 16);
      __syncwarp();
      transpose32(a);
    } else {
#pragma unroll
      for (int L = 0; L < 32; ++L) a[L] = 0u;
    }
    uint32_t x[R];
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = a[k];
    Blk<R>::store(smem + p0 * Blk<R>::U4, lane, x);
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = a[16 + k];
    Blk<R>::store(smem + (p0 + 1) * Blk<R>::U4, lane, x);
  }
}

template <int R>
__device__ __forceinline__ void column_to_words(const uint4 *bs, int cw, int lane, uint32_t (&a)[32]) {
  uint32_t v0[R], v1[R];
  Blk<R>::load(bs + (2 * cw) * Blk<R>::U4, lane, v0);
  Blk<R>::load(bs + (2 * cw + 1) * Blk<R>::U4, lane, v1);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    a[k] = (k < R) ? v0[k < R ? k : 0] : 0u;
    a[16 + k] = (k < R) ? v1[k < R ? k : 0] : 0u;
  }
  transpose32(a);
}

template <int R, bool ROWONLY = false>
__device__ __forceinline__ void store_tile_raw(const PassParams &p, uint4 *smem, int g, const uint32_t *red,
                                               uint32_t base, int TP) {
  if (PDBG(5)) return;
  if (int64_t(base) + TP <= p.raw_out.pos_lo || int64_t(base) >= p.raw_out.pos_hi) return;
  uint32_t *rs = reinterpret_cast<uint32_t *>(smem);
  const uint4 *bs = smem + bs_offset_u4<R>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int WPR = TP >> 1;
  const int64_t row0 = int64_t(g) * GROUP;
  const RawIO &io = p.raw_out;
  for (int cw = warp; cw < WPR; cw += NWARP) {
    uint32_t a[32];
    column_to_words<R>(bs, cw, lane, a);
    __syncwarp();
#pragma unroll
    for (int L = 0; L < 32; ++L) rs[stage_idx(32 * L + lane, cw)] = a[L];
  }
  __syncthreads();
  const bool inwin = int64_t(base) >= io.pos_lo && int64_t(base) + TP <= io.pos_hi;
  auto erased_at = [&](int64_t b, int64_t j) -> bool {
    const int64_t row = io.pkt ? b / io.pkt : b;
    return (io.merge_bits[row * io.bits_stride + (j >> 5)] >> (j & 31)) & 1u;
  };
  if (!ROWONLY && io.pkt && inwin) {
    for (int idx = tid; idx < WPR * (GROUP / 8); idx += NT) {
      const int cw = idx / (GROUP / 8), r8 = idx - cw * (GROUP / 8);
      const uint4 *srcw = reinterpret_cast<const uint4 *>(rs + stage_idx(8 * r8, cw));
      const uint4 lo = srcw[0], hi = srcw[1];
      uint4 a, b;  // positions 2cw (low halves) and 2cw + 1 (high halves), 8 symbols each
      a.x = __byte_perm(lo.x, lo.y, 0x5410); b.x = __byte_perm(lo.x, lo.y, 0x7632);
      a.y = __byte_perm(lo.z, lo.w, 0x5410); b.y = __byte_perm(lo.z, lo.w, 0x7632);
      a.z = __byte_perm(hi.x, hi.y, 0x5410); b.z = __byte_perm(hi.x, hi.y, 0x7632);
      a.w = __byte_perm(hi.z, hi.w, 0x5410); b.w = __byte_perm(hi.z, hi.w, 0x7632);
      const int64_t bb = row0 + 8 * r8;
      const int64_t j0 = int64_t(base) + 2 * cw;
      if (io.merge_src) {  // packet erasures: the 8 symbols share the flag
        // packet layout: merge_stride = positions per stripe group of merge_src
        const uint16_t *ms = io.merge_src + (bb / io.pkt) * io.merge_stride * io.pkt + bb % io.pkt;
        if (!erased_at(bb, j0)) a = __ldg(reinterpret_cast<const uint4 *>(ms + j0 * io.pkt));
        if (!erased_at(bb, j0 + 1)) b = __ldg(reinterpret_cast<const uint4 *>(ms + (j0 + 1) * io.pkt));
      }
      *reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, bb, j0))) = a;
      *reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, bb, j0 + 1))) = b;
    }
  } else if (R == 16 && !io.pkt && io.vec && TP == 32 && inwin && io.merge_src && io.pinv_log && io.pinv_val &&
             ((io.pinv_stride & 7) | (reinterpret_cast<uintptr_t>(io.pinv_log) & 15)) == 0) {
    // per-codeword patterns (rs.decode row by row): erased j < k get the
    // computed value times 1 / Pi'(row, j) (table-free products), survivors
    // are copied from merge_src; each thread's 16 row chunks in batches of 4
    // with all their loads (bitmask word, 1 / Pi' and survivor chunks) in
    // flight before any is consumed
    constexpr int NB = 4, PER = (GROUP * 4) / NT / NB;
#pragma unroll 1
    for (int h = 0; h < NB; ++h) {
      uint4 src[PER], pw[PER];
      uint32_t ebs[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = tid + (h * PER + i) * NT;
        const int r = idx >> 2, c = idx & 3;
        const int64_t b = row0 + r;
        const uint32_t pos0 = base + 8 * c;
        uint32_t eb = 0u;
        if (b < p.batch) eb = (io.merge_bits[b * io.bits_stride + (pos0 >> 5)] >> (pos0 & 31)) & 0xFFu;
        ebs[i] = eb;
        const bool ok = b < p.batch;
        src[i] = ok && eb != 0xFFu
                     ? __ldg(reinterpret_cast<const uint4 *>(io.merge_src + b * io.merge_stride + pos0))
                     : make_uint4(0u, 0u, 0u, 0u);
        pw[i] = ok && eb ? __ldg(reinterpret_cast<const uint4 *>(io.pinv_log + b * io.pinv_stride + pos0))
                         : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = tid + (h * PER + i) * NT;
        const int r = idx >> 2, c = idx & 3;
        const int64_t b = row0 + r;
        if (b >= p.batch) continue;
        uint4 val = make_uint4(rs[stage_idx(r, 4 * c + 0)], rs[stage_idx(r, 4 * c + 1)],
                               rs[stage_idx(r, 4 * c + 2)], rs[stage_idx(r, 4 * c + 3)]);
        uint32_t *vv = &val.x;
        const uint32_t *ss = &src[i].x, *pp = &pw[i].x;
        const uint32_t eb = ebs[i];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t w = vv[q];
          if ((eb >> (2 * q)) & 1u) w = (w & 0xFFFF0000u) | gf16_mul_t(w & 0xFFFFu, pp[q] & 0xFFFFu, red);
          else w = (w & 0xFFFF0000u) | (ss[q] & 0xFFFFu);
          if ((eb >> (2 * q + 1)) & 1u) w = (w & 0xFFFFu) | (gf16_mul_t(w >> 16, pp[q] >> 16, red) << 16);
          else w = (w & 0xFFFFu) | (ss[q] & 0xFFFF0000u);
          vv[q] = w;
        }
        reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, b, base)))[c] = val;
      }
    }
  } else if (!io.pkt && io.vec && TP == 32 && inwin && io.merge_src && !io.pinv_log) {
    // survivors merged from merge_src (decode, rs.py:140-148): each thread's
    // 16 row chunks in four batches of 4, all 4 survivor loads in flight before
    // any is consumed (a load per chunk would wait a full memory round trip
    // each: the stores below may alias merge_src for the compiler)
    constexpr int NBATCH = 4, HALF_ITEMS = (GROUP * 4) / NT / NBATCH;
#pragma unroll 1
    for (int h = 0; h < NBATCH; ++h) {
      uint4 src[HALF_ITEMS];
      uint32_t ebs[HALF_ITEMS];
#pragma unroll
      for (int i = 0; i < HALF_ITEMS; ++i) {
        const int idx = tid + (h * HALF_ITEMS + i) * NT;
        const int r = idx >> 2, c = idx & 3;
        const int64_t b = row0 + r;
        const uint32_t pos0 = base + 8 * c;
        uint32_t eb = 0xFFu;
        if (b < p.batch) eb = (io.merge_bits[b * io.bits_stride + (pos0 >> 5)] >> (pos0 & 31)) & 0xFFu;
        ebs[i] = eb;
        if (p.merge_tma && c < 2)  // prefetched by TMA into the spare area: [chunk][row][16 B]
          src[i] = smem[stage_offset_u4<R>() + c * GROUP + r];
        else
          src[i] = eb != 0xFFu ? __ldg(reinterpret_cast<const uint4 *>(io.merge_src + b * io.merge_stride + pos0))
                               : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int i = 0; i < HALF_ITEMS; ++i) {
        const int idx = tid + (h * HALF_ITEMS + i) * NT;
        const int r = idx >> 2, c = idx & 3;
        const int64_t b = row0 + r;
        if (b >= p.batch) continue;
        uint4 val = make_uint4(rs[stage_idx(r, 4 * c + 0)], rs[stage_idx(r, 4 * c + 1)],
                               rs[stage_idx(r, 4 * c + 2)], rs[stage_idx(r, 4 * c + 3)]);
        const uint32_t eb = ebs[i];
        if (eb != 0xFFu) {
          uint32_t *vv = &val.x;
          const uint32_t *ss = &src[i].x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t keep_lo = (eb >> (2 * q)) & 1u, keep_hi = (eb >> (2 * q + 1)) & 1u;
            const uint32_t msk = (keep_lo ? 0x0000FFFFu : 0u) | (keep_hi ? 0xFFFF0000u : 0u);
            vv[q] = (vv[q] & msk) | (ss[q] & ~msk);
          }
        }
        reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, b, base)))[c] = val;
      }
    }
  } else if (!io.pkt && io.vec && TP >= 8 && inwin) {
    const int lcpr = p.tpb - 3;
    for (int idx = tid; idx < (GROUP << lcpr); idx += NT) {
      const int r = idx >> lcpr, c = idx & ((1 << lcpr) - 1);
      const int64_t b = row0 + r;
      if (b >= p.batch) continue;
      uint4 val = make_uint4(rs[stage_idx(r, 4 * c + 0)], rs[stage_idx(r, 4 * c + 1)],
                             rs[stage_idx(r, 4 * c + 2)], rs[stage_idx(r, 4 * c + 3)]);
      const uint32_t pos0 = base + 8 * c;
      if (io.merge_src) {
        const uint32_t *mb = io.merge_bits + b * io.bits_stride;
        const uint32_t eb = (mb[pos0 >> 5] >> (pos0 & 31)) & 0xFFu;
        uint32_t *vv = &val.x;
        if (io.pinv_log && eb) {
          bool eb_done = false;
          // erased j: computed * alpha^pinv_log(b, j) (division by Pi'(j),
          // rs.py:141-148); the 8 log gathers, then the 8 exp gathers, are
          // issued together, and both exponents are < mord so one conditional
          // subtraction reduces their sum
          const uint16_t *pl = io.pinv_log + b * io.pinv_stride + pos0;
          uint32_t pw[4];
          if (((io.pinv_stride & 7) | (reinterpret_cast<uintptr_t>(io.pinv_log) & 15)) == 0) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(pl));
            pw[0] = q.x, pw[1] = q.y, pw[2] = q.z, pw[3] = q.w;
          } else {
#pragma unroll
            for (int h = 0; h < 4; ++h) pw[h] = uint32_t(__ldg(pl + 2 * h)) | (uint32_t(__ldg(pl + 2 * h + 1)) << 16);
          }
          if constexpr (R == 16) {
            if (io.pinv_val) {  // 1 / Pi' as values: table-free products
#pragma unroll
              for (int h = 0; h < 8; ++h) {
                if (!((eb >> h) & 1u)) continue;
                const uint32_t sh = 16 * (h & 1);
                const uint32_t y = gf16_mul((vv[h >> 1] >> sh) & 0xFFFFu, (pw[h >> 1] >> sh) & 0xFFFFu);
                vv[h >> 1] = (vv[h >> 1] & ~(0xFFFFu << sh)) | (y << sh);
              }
              eb_done = true;
            }
          }
          uint32_t lg[8];
#pragma unroll
          for (int h = 0; h < 8 && !eb_done; ++h) {
            const uint32_t x = (vv[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
            lg[h] = (((eb >> h) & 1u) && x) ? uint32_t(__ldg(io.log_tab + x)) : 0u;
          }
#pragma unroll
          for (int h = 0; h < 8 && !eb_done; ++h) {
            if (!((eb >> h) & 1u)) continue;
            const uint32_t sh = 16 * (h & 1);
            const uint32_t x = (vv[h >> 1] >> sh) & 0xFFFFu;
            uint32_t t = lg[h] + ((pw[h >> 1] >> sh) & 0xFFFFu);
            t = t >= io.mord ? t - io.mord : t;
            const uint32_t y = x ? uint32_t(__ldg(io.exp_tab + t)) : 0u;
            vv[h >> 1] = (vv[h >> 1] & ~(0xFFFFu << sh)) | (y << sh);
          }
        }
        if (eb != 0xFFu) {
          const uint4 src =
              __ldg(reinterpret_cast<const uint4 *>(io.merge_src + b * io.merge_stride + pos0));
          const uint32_t *ss = &src.x;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint32_t keep_lo = (eb >> (2 * h)) & 1u, keep_hi = (eb >> (2 * h + 1)) & 1u;
            const uint32_t msk = (keep_lo ? 0x0000FFFFu : 0u) | (keep_hi ? 0xFFFF0000u : 0u);
            vv[h] = (vv[h] & msk) | (ss[h] & ~msk);
          }
        }
      }
      reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, b, base)))[c] = val;
    }
  } else {
    for (int idx = tid; idx < GROUP * WPR; idx += NT) {
      const int r = idx / WPR, cw = idx - r * WPR;
      const int64_t b = row0 + r;
      if (b >= p.batch) continue;
      const uint32_t w = rs[stage_idx(r, cw)];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t pos = int64_t(base) + 2 * cw + h;
        if (pos < io.pos_lo || pos >= io.pos_hi) continue;
        uint16_t v = uint16_t(h ? (w >> 16) : (w & 0xFFFFu));
        if (io.merge_src) {
          if (!erased_at(b, pos)) {
            v = io.pkt ? io.merge_src[((b / io.pkt) * io.merge_stride + pos) * io.pkt + b % io.pkt]
                       : io.merge_src[b * io.merge_stride + pos];
          } else if (io.pinv_log && v) {
            bool done = false;
            if constexpr (R == 16) {
              if (io.pinv_val) {
                v = uint16_t(gf16_mul(v, io.pinv_log[b * io.pinv_stride + pos]));
                done = true;
              }
            }
            if (!done) {
              uint32_t t = uint32_t(io.log_tab[v]) + io.pinv_log[b * io.pinv_stride + pos];
              v = io.exp_tab[t >= io.mord ? t - io.mord : t];
            }
          }
        }
        *const_cast<uint16_t *>(raw_addr(io, b, pos)) = v;
      }
    }
  }
}

// Raw row-major output straight from the last round's registers (R = 16, row
// layout, tile = positions 32t .. 32t+31 inside the output window, last round
// over tile bits 1 and 0): the thread's four blocks are the consecutive
// positions q0 .. q0+3 (x0..x3) of its lane-word, so two 32x32 bit transposes
// in registers give, for every L, the 8 bytes of row 32L + lane at those
// positions.  The rows leave through a half-tile staging area in the spare
// shared memory (512 rows x 64 B at a time, the column-major swizzled word
// layout of stage_idx) as coalesced 16-byte row chunks -- while the next
// tile's blocks already stream into the tile buffer.
__device__ __forceinline__ int stage_idx_h(int r, int cw) { return cw * (GROUP / 2) + (r ^ (8 * ((cw >> 2) & 3))); }

__device__ __forceinline__ void store_rows_from_regs(const PassParams &p, uint4 *smem, int g, uint32_t base,
                                                     int q0, uint32_t (&x0)[16], uint32_t (&x1)[16],
                                                     uint32_t (&x2)[16], uint32_t (&x3)[16]) {
  uint32_t *rs = reinterpret_cast<uint32_t *>(smem + stage_offset_u4<16>());
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t A[32], B[32];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    A[k] = x0[k];
    A[16 + k] = x1[k];
    B[k] = x2[k];
    B[16 + k] = x3[k];
  }
  transpose32(A);
  transpose32(B);
  const int cw = q0 >> 1;
  const RawIO &io = p.raw_out;
  const int64_t row0 = int64_t(g) * GROUP;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      rs[stage_idx_h(32 * l + lane, cw)] = A[16 * h + l];
      rs[stage_idx_h(32 * l + lane, cw + 1)] = B[16 * h + l];
    }
    __syncthreads();
    if (!(PDBG(5))) {
#pragma unroll 4
      for (int i = 0; i < (GROUP / 2) * 4 / NT; ++i) {
        const int idx = tid + i * NT;
        const int r = idx >> 2, c = idx & 3;
        const int64_t b = row0 + (GROUP / 2) * h + r;
        if (b < p.batch) {
          const uint4 val = make_uint4(rs[stage_idx_h(r, 4 * c + 0)], rs[stage_idx_h(r, 4 * c + 1)],
                                       rs[stage_idx_h(r, 4 * c + 2)], rs[stage_idx_h(r, 4 * c + 3)]);
          reinterpret_cast<uint4 *>(const_cast<uint16_t *>(raw_addr(io, b, base)))[c] = val;
        }
      }
    }
    if (h == 0) __syncthreads();  // half 1 refills the staging area
  }
}

}  // namespace

// Multiplier: the compile-time-polynomial GF<R, POLY>, or (POLY == 0) the
// runtime-taps GFrt<R> for any other primitive polynomial.
template <int R, uint32_t POLY>
struct Mul {
  __device__ __forceinline__ explicit Mul(uint32_t) {}
  __device__ __forceinline__ void acc(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) const {
    using F = GF<R, POLY>;
#if defined(LCH_MUL_LAZY)
    F::mul_acc_lazy(u, v, f);
#elif defined(LCH_MUL_LAZY2)
    F::mul_acc_lazy2(u, v, f);
#elif defined(LCH_MUL_LOOP)
    F::mul_acc_l(u, v, f);
#elif defined(LCH_MUL_1BIT)
    F::mul_acc_1(u, v, f);
#elif !defined(LCH_MUL_2BIT)
    F::mul_acc_n2(u, v, f);
#else
    F::mul_acc(u, v, f);
#endif
  }
  __device__ __forceinline__ void acc2(uint32_t (&u0)[R], const uint32_t (&v0)[R], uint32_t (&u1)[R],
                                       const uint32_t (&v1)[R], uint32_t f) const {
    using F = GF<R, POLY>;
#if defined(LCH_MUL_LOOP)
    F::mul_acc2_l(u0, v0, u1, v1, f);
#elif defined(LCH_MUL_1BIT)
    F::mul_acc2_1(u0, v0, u1, v1, f);
#elif !defined(LCH_MUL_2BIT)
    F::mul_acc2_n2(u0, v0, u1, v1, f);
#else
    F::mul_acc2(u0, v0, u1, v1, f);
#endif
  }
  __device__ __forceinline__ void mul(uint32_t (&a)[R], const uint32_t (&v)[R], uint32_t f) const {
    GF<R, POLY>::mul(a, v, f);
  }
};
template <int R>
struct Mul<R, 0u> {
  GFrt<R> g;
  __device__ __forceinline__ explicit Mul(uint32_t taps) : g{taps} {}
  __device__ __forceinline__ void acc(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) const {
    g.mul_acc(u, v, f);
  }
  __device__ __forceinline__ void acc2(uint32_t (&u0)[R], const uint32_t (&v0)[R], uint32_t (&u1)[R],
                                       const uint32_t (&v1)[R], uint32_t f) const {
    g.mul_acc2(u0, v0, u1, v1, f);
  }
  __device__ __forceinline__ void mul(uint32_t (&a)[R], const uint32_t (&v)[R], uint32_t f) const {
    g.mul(a, v, f);
  }
};

// The 32 factors of a single scaling over a full tile (lane l: tile position
// l), requested ahead of the phase so the load's latency hides behind the
// work in between (the raw tile's transposes, the rounds).
__device__ __forceinline__ uint32_t scale_factors(const PassOp *ops, const uint32_t *tpos, uint32_t base,
                                                  int64_t trow) {
  return uint32_t(__ldg(ops[0].table + trow * ops[0].tab_stride + (base | tpos[threadIdx.x & 31])));
}

// gdst (optional): the tile's blocks in the BS output buffer -- the scaled
// blocks then also leave straight from the registers (no later pass over the
// tile in shared memory to store them).
template <int R, uint32_t POLY>
__device__ __forceinline__ void scale_phase(const PassOp *ops, int nops, uint4 *smem,
                                            const uint32_t *tpos, uint32_t base, int TP,
                                            int64_t trow, const Mul<R, POLY> &mm, uint4 *gdst = nullptr,
                                            uint32_t fl_early = 0u, bool have_early = false) {
  constexpr int U4 = Blk<R>::U4;
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  if (nops == 1 && TP == 32) {
    // One scaling of a full tile: every warp reads the tile's 32 factors in
    // ONE coalesced load (lane l: position l) instead of one dependent global
    // load per position, and the positions with a nonzero factor -- the only
    // ones that cost a multiply: the decode's Pi-bar is zero on the erased
    // positions and Pi'^-1 on the survivors -- are dealt round-robin to the
    // warps by their rank, so every warp multiplies within one position of
    // the same count and the barrier behind the phase waits for nobody.
    // (the caller may have requested the factors earlier: scale_factors)
    const uint32_t fl = have_early ? fl_early : scale_factors(ops, tpos, base, trow);
    const uint32_t nz = __ballot_sync(0xffffffffu, fl != 0u);
    const uint32_t lt = (1u << lane) - 1u;
    // rank of this lane's position among the nonzero ones, then among the zero ones
    const int rk = fl != 0u ? __popc(nz & lt) : __popc(nz) + __popc(~nz & lt);
    const bool mine = (rk & (NWARP - 1)) == warp;
    const uint32_t mine_nz = __ballot_sync(0xffffffffu, mine && fl != 0u);
    const uint32_t mine_z = __ballot_sync(0xffffffffu, mine && fl == 0u);
    for (uint32_t m = mine_nz; m; m &= m - 1u) {
      const int q = __ffs(int(m)) - 1;
      const uint32_t f = __shfl_sync(0xffffffffu, fl, q);
      uint32_t v[R], acc[R];
      Blk<R>::load(smem + q * U4, lane, v);
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0u;
      mm.acc(acc, v, f);
      Blk<R>::store(smem + q * U4, lane, acc);
      if (gdst) Blk<R>::store_g(gdst + size_t(base | tpos[q]) * U4, lane, acc);
    }
    for (uint32_t m = mine_z; m; m &= m - 1u) {  // zero factors: the block is zero
      const int q = __ffs(int(m)) - 1;
      uint32_t z[R];
#pragma unroll
      for (int b = 0; b < R; ++b) z[b] = 0u;
      Blk<R>::store(smem + q * U4, lane, z);
      if (gdst) Blk<R>::store_g(gdst + size_t(base | tpos[q]) * U4, lane, z);
    }
    return;
  }
  for (int q = warp; q < TP; q += NWARP) {
    uint32_t v[R];
    Blk<R>::load(smem + q * U4, lane, v);
    for (int o = 0; o < nops; ++o) {
      const uint32_t f = __shfl_sync(
          0xffffffffu, uint32_t(__ldg(ops[o].table + trow * ops[o].tab_stride + (base | tpos[q]))), 0);
      uint32_t acc[R];
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0u;
      if (f) mm.acc(acc, v, f);
#pragma unroll
      for (int b = 0; b < R; ++b) v[b] = acc[b];
    }
    Blk<R>::store(smem + q * U4, lane, v);
    if (gdst) Blk<R>::store_g(gdst + size_t(base | tpos[q]) * U4, lane, v);
  }
}

// One LCH butterfly on a pair of bit-sliced positions (u at the block's lower
// half): forward transform.py:126-133 (u' = u + f v, v' = u' + v) or inverse
// transform.py:165-169 (v' = u + v, u' = u + f v').  f is warp-uniform.
template <int R, uint32_t POLY>
__device__ __forceinline__ void butterfly(uint32_t (&u)[R], uint32_t (&v)[R], uint32_t f, int kind,
                                          const Mul<R, POLY> &mm) {
  using F = GF<R, 16u>;  // xor_into only (polynomial-independent)
  if (kind != OP_FWD) F::xor_into(v, u);
  // zero factors (block 0 of every level at shift 0, transform.py:154-161)
  // are a warp-uniform skip
  if (f) mm.acc(u, v, f);
  if (kind != OP_INV) F::xor_into(v, u);
}

// Two butterflies sharing one factor (pairs (u0, v0) and (u1, v1)).
template <int R, uint32_t POLY>
__device__ __forceinline__ void butterfly2(uint32_t (&u0)[R], uint32_t (&v0)[R], uint32_t (&u1)[R],
                                           uint32_t (&v1)[R], uint32_t f, int kind, const Mul<R, POLY> &mm) {
  using F = GF<R, 16u>;
  if (kind != OP_FWD) {
    F::xor_into(v0, u0);
    F::xor_into(v1, u1);
  }
  if (f) mm.acc2(u0, v0, u1, v1, f);
  if (kind != OP_INV) {
    F::xor_into(v0, u0);
    F::xor_into(v1, u1);
  }
}

// Butterfly factors of one tile (transform.py:112,123: w_hat[i][c >> (i+1)] ^
// W^_i(shift), with c the u position): entry (op, q_u) of the tile's table.
// Each thread owns <= 2 entries; fetch() issues the global loads, put()
// writes them to shared memory later so their latency hides behind compute.
struct FactorLoader {
  static constexpr int PER = (MAXOPS * (1 << (TPB_MAX - 1)) + NT - 1) / NT;
  uint32_t v[PER];
  int slot[PER];
  __device__ __forceinline__ void fetch(const PassParams &p, const uint32_t *tpos, uint32_t base) {
    const int lh = p.tpb - 1 < 0 ? 0 : p.tpb - 1;  // log2 of the pairs per op
    const int n = p.nops << lh;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * NT;
      slot[k] = -1;
      if (p.tpb > 0 && e < n) {
        const int o = e >> lh, pp = e & ((1 << lh) - 1);
        const PassOp &op = p.ops[o];
        const int m = op.mloc;
        const int qu = ((pp >> m) << (m + 1)) | (pp & ((1 << m) - 1));
        const int lvl = op.level;
        v[k] = op.kind == OP_INVFWD
                   ? op.hs
                   : uint32_t(__ldg(p.w_hat + p.w_hat_off[lvl] + ((base | tpos[qu]) >> (lvl + 1)))) ^ op.hs;
        if (PDBG(256)) v[k] = uint32_t(p.dbg) >> 16;  // experiment: one forced factor
        slot[k] = o * (1 << TPB_MAX) + qu;
      }
    }
  }
  __device__ __forceinline__ void put(uint32_t *fac) const {
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (slot[k] >= 0) fac[slot[k]] = v[k];
  }
};

// Instances by the features a pass needs (V bit 0: raw input, bit 1: raw
// output, bit 2: per-position scalings / gather epilogue, bit 3: every round
// is a straight-line one, so the general round path is left out); code a pass cannot reach is
// compiled out, which keeps the hot loop's code footprint small (the pure
// butterfly passes run 5-7 % faster in the V = 0 instance).
template <int R, uint32_t POLY, int V>
// 2 CTAs per SM (128 registers: 4 positions x 16 planes + the multiply's
// chain).  Measured: 3 CTAs at 80 registers made the pure butterfly passes
// 24-28 % slower (V = 24: 165 -> 204 us), spills in the others.
#ifndef LCH_PASS_MINB
#define LCH_PASS_MINB(V) 2
#endif
__global__ void __launch_bounds__(NT, LCH_PASS_MINB(V)) pass_kernel(const __grid_constant__ PassParams p) {
  constexpr bool RIN = V & 1, ROUT = V & 2, EXTRA = V & 4, SHAPED = V & 8;
  // bit 6: scalings before the rounds only; bit 8: after them (and the gather epilogue) only
  constexpr bool PRE_OK = EXTRA && !(V & 256), POST_OK = EXTRA && !(V & 64);
  // bits 4-5: every round follows one pattern -- 1: inverse (op along m0 with
  // distinct factors, op along m1 shared), 2: forward (m0 shared, m1 distinct)
  constexpr int PAT = (V >> 4) & 3;
  constexpr bool ROWONLY = V & 128;  // raw I/O in row layout only (no packet paths)
  // bit 9: raw row-major output straight from the last round's registers
  // (launch_pass picks it when every tile qualifies, see store_rows_from_regs)
  constexpr bool RREG = (V & 512) && R == 16;
  // bit 10: TMA-staged raw input tiles go straight into the first round's
  // registers (raw_tma_tile_to_regs; launch_pass checks the conditions)
  constexpr bool FUSEIN = (V & 1024) && R == 16;
  constexpr int U4 = Blk<R>::U4;
  // 128-byte aligned: TMA tensor copies land here
  extern __shared__ __align__(128) uint4 smem[];
  uint4 *const bsm = smem + bs_offset_u4<R>();
  __shared__ uint32_t tpos[1 << TPB_MAX];
  __shared__ uint32_t fac[2][MAXOPS * (1 << TPB_MAX)];
  __shared__ __align__(8) uint64_t bar, bar_m;
  // (raw-output instances) (x << 16) mod p / (x << 24) mod p for the
  // per-codeword division by Pi' (gf16_mul_t): two lookups instead of folds
  __shared__ uint32_t red16[(V & 2) && R == 16 ? 384 : 1];
  unsigned phase = 0, phase_m = 0;
  const Mul<R, POLY> mm(__shfl_sync(0xffffffffu, p.taps, 0));
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index through a shuffle: provably warp-uniform for the compiler, so
  // the butterfly factors and their digit tests live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int TP = 1 << p.tpb;
  const int ntile = 1 << p.lgnt;
  const int total = ntile * p.ngroups;
  int tl = blockIdx.x;
  if (tl >= total) return;
  if (tid < TP) {
    uint32_t o = 0;
    for (int m = 0; m < p.tpb; ++m) o |= ((uint32_t(tid) >> m) & 1u) << p.gbit[m];
    tpos[tid] = o;
  }
  // tile base: the tile index spread over the non-tile bits (ascending), i.e.
  // a zero inserted at every tile bit
  auto base_of = [&](int lin) {
    uint32_t b = uint32_t(lin) & uint32_t(ntile - 1);
#pragma unroll
    for (int m = 0; m < TPB_MAX; ++m)
      if (m < p.tpb) {
        const uint32_t lm = p.ins_mask[m];
        b = ((b & ~lm) << 1) | (b & lm);
      }
    return b;
  };
  int g = tl >> p.lgnt;
  uint32_t base = base_of(tl);
  if constexpr ((V & 2) && R == 16) {
    if (POLY == 0x1100Bu)
      for (int i = tid; i < 384; i += NT) red16[i] = gf16_fold(i < 256 ? uint32_t(i) << 16 : uint32_t(i - 256) << 24);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar_m, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // tile blocks (one contiguous buffer)
  auto blk = [&](int q) -> uint4 * { return bsm + q * U4; };
  issue_tile<R, !RIN, ROWONLY>(p, smem, tpos, g, base, TP, &bar);
  int fb = 0;  // factor-table buffer of the current tile
  {
    FactorLoader fl;
    fl.fetch(p, tpos, base);
    fl.put(fac[0]);
  }
  if (!RIN || p.in_mode == IO_BS || p.raw_tma || p.raw_bulk) {
    mbar_wait(&bar, phase);
    phase ^= 1u;
  }
  __syncthreads();

  // The last round keeps its data in registers and stores it straight to the
  // BS output, so the next tile's loads can stream into shared memory while
  // it computes.
  const bool reg_path = p.nrounds > 0 && (!POST_OK || (p.npost == 0 && !p.gt_out)) &&
                        (!ROUT || p.out_mode == IO_BS || RREG);

  for (;;) {
    const int next = tl + int(gridDim.x);
    const bool has_next = next < total;
    if (ROUT && R == 16 && p.merge_tma && threadIdx.x == 0) {
      // survivors of position chunks 0-1 of this tile, for the output merge
      uint4 *dst = smem + stage_offset_u4<R>();
      fence_proxy_async();
      mbar_expect_tx(&bar_m, 32u * 1024u);
      const int c0 = int(int64_t(base) >> 3);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int rb = 0; rb < 4; ++rb)
          tma_load_3d(dst + c * GROUP + rb * 256, &p.tm_merge, 0, c0 + c, g * GROUP + rb * 256, &bar_m);
    }
    const int64_t trow = p.pkt ? (int64_t(g) * GROUP) / p.pkt : 0;
    const bool pre_early = PRE_OK && p.npre == 1 && TP == 32, post_early = POST_OK && p.npost == 1 && TP == 32;
    uint32_t fl_pre = 0u, fl_post = 0u;
    if (pre_early) fl_pre = scale_factors(p.pre, tpos, base, trow);
    if (RIN && p.in_mode == IO_RAW && !FUSEIN) {
      if (!(PDBG(128))) {
        if (R == 16 && p.raw_tma)
          finish_tile_raw_tma<R>(smem);
        else if (R == 16 && p.raw_bulk)
          finish_tile_raw_bulk<R>(smem, int64_t(base) >= p.raw_in.pos_lo && int64_t(base) < p.raw_in.pos_hi);
        else
          finish_tile_raw<R>(smem, TP);
      }
      __syncthreads();
    }
    if (PRE_OK && p.npre) {
      scale_phase<R, POLY>(p.pre, p.npre, bsm, tpos, base, TP, trow, mm, nullptr, fl_pre, pre_early);
      __syncthreads();
    }
    if (post_early) fl_post = scale_factors(p.post, tpos, base, trow);
    for (int rd = 0; rd < p.nrounds; ++rd) {
      const PassRound &rr = p.rounds[rd];
      const bool last_reg = reg_path && rd == p.nrounds - 1;
      const int M0 = 1 << rr.m0;
      const bool has1 = rr.m1 >= 0;
      const int M1 = has1 ? (1 << rr.m1) : 0;
      const bool active = warp < (1 << rr.nw);
      const int q0 = rr.q0w[warp];
      uint32_t a0[R], a1[R], a2[R], a3[R];
      if (FUSEIN && rd == 0) {
        if constexpr (FUSEIN) raw_tma_tile_to_regs<R>(smem, a0, a1, a2, a3);
      } else if (active && !(PDBG(32))) {
        Blk<R>::load(blk(q0), lane, a0);
        Blk<R>::load(blk(q0 | M0), lane, a1);
        if (has1) {
          Blk<R>::load(blk(q0 | M1), lane, a2);
          Blk<R>::load(blk(q0 | M0 | M1), lane, a3);
        }
      }
      FactorLoader nfl;
      if (last_reg) {
        __syncthreads();
        if (has_next) {
          const uint32_t nb = base_of(next);
          issue_tile<R, !RIN, ROWONLY>(p, smem, tpos, next >> p.lgnt, nb, TP, &bar);
          if (!(PDBG(64))) nfl.fetch(p, tpos, nb);
        }
      }
      if (active && (SHAPED || rr.shape != 0) && !(PDBG(2))) {
        // straight-line rounds: [op along m0] or [op along m0, op along m1];
        // ops whose pairs share the factor run as one two-vector multiply
        const uint32_t *ft = fac[fb] + rr.op_begin * (1 << TPB_MAX);
        if constexpr (PAT == 3) {
          // pattern 3 (launch_pass rewrites the rounds): a round is the op with
          // distinct factors along m0 (shape 1, 2) and/or the op with a shared
          // factor along m1 (shape 2, 3), in either order (rev: m1 first), so
          // one copy of each multiply body serves inverse, forward and mixed
          // passes
          const bool has_d = rr.shape != 3, has_s = rr.shape != 1;
          const int kd = p.ops[rr.op_begin].kind, ks = p.ops[rr.op_begin + (has_d ? 1 : 0)].kind;
          const uint32_t *fs = ft + (has_d ? (1 << TPB_MAX) : 0);
#pragma unroll 1
          for (int step = 0; step < 2; ++step) {
            if ((step == 0) == (rr.rev != 0)) {
              if (has_s) {
                const uint32_t f = __shfl_sync(0xffffffffu, fs[q0], 0);
                butterfly2<R, POLY>(a0, a2, a1, a3, f, ks, mm);
              }
            } else if (has_d) {
              const uint32_t f1 = __shfl_sync(0xffffffffu, ft[q0], 0);
              const uint32_t f2 = __shfl_sync(0xffffffffu, ft[q0 | M1], 0);
              butterfly<R, POLY>(a0, a1, f1, kd, mm);
              butterfly<R, POLY>(a2, a3, f2, kd, mm);
            }
          }
        } else {
        const PassOp &oa = p.ops[rr.op_begin];
        const uint32_t fa = __shfl_sync(0xffffffffu, ft[q0], 0);
        const int inv_a = PAT == 2 ? int(OP_FWD) : oa.kind;
        if (PAT ? PAT == 2 : oa.shared) {
          butterfly2<R, POLY>(a0, a1, a2, a3, fa, inv_a, mm);
        } else {
          const uint32_t fa2 = __shfl_sync(0xffffffffu, ft[q0 | M1], 0);
          butterfly<R, POLY>(a0, a1, fa, inv_a, mm);
          butterfly<R, POLY>(a2, a3, fa2, inv_a, mm);
        }
        if (rr.shape == 2) {
          const uint32_t *fu = ft + (1 << TPB_MAX);
          const PassOp &ob = p.ops[rr.op_begin + 1];
          const uint32_t fb1 = __shfl_sync(0xffffffffu, fu[q0], 0);
          const int inv_b = PAT == 2 ? int(OP_FWD) : ob.kind;
          if (PAT ? PAT == 1 : ob.shared) {
            butterfly2<R, POLY>(a0, a2, a1, a3, fb1, inv_b, mm);
          } else {
            const uint32_t fb2 = __shfl_sync(0xffffffffu, fu[q0 | M0], 0);
            butterfly<R, POLY>(a0, a2, fb1, inv_b, mm);
            butterfly<R, POLY>(a1, a3, fb2, inv_b, mm);
          }
        }
        }
        if (!last_reg && !(PDBG(32))) {
          Blk<R>::store(blk(q0), lane, a0);
          Blk<R>::store(blk(q0 | M0), lane, a1);
          Blk<R>::store(blk(q0 | M1), lane, a2);
          Blk<R>::store(blk(q0 | M0 | M1), lane, a3);
        }
      } else if (!SHAPED && active) {
        // A round's ops are [along m0]* [along m1]*.  Along m0 the pairs are
        // (a0,a1), (a2,a3); at the first m1 op a1 and a2 swap once, so the same
        // two inlined butterflies (one multiply body each) serve both bits.
        bool sw = false;
        for (int o = rr.op_begin; o < ((PDBG(2)) ? rr.op_begin : rr.op_end); ++o) {
          const PassOp &op = p.ops[o];
          const int inv = op.kind;
          if (op.m == 1 && !sw) {
#pragma unroll
            for (int b = 0; b < R; ++b) {
              const uint32_t x = a1[b];
              a1[b] = a2[b];
              a2[b] = x;
            }
            sw = true;
          }
          const uint32_t *ft = fac[fb] + o * (1 << TPB_MAX);
          const uint32_t f1 = __shfl_sync(0xffffffffu, ft[q0], 0);
          butterfly<R, POLY>(a0, a1, f1, inv, mm);
          if (has1) {
            const uint32_t f2 = __shfl_sync(0xffffffffu, ft[sw ? (q0 | M0) : (q0 | M1)], 0);
            butterfly<R, POLY>(a2, a3, f2, inv, mm);
          }
        }
        if (sw) {
#pragma unroll
          for (int b = 0; b < R; ++b) {
            const uint32_t x = a1[b];
            a1[b] = a2[b];
            a2[b] = x;
          }
        }
        if (!last_reg) {
          Blk<R>::store(blk(q0), lane, a0);
          Blk<R>::store(blk(q0 | M0), lane, a1);
          if (has1) {
            Blk<R>::store(blk(q0 | M1), lane, a2);
            Blk<R>::store(blk(q0 | M0 | M1), lane, a3);
          }
        }
      }
      if (last_reg) {
        // The tile leaves straight from registers: coalesced 512-byte
        // streaming stores per chunk (no staging, no wait on earlier stores),
        // overlapping the next tile's rounds.
        uint4 *dst = p.bs_out + ((size_t(g) << p.lgH) * U4);
        if constexpr (RREG) {
          // forward pattern, last round over bits (1, 0): a0, a2, a1, a3 are
          // the positions q0, q0 + 1, q0 + 2, q0 + 3
          store_rows_from_regs(p, smem, g, base, q0, a0, a2, a1, a3);
        } else
        if (active && !(PDBG(5))) {
          Blk<R>::store_g(dst + size_t(base | tpos[q0]) * U4, lane, a0);
          Blk<R>::store_g(dst + size_t(base | tpos[q0 | M0]) * U4, lane, a1);
          if (has1) {
            Blk<R>::store_g(dst + size_t(base | tpos[q0 | M1]) * U4, lane, a2);
            Blk<R>::store_g(dst + size_t(base | tpos[q0 | M0 | M1]) * U4, lane, a3);
          }
        }
        if (has_next && !(PDBG(64))) nfl.put(fac[fb ^ 1]);
      }
      if (!last_reg) __syncthreads();
    }
    if (!reg_path) {
      // BS output of a scaled tile leaves from the scaling's registers
      const bool bs_from_scale = POST_OK && p.npost && (!ROUT || p.out_mode == IO_BS) && !(PDBG(5));
      if (POST_OK && p.npost) {
        scale_phase<R, POLY>(p.post, p.npost, bsm, tpos, base, TP, trow, mm,
                             bs_from_scale ? p.bs_out + ((size_t(g) << p.lgH) * U4) : nullptr, fl_post, post_early);
        __syncthreads();
      }
      if (POST_OK && p.gt_out) {
        // derivative gather over the tile bits (derivative.py:60-70), for the
        // output positions below 2^gt_lgH
        uint4 *gdst = p.gt_out + ((size_t(g) << p.gt_lgH) * U4);
        for (int q = warp; q < TP; q += NWARP) {
          const uint32_t pos = base | tpos[q];
          if (pos >= (1u << p.gt_lgH)) continue;
          uint32_t acc[R];
#pragma unroll
          for (int b = 0; b < R; ++b) acc[b] = 0u;
          for (int m = 0; m < p.tpb; ++m) {
            if ((q >> m) & 1) continue;
            uint32_t x[R];
            Blk<R>::load(bsm + (q | (1 << m)) * U4, lane, x);
#pragma unroll
            for (int b = 0; b < R; ++b) acc[b] ^= x[b];
          }
          Blk<R>::store(gdst + size_t(pos) * U4, lane, acc);
        }
      }
      if (!ROUT || p.out_mode == IO_BS) {
        if (!bs_from_scale) store_tile_bs<R>(p, bsm, tpos, g, base, TP);
      } else {
        if (R == 16 && p.merge_tma) {
          mbar_wait(&bar_m, phase_m);
          phase_m ^= 1u;
        }
        store_tile_raw<R, ROWONLY>(p, smem, g, red16, base, TP);
      }
      __syncthreads();
      if (has_next) {
        const uint32_t nb = base_of(next);
        issue_tile<R, !RIN, ROWONLY>(p, smem, tpos, next >> p.lgnt, nb, TP, &bar);
        FactorLoader fl;
        if (!(PDBG(64))) {
          fl.fetch(p, tpos, nb);
          fl.put(fac[fb ^ 1]);
        }
      }
    }
    if (!has_next) {
      if (lane == 0) tma_store_wait_all();
      break;
    }
    if (!RIN || p.in_mode == IO_BS || p.raw_tma || p.raw_bulk) {
      mbar_wait(&bar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    fb ^= 1;
    tl = next;
    g = tl >> p.lgnt;
    base = base_of(tl);
  }
}

// The dynamic shared-memory opt-in is a per-device function attribute: set it
// once per (kernel, device) — a process may drive several GPUs.
template <class K>
static cudaError_t smem_optin(K *kernel, int bytes, std::atomic<uint64_t> &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

static int sm_count() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) {
    cudaGetLastError();
    nsm = 148;
  }
  return nsm;
}


// One pass_kernel instance and its launch.  The instances are compiled in
// separate translation units (this file built with -DLCH_PASS_TU=V, in
// parallel), the main unit only declares them.
template <int R, uint32_t POLY, int V>
cudaError_t launch_pass_v(const PassParams &p, unsigned ctas, size_t smem, cudaStream_t s) {
  static std::atomic<uint64_t> done{0};
  cudaError_t e = smem_optin(pass_kernel<R, POLY, V>, int(pass_smem_bytes(R, TPB_MAX, true)), done);
  if (e != cudaSuccess) return e;
  // persistent CTAs: as many as fit on the device (2 or 3 per SM)
  static std::atomic<int> occ_cache[2] = {{0}, {0}};
  std::atomic<int> &oc = occ_cache[smem > pass_smem_bytes(R, TPB_MAX, false) ? 1 : 0];
  int occ = oc.load(std::memory_order_relaxed);
  if (occ <= 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_kernel<R, POLY, V>, NT, smem) != cudaSuccess ||
        occ <= 0) {
      cudaGetLastError();
      occ = 2;
    }
    oc.store(occ, std::memory_order_relaxed);
  }
  const unsigned maxc = unsigned(occ) * unsigned(sm_count());
  pass_kernel<R, POLY, V><<<std::min(ctas, maxc), NT, smem, s>>>(p);
  return cudaGetLastError();
}

#ifdef LCH_PASS_TU
#if LCH_PASS_TU == 0 || LCH_PASS_TU == 7
template cudaError_t launch_pass_v<8, 0x11Du, LCH_PASS_TU>(const PassParams &, unsigned, size_t, cudaStream_t);
#endif
#if LCH_PASS_TU == 7  // any other primitive polynomial (taps at run time)
template cudaError_t launch_pass_v<8, 0u, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
template cudaError_t launch_pass_v<16, 0u, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
#endif
template cudaError_t launch_pass_v<16, 0x1100Bu, LCH_PASS_TU>(const PassParams &, unsigned, size_t,
                                                                cudaStream_t);
#else  // the main unit: every kernel but the pass instances
extern template cudaError_t launch_pass_v<8, 0u, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0u, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<8, 0x11Du, 0>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<8, 0x11Du, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 0>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 1>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 2>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 4>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 5>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 7>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 8>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 9>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 10>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 12>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 24>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 25>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 28>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 29>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 46>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 153>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 157>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 170>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 174>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 221>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 108>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 284>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 430>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 13>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 44>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 40>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 42>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 56>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 682>(const PassParams &, unsigned, size_t, cudaStream_t);
extern template cudaError_t launch_pass_v<16, 0x1100Bu, 1177>(const PassParams &, unsigned, size_t, cudaStream_t);

constexpr int GNT = 512;  // gather threads per CTA

// Tile bits are sorted, so the tile positions below 2^lgH_out (the outputs)
// are exactly q < 2^nlow with nlow = #tile bits below lgH_out (base < 2^lgH_out).
// Only the y values over the summed tile bits are staged in shared memory
// (each is read by up to nbits outputs); T_in and the special bit's partner
// y_(j | 2^special) are read once per output straight from global memory.
// A CTA covers one tile for 2^lwpc consecutive lane-words (small tiles take
// more words so every CTA moves a useful amount of data).
template <int R, uint32_t POLY>
__global__ void __launch_bounds__(GNT, 2) gather_kernel(const __grid_constant__ GatherParams p) {
  constexpr int CH = R / 4;  // 16-byte chunks of one lane-word
  constexpr int U4 = Blk<R>::U4;
  extern __shared__ uint4 smem[];
  const int tid = threadIdx.x;
  const int np = 1 << p.nbits;
  int nlow = 0;
  while (nlow < p.nbits && p.bits[nlow] < p.lgH_out) ++nlow;
  const int nout = 1 << nlow;
  const int lw = p.lwpc, WPC = 1 << lw;
  const int wblocks = 32 >> lw;
  // blockIdx.x enumerates (group, lane-word block) fastest, so the CTAs that
  // read the different 64-byte lane-word slices of the same 2 KB position
  // blocks are scheduled together (DRAM row locality)
  const int g = blockIdx.x / wblocks, w0 = (blockIdx.x - g * wblocks) * WPC;
  uint4 *ytile = smem;
  const uint32_t t = blockIdx.y;
  uint32_t base = 0;
  for (int i = 0; i < p.nnb; ++i) base |= ((t >> i) & 1u) << p.nbit[i];
  const uint32_t hout = 1u << p.lgH_out;
  if (base >= hout) return;  // every position of the tile is >= hout
  auto pos_of = [&](int q) {
    uint32_t o = base;
    for (int m = 0; m < p.nbits; ++m) o |= ((uint32_t(q) >> m) & 1u) << p.bits[m];
    return o;
  };
  // e = q * WPC + word offset; the chunk swizzle keeps quarter-warps conflict-free
  auto slot = [](int e, int c) { return e * CH + (c ^ ((e >> 1) & (CH - 1))); };
  const uint4 *src = p.y + ((size_t(g) << p.lgH_in) * U4);
  for (int idx = tid; idx < (np << lw) * CH; idx += GNT) {
    const int e = idx / CH, c = idx - e * CH;
    const int q = e >> lw, wl = e & (WPC - 1);
    cp_async16(ytile + slot(e, c), src + size_t(pos_of(q)) * U4 + Blk<R>::chunk(w0 + wl, c));
  }
  cp_async_wait_all();
  __syncthreads();
  auto ld = [&](const uint4 *tile, int e, uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint4 x = tile[slot(e, c)];
      v[4 * c + 0] = x.x;
      v[4 * c + 1] = x.y;
      v[4 * c + 2] = x.z;
      v[4 * c + 3] = x.w;
    }
  };
  auto ldg = [&](const uint4 *blk, int w, uint32_t (&v)[R]) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint4 x = __ldcs(blk + Blk<R>::chunk(w, c));
      v[4 * c + 0] = x.x;
      v[4 * c + 1] = x.y;
      v[4 * c + 2] = x.z;
      v[4 * c + 3] = x.w;
    }
  };
  const uint4 *tin = p.t_in ? p.t_in + ((size_t(g) << p.lgH_out) * U4) : nullptr;
  uint4 *tout = p.t_out + ((size_t(g) << p.lgH_out) * U4);
  for (int e = tid; e < (nout << lw); e += GNT) {
    const int q = e >> lw, wl = e & (WPC - 1);
    const uint32_t pos = pos_of(q);
    uint32_t acc[R];
    if (tin) {
      ldg(tin + size_t(pos) * U4, w0 + wl, acc);
    } else {
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0u;
    }
    for (int m = 0; m < p.nbits; ++m) {
      if ((q >> m) & 1) continue;
      uint32_t x[R];
      ld(ytile, e | (1 << (m + lw)), x);
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] ^= x[b];
    }
    for (int d = 0; d < p.ndirect; ++d) {  // non-tile summed bits: CTA-uniform test
      if ((pos >> p.dbits[d]) & 1u) continue;
      uint32_t x[R];
      ldg(src + size_t(pos | (1u << p.dbits[d])) * U4, w0 + wl, x);
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] ^= x[b];
    }
    if (p.sb >= 0) {  // the output has the special (top) bit clear
      uint32_t x[R], z[R], cz[R];
      ldg(src + size_t(pos | (1u << p.sb)) * U4, w0 + wl, z);
      ld(ytile, e, x);
#pragma unroll
      for (int b = 0; b < R; ++b) z[b] ^= x[b];
      Mul<R, POLY>(p.taps).mul(cz, z, p.c);  // c is a kernel constant: uniform
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] ^= cz[b];
    }
#pragma unroll
    for (int c = 0; c < CH; ++c)
      tout[size_t(pos) * U4 + Blk<R>::chunk(w0 + wl, c)] =
          make_uint4(acc[4 * c + 0], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
  }
}

size_t gather_smem_bytes(int R, const GatherParams &p) {
  return ((size_t(1) << p.nbits) * R * 4) << p.lwpc;
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
  if (p.phi) {
    // x = log of the locator value at pos (Pi_bar if surviving, Pi' if erased)
    const bool erased = (p.bits_e[size_t(vec) * words + (pos >> 5)] >> (pos & 31)) & 1u;
    const uint16_t r = p.rx[size_t(vec) * p.rx_stride + pos];
    p.phi[size_t(vec) * p.rx_stride + pos] =
        (erased || r == 0) ? uint16_t(0) : p.exp[(uint32_t(p.log[r]) + x) % p.mod];
    if (pos < p.k)
      p.pinv_log[size_t(vec) * p.k + pos] = erased ? uint16_t((p.mod - x) % p.mod) : uint16_t(0);
  } else if (p.exp) {
    const uint16_t val = p.exp[x];
    if (p.loc_out) p.loc_out[idx] = val;
    if (p.log_out) p.log_out[idx] = uint16_t(x);
  } else {
    p.data[idx] = x;
  }
}

// Whole erasure locator of one pattern per CTA for r = 16 (walsh.py:97-114):
// R^w = FWHT(FWHT(indicator) * FWHT(log)) mod 2^16 - 1, the 2^16 residues
// held in shared memory as uint16 (ones' complement: 0xFFFF == 0 until the
// final normalisation).  The Walsh-Hadamard stages commute, so the two
// transforms run as rounds over 4-bit groups G0, G1, G2, G3 | G3, G2, G1, G0
// with the pointwise product fused into the G3 round (7 shared-memory round
// trips, 16 values per thread slot in registers).  The first round reads the
// indicator straight from the bitmask; the last writes the epilogue (locator
// values / logs, or phi = rx * Pi_bar and -log Pi' for the decode).
constexpr int LOC_NT = 1024;
constexpr int LOC_SMEM = 65536 * 2 + 384 * 4;  // residues + gf16_red tables

// x mod (2^16 - 1) folded once: (x & 0xFFFF) + (x >> 16) = x - 65535 * (x >> 16)
// (shift + IMAD: keeps half of the work off the integer ALU pipe)
__device__ __forceinline__ uint32_t fold16(uint32_t x) { return x - 65535u * (x >> 16); }

// 16-point WHT mod 2^16 - 1 with lazy reduction: inputs <= m, stage h adds
// m * 2^h before subtracting (a - b + m 2^h >= 0), so values stay below
// m * 2^(h+1) < 2^21; two folds bring them back to <= m (0xFFFF == 0).
__device__ __forceinline__ void wht16(uint32_t (&v)[16]) {
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (!(e & (1 << h))) {
        const uint32_t a = v[e], b = v[e | (1 << h)];
        v[e] = a + b;
        v[e | (1 << h)] = a - b + (0xFFFFu << h);
      }
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = fold16(fold16(v[e]));
}

// Shared-memory layout of the 2^16 residues: uint16 pairs (positions 2w,
// 2w + 1) in 32-bit words, word w stored at lsw(w) = w ^ (((w >> 7) & 3) << 3)
// so that the rounds over position bits 4-7 (whose lanes step the word index
// by 2^7) spread over all banks; the swizzle moves whole 32-byte chunks, so
// the 16-position slot vectors of the first/last round stay contiguous.
__device__ __forceinline__ uint32_t lsw(uint32_t w) { return w ^ (((w >> 7) & 3u) << 3); }

__global__ void __launch_bounds__(LOC_NT) locator16_kernel(const __grid_constant__ FwhtParams p) {
  extern __shared__ uint16_t sv[];  // 2^16 residues, then the gf16_red tables
  uint32_t *const sw = reinterpret_cast<uint32_t *>(sv);
  uint32_t *const red = sw + 32768;
  constexpr uint32_t M = 0xFFFFu;
  const int64_t vec = blockIdx.x;
  const uint32_t *bits = p.bits + vec * 2048;
  const int tid = threadIdx.x;
  if (tid < 384) red[tid] = gf16_fold(tid < 256 ? uint32_t(tid) << 16 : uint32_t(tid - 256) << 24);
  // G0 of the first transform, from the bitmask (16 bits per slot), stored as
  // two 16-byte vectors per slot
  for (int slot = tid; slot < 4096; slot += LOC_NT) {
    const uint32_t w = (bits[slot >> 1] >> (16 * (slot & 1))) & 0xFFFFu;
    uint32_t v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = (w >> e) & 1u;
    wht16(v);
    uint4 *dst = reinterpret_cast<uint4 *>(sw + lsw(uint32_t(slot) << 3));
    dst[0] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
    dst[1] = make_uint4(v[8] | (v[9] << 16), v[10] | (v[11] << 16), v[12] | (v[13] << 16),
                        v[14] | (v[15] << 16));
  }
  __syncthreads();
  // A round over position bits b0..b0+3 (b0 >= 1): a thread takes the two
  // slots that differ in position bit 0 together, one 32-bit word per pair.
  auto round = [&](int b0, bool mul) {
    const int lb = b0 - 1;  // word-index bits below the round's bits
    for (int sp = tid; sp < 2048; sp += LOC_NT) {
      const uint32_t lo = uint32_t(sp) & ((1u << lb) - 1u), hi = uint32_t(sp) >> lb;
      const uint32_t w0 = (hi << (lb + 4)) | lo;
      uint32_t va[16], vb[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t x = sw[lsw(w0 | (uint32_t(e) << lb))];
        va[e] = x & 0xFFFFu;
        vb[e] = x >> 16;
      }
      wht16(va);
      wht16(vb);
      if (mul) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint2 m = __ldg(reinterpret_cast<const uint2 *>(p.post_mul) + (w0 | (uint32_t(e) << lb)));
          va[e] = fold16(fold16(va[e] * m.x));
          vb[e] = fold16(fold16(vb[e] * m.y));
        }
        wht16(va);
        wht16(vb);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) sw[lsw(w0 | (uint32_t(e) << lb))] = va[e] | (vb[e] << 16);
    }
    __syncthreads();
  };
  round(4, false);
  round(8, false);
  round(12, true);  // end of the first transform, product, start of the second
  round(8, false);
  round(4, false);
  // G0 of the second transform + epilogue
  const uint32_t *bits_e = p.bits_e ? p.bits_e + vec * 2048 : nullptr;
  for (int slot = tid; slot < 4096; slot += LOC_NT) {
    uint32_t v[16];
    const uint4 *src = reinterpret_cast<const uint4 *>(sw + lsw(uint32_t(slot) << 3));
    const uint4 x0 = src[0], x1 = src[1];
    const uint32_t w8[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = (w8[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
    wht16(v);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = fold16(v[e]) == M ? 0u : fold16(v[e]);  // normalise
    const uint32_t j0 = uint32_t(slot) << 4;
    if (p.phi) {
      const uint32_t er = (bits_e[slot >> 1] >> (16 * (slot & 1))) & 0xFFFFu;
      const uint4 *rxv = reinterpret_cast<const uint4 *>(p.rx + vec * p.rx_stride + j0);
      const uint4 r0 = __ldcs(rxv), r1 = __ldcs(rxv + 1);
      const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      // one independent exp gather per position: Pi-bar = alpha^v on survivors
      // (phi = rx * Pi-bar by the table-free multiply), 1 / Pi' = alpha^-v on
      // erasures (stored as values for the output epilogue)
      uint32_t ex[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const bool erased = (er >> e) & 1u;
        ex[e] = __ldg(p.exp + (erased ? (v[e] ? M - v[e] : 0u) : v[e]));
      }
      uint32_t o[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        uint32_t pair = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int e = 2 * h + q;
          const uint32_t r = (rw[h] >> (16 * q)) & 0xFFFFu;
          pair |= (((er >> e) & 1u) ? 0u : gf16_mul_t(r, ex[e], red)) << (16 * q);
        }
        o[h] = pair;
      }
      uint4 *dst = reinterpret_cast<uint4 *>(p.phi + vec * p.rx_stride + j0);
      __stcs(dst, make_uint4(o[0], o[1], o[2], o[3]));
      __stcs(dst + 1, make_uint4(o[4], o[5], o[6], o[7]));
      if (j0 < p.k) {
        uint16_t *pl = p.pinv_log + vec * p.k;
        uint32_t pv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pv[e] = ((er >> e) & 1u) ? ex[e] : 0u;
        if (j0 + 16 <= p.k && (p.k & 7) == 0) {
          uint4 *pd = reinterpret_cast<uint4 *>(pl + j0);
          pd[0] = make_uint4(pv[0] | (pv[1] << 16), pv[2] | (pv[3] << 16), pv[4] | (pv[5] << 16),
                             pv[6] | (pv[7] << 16));
          pd[1] = make_uint4(pv[8] | (pv[9] << 16), pv[10] | (pv[11] << 16), pv[12] | (pv[13] << 16),
                             pv[14] | (pv[15] << 16));
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (j0 + e < p.k) pl[j0 + e] = uint16_t(pv[e]);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const size_t idx = size_t(vec) * 65536 + j0 + e;
        if (p.log_out) p.log_out[idx] = uint16_t(v[e]);
        if (p.loc_out) p.loc_out[idx] = __ldg(p.exp + v[e]);
      }
    }
  }
}

cudaError_t launch_locator16(const FwhtParams &p, cudaStream_t s) {
  static std::atomic<uint64_t> done{0};
  cudaError_t e = smem_optin(locator16_kernel, LOC_SMEM, done);
  if (e != cudaSuccess) return e;
  locator16_kernel<<<unsigned(p.nvec), LOC_NT, LOC_SMEM, s>>>(p);
  return cudaGetLastError();
}

// decode rows from the locator logs, one row set per pattern (blockIdx.y):
// pi_row[j] = erased ? 0 : exp[x], pinv[j] = (erased && j < k) ? exp[(m - x) % m] : 0
// (rs.py:130-148)
__global__ void decode_rows_kernel(const uint16_t *logs, const uint32_t *bits,
                                   const uint16_t *exp, uint32_t m, uint32_t n, uint32_t k,
                                   uint16_t *pi_row, uint16_t *pinv) {
  const size_t pat = blockIdx.y, words = (n + 31) / 32;
  logs += pat * n;
  bits += pat * words;
  pi_row += pat * n;
  pinv += pat * k;
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

// packet-major: element index i -> (group, position, packet offset), the
// packet offset fastest so stores coalesce
__global__ void gen_packets_kernel(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                                   uint32_t mask, uint16_t *out, int64_t npos, int64_t pkt) {
  const int64_t total = batch * len;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sidx = i % pkt, rest = i / pkt;
    const int64_t j = rest % len, g = rest / len;
    const int64_t b = g * pkt + sidx;
    out[(g * npos + j) * pkt + sidx] = uint16_t(key_d(seed, cw0 + uint64_t(b), uint64_t(j)) & mask);
  }
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

size_t pass_smem_bytes(int R, int tpb, bool stage) {
  // [raw staging (R = 8 only)] [BS tile] [half-tile area: the decode merge's
  // prefetched survivors (raw-output passes only, R = 16)]
  (void)tpb;
  const size_t tile = (size_t(1) << TPB_MAX) * 8 * R * 16;
  const size_t pre = R == 16 ? 0 : size_t(GROUP) * (size_t(1) << TPB_MAX) * 2;
  return pre + tile + ((stage || R != 16) ? tile / 2 : 0);
}

template <int R, uint32_t POLY>
cudaError_t launch_pass(const PassParams &p, int ngroups, cudaStream_t s) {
  (void)0;
  int v = (p.in_mode == IO_RAW ? 1 : 0) | (p.out_mode == IO_RAW ? 2 : 0) |
          ((p.npre || p.npost || p.gt_out) ? 4 : 0);
  bool shaped = p.nrounds > 0;
  for (int r = 0; r < p.nrounds; ++r) shaped = shaped && p.rounds[r].shape != 0;
  if (shaped && v != 3 && v != 7) {
    v |= 8;
    // one butterfly pattern for every round (inverse- or forward-only passes)
    for (int pat = 1; pat <= 2; ++pat) {
      bool ok = true;
      for (int r = 0; r < p.nrounds && ok; ++r) {
        const PassRound &rr = p.rounds[r];
        const PassOp &a = p.ops[rr.op_begin];
        ok = a.kind == (pat == 1 ? OP_INV : OP_FWD) && (a.shared != 0) == (pat == 2);
        if (ok && rr.shape == 2) {
          const PassOp &b = p.ops[rr.op_begin + 1];
          ok = b.kind == a.kind && (b.shared != 0) == (pat == 1);
        }
      }
      const int vp = v | (pat << 4);
      // the instantiated ones (inverse pattern: the op kinds stay runtime
      // values there, a compile-time kind measured slower)
      if (ok && (vp == 24 || vp == 25 || vp == 28 || vp == 29 || vp == 40 || vp == 42 || vp == 44 || vp == 46)) {
        v = vp;
        break;
      }
    }
  }
  // mixed inverse / forward rounds (the encode's fused middle pass): the
  // pattern-3 instance runs every straight-line round from one copy of each
  // multiply body.  Its rounds are [distinct-factor op along m0] and/or
  // [shared-factor op along m1] in either order, so forward rounds swap their
  // bits (of a round's two levels the higher one always shares its factor).
  PassParams p3;
  static const bool force3 = std::getenv("LCH_FORCE_PAT3") != nullptr;
  if constexpr (R == 16 && POLY != 0u) {
    if (shaped && (v == 8 || (force3 && (v == 24 || v == 40)))) {
      p3 = p;
      bool ok = true;
      for (int r = 0; r < p3.nrounds && ok; ++r) {
        PassRound &rr = p3.rounds[r];
        PassOp &a = p3.ops[rr.op_begin];
        rr.rev = 0;
        if (rr.shape == 2) {
          PassOp &b = p3.ops[rr.op_begin + 1];
          if (a.shared && !b.shared) {
            std::swap(a, b);
            std::swap(rr.m0, rr.m1);
            a.m = 0;
            b.m = 1;
            rr.rev = 1;
          } else if (a.shared || !b.shared) {
            ok = false;
          }
        } else if (a.shared) {  // a single shared-factor op: along m1
          std::swap(rr.m0, rr.m1);
          a.m = 1;
          rr.shape = 3;
        }
      }
      if (ok) {
        const size_t smem3 = pass_smem_bytes(R, p.tpb, false);
        const int64_t total3 = (int64_t(1) << (p.lgH - p.tpb)) * ngroups;
        return launch_pass_v<R, POLY, 56>(p3, unsigned(std::min<int64_t>(total3, int64_t(4) * sm_count())), smem3, s);
      }
    }
  }
  // row-layout raw I/O (no stripe packets): the packet code paths compiled out
  const bool rows = (p.in_mode != IO_RAW || p.raw_in.pkt == 0) && (p.out_mode != IO_RAW || p.raw_out.pkt == 0);
  if (rows && (v == 25 || v == 29 || v == 42 || v == 46)) v |= 128;
  if (v & 4) {  // scalings only before, or only after the rounds
    const int vs = v | (!(p.npost || p.gt_out) ? 64 : !p.npre ? 256 : 0);
    if (vs == 221 || vs == 108 || vs == 284 || vs == 430) v = vs;
  }
  // raw output from the last round's registers: every tile inside the output
  // window, row layout, 16-byte aligned rows, no merge, last round over tile
  // bits (1, 0) in the forward pattern
  static const bool no_rreg = std::getenv("LCH_NO_RREG") != nullptr;
  if (R == 16 && v == 170 && !no_rreg && p.tpb == 5 && p.nrounds > 0) {
    const RawIO &o = p.raw_out;
    const PassRound &lr = p.rounds[p.nrounds - 1];
    bool ok = o.pkt == 0 && o.vec && !o.merge_src && o.pos_lo == 0 && o.pos_hi >= (int64_t(1) << p.lgH) &&
              lr.shape == 2 && lr.m0 == 1 && lr.m1 == 0 && p.npost == 0 && !p.gt_out;
    for (int m = 0; m < p.tpb; ++m) ok = ok && p.gbit[m] == m;
    if (ok) v = 682;
  }
  // TMA raw input tiles straight into the first round's registers: no
  // pre-scaling, first round over tile bits (0, 1) with every warp active
  static const bool no_fusein = std::getenv("LCH_NO_FUSEIN") != nullptr;
  if (R == 16 && v == 153 && !no_fusein && p.raw_tma && p.tpb == 5 && p.nrounds > 1 && p.npre == 0) {
    const PassRound &fr = p.rounds[0];
    bool ok = fr.m0 == 0 && fr.m1 == 1 && fr.nw == 3;
    for (int w = 0; w < NWARP; ++w) ok = ok && fr.q0w[w] == 4 * w;
    if (ok) v = 1177;
  }
  if (std::getenv("LCH_NO_LEAN")) v = 7;
  const size_t smem = pass_smem_bytes(R, p.tpb, p.out_mode == IO_RAW);
  const int64_t total = (int64_t(1) << (p.lgH - p.tpb)) * ngroups;
  const unsigned ctas = unsigned(std::min<int64_t>(total, int64_t(4) * sm_count()));
  if constexpr (POLY == 0u) {  // runtime polynomial: one generic instance
    (void)v;
    return launch_pass_v<R, 0u, 7>(p, ctas, smem, s);
  } else if constexpr (R == 16) {
    switch (v) {  // the instances the codec's passes use; everything else runs generic
      case 0: return launch_pass_v<R, POLY, 0>(p, ctas, smem, s);
      case 1: return launch_pass_v<R, POLY, 1>(p, ctas, smem, s);
      case 2: return launch_pass_v<R, POLY, 2>(p, ctas, smem, s);
      case 4: return launch_pass_v<R, POLY, 4>(p, ctas, smem, s);
      case 5: return launch_pass_v<R, POLY, 5>(p, ctas, smem, s);
      case 8: return launch_pass_v<R, POLY, 8>(p, ctas, smem, s);
      case 9: return launch_pass_v<R, POLY, 9>(p, ctas, smem, s);
      case 10: return launch_pass_v<R, POLY, 10>(p, ctas, smem, s);
      case 12: return launch_pass_v<R, POLY, 12>(p, ctas, smem, s);
      case 24: return launch_pass_v<R, POLY, 24>(p, ctas, smem, s);
      case 25: return launch_pass_v<R, POLY, 25>(p, ctas, smem, s);
      case 28: return launch_pass_v<R, POLY, 28>(p, ctas, smem, s);
      case 29: return launch_pass_v<R, POLY, 29>(p, ctas, smem, s);
      case 46: return launch_pass_v<R, POLY, 46>(p, ctas, smem, s);
      case 153: return launch_pass_v<R, POLY, 153>(p, ctas, smem, s);
      case 157: return launch_pass_v<R, POLY, 157>(p, ctas, smem, s);
      case 170: return launch_pass_v<R, POLY, 170>(p, ctas, smem, s);
      case 174: return launch_pass_v<R, POLY, 174>(p, ctas, smem, s);
      case 221: return launch_pass_v<R, POLY, 221>(p, ctas, smem, s);
      case 108: return launch_pass_v<R, POLY, 108>(p, ctas, smem, s);
      case 284: return launch_pass_v<R, POLY, 284>(p, ctas, smem, s);
      case 430: return launch_pass_v<R, POLY, 430>(p, ctas, smem, s);
      case 13: return launch_pass_v<R, POLY, 13>(p, ctas, smem, s);
      case 44: return launch_pass_v<R, POLY, 44>(p, ctas, smem, s);
      case 40: return launch_pass_v<R, POLY, 40>(p, ctas, smem, s);
      case 42: return launch_pass_v<R, POLY, 42>(p, ctas, smem, s);
      case 682: return launch_pass_v<R, POLY, 682>(p, ctas, smem, s);
      case 1177: return launch_pass_v<R, POLY, 1177>(p, ctas, smem, s);
      default: return launch_pass_v<R, POLY, 7>(p, ctas, smem, s);
    }
  } else {  // r = 8: the lean and the generic instance only
    return (v & 7) == 0 ? launch_pass_v<R, POLY, 0>(p, ctas, smem, s) : launch_pass_v<R, POLY, 7>(p, ctas, smem, s);
  }
}

template <int R, uint32_t POLY>
cudaError_t launch_gather(const GatherParams &p, int ngroups, cudaStream_t s) {
  const size_t smem = gather_smem_bytes(R, p);
  if (smem > GATHER_SMEM_CAP) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> done{0};
  cudaError_t e = smem_optin(gather_kernel<R, POLY>, int(GATHER_SMEM_CAP), done);
  if (e != cudaSuccess) return e;
  dim3 grid(unsigned(ngroups) * (32u >> p.lwpc), 1u << (p.lgH_in - p.nbits));
  gather_kernel<R, POLY><<<grid, GNT, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwht(const FwhtParams &p, cudaStream_t s) {
  const int64_t blocks = p.nvec * (int64_t(1) << (p.lgn - p.tb));
  fwht_kernel<<<unsigned(blocks), 1 << p.tb, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_decode_rows(const uint16_t *logs, const uint32_t *bits, const uint16_t *exp,
                               uint32_t m, uint32_t n, uint32_t k, uint16_t *pi_row,
                               uint16_t *pinv, int64_t np, cudaStream_t s) {
  decode_rows_kernel<<<dim3((n + 255) / 256, unsigned(np)), 256, 0, s>>>(logs, bits, exp, m, n, k,
                                                                         pi_row, pinv);
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

__global__ void xor_views_kernel(uint16_t *out, int64_t so, const uint16_t *a, int64_t sa,
                                 const uint16_t *b, int64_t sb, int64_t batch, int64_t len,
                                 int64_t pkt) {
  const int64_t total = batch * len;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t oo, oa, ob;
    if (pkt) {
      const int64_t t = i % pkt, rest = i / pkt, j = rest % len, g = rest / len;
      oo = (g * so + j) * pkt + t;
      oa = (g * sa + j) * pkt + t;
      ob = (g * sb + j) * pkt + t;
    } else {
      const int64_t r = i / len, j = i - r * len;
      oo = r * so + j;
      oa = r * sa + j;
      ob = r * sb + j;
    }
    out[oo] = b ? uint16_t(a[oa] ^ b[ob]) : a[oa];
  }
}

cudaError_t launch_xor_views(uint16_t *out, int64_t so, const uint16_t *a, int64_t sa,
                             const uint16_t *b, int64_t sb, int64_t batch, int64_t len, int64_t pkt,
                             cudaStream_t s) {
  const int64_t total = batch * len;
  const int blocks = int(total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32);
  xor_views_kernel<<<blocks, 256, 0, s>>>(out, so, a, sa, b, sb, batch, len, pkt);
  return cudaGetLastError();
}

// Shard-file layouts (reference shardfile.py:16-20,109-140): a file is
// stripes [S][k] of w-byte little-endian symbols (zero padded); shard j holds
// symbol j of every stripe.  The codec's packet layout [positions][P] (one
// stripe group, lanes = stripes) is exactly the shard layout.
__global__ void stripes_to_packets_kernel(const uint8_t *bytes, int64_t len, int w, int64_t k,
                                          int64_t S, uint16_t *pk, int64_t P) {
  const int64_t total = k * P;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = i / P, sidx = i - j * P;
    uint32_t v = 0;
    if (sidx < S) {
      const int64_t off = (sidx * k + j) * w;
      if (off < len) v = bytes[off];
      if (w == 2 && off + 1 < len) v |= uint32_t(bytes[off + 1]) << 8;
    }
    pk[i] = uint16_t(v);
  }
}

__global__ void packets_to_stripes_kernel(const uint16_t *pk, int64_t P, int64_t k, int w,
                                          uint8_t *bytes, int64_t len) {
  for (int64_t off = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; off < len;
       off += int64_t(gridDim.x) * blockDim.x) {
    const int64_t sym = off / w, sidx = sym / k, j = sym - sidx * k;
    const uint16_t v = pk[j * P + sidx];
    bytes[off] = uint8_t(w == 2 && (off & 1) ? (v >> 8) : (v & 0xFF));
  }
}

// shard payloads [rows][S * w] <-> packets [rows][P] (lanes >= S are zero)
__global__ void payload_packets_kernel(const uint8_t *pay, uint16_t *pk, int64_t rows, int64_t S,
                                       int64_t P, int w, int to_packets, uint8_t *pay_out,
                                       const uint16_t *pk_in) {
  const int64_t total = rows * P;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / P, sidx = i - row * P;
    if (to_packets) {
      uint32_t v = 0;
      if (sidx < S) {
        const uint8_t *src = pay + (row * S + sidx) * w;
        v = w == 2 ? uint32_t(src[0]) | (uint32_t(src[1]) << 8) : src[0];
      }
      pk[i] = uint16_t(v);
    } else if (sidx < S) {
      const uint16_t v = pk_in[i];
      uint8_t *dst = pay_out + (row * S + sidx) * w;
      dst[0] = uint8_t(v & 0xFF);
      if (w == 2) dst[1] = uint8_t(v >> 8);
    }
  }
}

// out[i] = a[i] * b[i] in GF(2^r) via the log/exp tables (transform.py:204-205)
__global__ void pointwise_mul_kernel(const uint16_t *a, const uint16_t *b, uint16_t *out, int64_t count,
                                     const uint16_t *log, const uint16_t *exp, uint32_t m) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = a[i], y = b[i];
    uint32_t r = 0;
    if (m == 0xFFFFu && !log) {
      r = gf16_mul(x, y);  // r = 16 with x^16 + x^12 + x^3 + x + 1: no tables
    } else if (x && y) {
      uint32_t e = uint32_t(__ldg(log + x)) + __ldg(log + y);
      e = e >= m ? e - m : e;
      r = __ldg(exp + e);
    }
    out[i] = uint16_t(r);
  }
}

// Formal derivative by the direct per-coefficient formula (derivative.py:26-43):
// out[j] = sum over clear bits l of j (j + 2^l < h) of W'_l * d[j + 2^l].  A
// generic shift-and-reduce product (any r <= 16, any polynomial): an
// independent path from the B-scaled gather of lch_derivative.
__device__ __forceinline__ uint32_t gf_mul_generic(uint32_t a, uint32_t b, int r, uint32_t poly) {
  uint32_t z = 0;
  for (int i = 0; i < r; ++i)
    if ((b >> i) & 1u) z ^= a << i;
  for (int i = 2 * r - 2; i >= r; --i)
    if ((z >> i) & 1u) z ^= poly << (i - r);
  return z;
}

__global__ void derivative_direct_kernel(const uint16_t *in, uint16_t *out, int64_t batch, int64_t stride,
                                         int lg_h, WPrime wp) {
  const int64_t h = int64_t(1) << lg_h, total = batch * h;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i >> lg_h, j = i & (h - 1);
    const uint16_t *row = in + b * stride;
    uint32_t acc = 0;
    for (int l = 0; l < lg_h; ++l) {
      if ((j >> l) & 1) continue;
      const uint32_t d = __ldg(row + j + (int64_t(1) << l));
      if (d) acc ^= gf_mul_generic(wp.w[l], d, wp.r, wp.poly);
    }
    out[b * stride + j] = uint16_t(acc);
  }
}

static int grid_for(int64_t total) {
  return int(total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32);
}

__global__ void expand_rows_kernel(const uint16_t *comp, int64_t cs, const int32_t *rank, uint16_t *full,
                                   int64_t n, int64_t rows) {
  const int64_t total = rows * n;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / n, j = i - r * n;
    const int32_t q = __ldg(rank + j);
    full[i] = q >= 0 ? comp[r * cs + q] : uint16_t(0);
  }
}

cudaError_t launch_expand_rows(const uint16_t *comp, int64_t comp_stride, const int32_t *rank, uint16_t *full,
                               int64_t n, int64_t rows, cudaStream_t s) {
  expand_rows_kernel<<<grid_for(rows * n), 256, 0, s>>>(comp, comp_stride, rank, full, n, rows);
  return cudaGetLastError();
}

__global__ void expand_packets_kernel(const uint4 *comp, int64_t comp_pos, const int32_t *rank,
                                      int64_t rank_stride, uint4 *full, int64_t n, int64_t pk4, int64_t groups) {
  const int64_t total = groups * n * pk4;  // in uint4 (8 symbols)
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i % pk4, rest = i / pk4, j = rest % n, g = rest / n;
    const int32_t q = __ldg(rank + g * rank_stride + j);
    full[i] = q >= 0 ? __ldcs(comp + (g * comp_pos + q) * pk4 + t) : make_uint4(0u, 0u, 0u, 0u);
  }
}

cudaError_t launch_expand_packets(const uint16_t *comp, int64_t comp_pos, const int32_t *rank,
                                  int64_t rank_stride, uint16_t *full, int64_t n, int64_t pkt, int64_t groups,
                                  cudaStream_t s) {
  const int64_t pk4 = pkt / 8;
  expand_packets_kernel<<<grid_for(groups * n * pk4), 256, 0, s>>>(
      reinterpret_cast<const uint4 *>(comp), comp_pos, rank, rank_stride, reinterpret_cast<uint4 *>(full), n,
      pk4, groups);
  return cudaGetLastError();
}

cudaError_t launch_derivative_direct(const uint16_t *in, uint16_t *out, int64_t batch, int64_t stride,
                                     int lg_h, const WPrime &wp, cudaStream_t s) {
  derivative_direct_kernel<<<grid_for(batch << lg_h), 256, 0, s>>>(in, out, batch, stride, lg_h, wp);
  return cudaGetLastError();
}

cudaError_t launch_pointwise_mul(const uint16_t *a, const uint16_t *b, uint16_t *out, int64_t count,
                                 const uint16_t *log, const uint16_t *exp, uint32_t m, cudaStream_t s) {
  pointwise_mul_kernel<<<grid_for(count), 256, 0, s>>>(a, b, out, count, log, exp, m);
  return cudaGetLastError();
}

cudaError_t launch_stripes_to_packets(const uint8_t *bytes, int64_t len, int w, int64_t k, int64_t S,
                                      uint16_t *pk, int64_t P, cudaStream_t s) {
  stripes_to_packets_kernel<<<grid_for(k * P), 256, 0, s>>>(bytes, len, w, k, S, pk, P);
  return cudaGetLastError();
}
cudaError_t launch_packets_to_stripes(const uint16_t *pk, int64_t P, int64_t k, int w, uint8_t *bytes,
                                      int64_t len, cudaStream_t s) {
  packets_to_stripes_kernel<<<grid_for(len), 256, 0, s>>>(pk, P, k, w, bytes, len);
  return cudaGetLastError();
}
cudaError_t launch_payload_packets(const uint8_t *pay, uint16_t *pk, int64_t rows, int64_t S, int64_t P,
                                   int w, int to_packets, uint8_t *pay_out, const uint16_t *pk_in,
                                   cudaStream_t s) {
  payload_packets_kernel<<<grid_for(rows * P), 256, 0, s>>>(pay, pk, rows, S, P, w, to_packets, pay_out,
                                                             pk_in);
  return cudaGetLastError();
}

cudaError_t launch_gen_packets(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                               uint32_t mask, uint16_t *out, int64_t npos, int64_t pkt,
                               cudaStream_t s) {
  const int64_t total = batch * len;
  const int blocks = int(total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32);
  gen_packets_kernel<<<blocks, 256, 0, s>>>(seed, cw0, batch, len, mask, out, npos, pkt);
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
template cudaError_t launch_pass<16, 0u>(const PassParams &, int, cudaStream_t);
template cudaError_t launch_pass<8, 0u>(const PassParams &, int, cudaStream_t);
template cudaError_t launch_gather<16, 0x1100Bu>(const GatherParams &, int, cudaStream_t);
template cudaError_t launch_gather<8, 0x11Du>(const GatherParams &, int, cudaStream_t);
template cudaError_t launch_gather<16, 0u>(const GatherParams &, int, cudaStream_t);
template cudaError_t launch_gather<8, 0u>(const GatherParams &, int, cudaStream_t);
#endif  // LCH_PASS_TU

}  // namespace lch
