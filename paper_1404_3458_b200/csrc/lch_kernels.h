// Kernel parameter blocks and launchers (device side in lch_kernels.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lch {

constexpr int NT = 256;        // threads per CTA (8 warps)
constexpr int NWARP = NT / 32;
constexpr int TPB_MAX = 5;     // tile = 2^5 positions x 1024 batch lanes
constexpr int GROUP = 1024;    // batch lanes per CTA: 32 threads x 32 bits
constexpr int MAXOPS = 24;
constexpr int MAXROUNDS = 12;
constexpr int MAXSCALE = 4;

// OP_INVFWD: an inverse level followed by the forward level on the same bit,
// v' = u + v; u'' = u + (f_inv + f_fwd) v'; v'' = u'' + v' (one multiply; the
// table parts of the two factors cancel, so its factor is hs alone)
enum OpKind : int { OP_FWD = 0, OP_INV = 1, OP_SCALE = 2, OP_INVFWD = 3 };
enum IoMode : int { IO_BS = 0, IO_RAW = 1 };

struct PassOp {
  int kind;
  int m;                  // FWD/INV: which bit of the round (0 -> m0, 1 -> m1)
  int mloc;               // FWD/INV: the op's local tile bit
  int level;              // global butterfly level i
  uint32_t hs;            // W^_i(shift) (0 for shift 0)
  const uint16_t *table;  // per-position factors (SCALE), indexed by position
  int64_t tab_stride;     // SCALE: + (stripe group) * tab_stride (0: one row for all)
  int shared;             // FWD/INV: both pairs of the round share the factor (the
                          // other round bit lies below the level, transform.py:123)
};

// A round: every thread holds the 4 positions spanned by tile bits m0, m1
// (radix-4, two levels per shared-memory round trip); the warp index
// enumerates the remaining nw tile bits obit[].
struct PassRound {
  int m0, m1;             // local tile bits (m1 = -1: only m0 exists, tpb == 1)
  int nw;
  int obit[TPB_MAX];
  int op_begin, op_end;   // butterfly ops of the round in ops[]
  uint8_t q0w[NWARP];     // warp w's first tile position (obit[] spread of w), precomputed
  int shape;              // 0 general; 1: one op along m0; 2: one along m0 then one along m1;
                          // 3 (pattern-3 instances): one op along m1
  int rev;                // pattern-3 instances: the op along m1 runs first
};

// Raw uint16 batch: element (b, j) at ptr[b * row_stride + j].
// Decode epilogue: if merge_src, out(b, j) = erased(j) ? computed : merge_src(b, j)
// with erased(j) = bit j of merge_bits.
// Raw uint16 batch: element (b, j) at ptr[b * row_stride + j].
// Decode epilogue (merge_src != null): out(b, j) = erased(b, j) ? computed' :
// merge_src(b, j), with erased(b, j) = bit j of merge_bits + b * bits_stride
// (bits_stride = 0: one shared pattern) and computed' = computed, or, with
// per-codeword patterns (pinv_log != null), computed * alpha^pinv_log(b, j)
// (division by Pi'(j), rs.py:141-148) through the log/exp tables.
struct RawIO {
  uint16_t *ptr;
  int64_t row_stride;
  // packet-major layout (pkt > 0): element (b, j) at
  // ptr[((b / pkt) * npos + (j - pos_lo)) * pkt + b % pkt]; row-major
  // otherwise.  Only positions j in [pos_lo, pos_hi) exist in the buffer
  // (loads outside read 0, stores outside are dropped).
  int64_t pkt, npos;
  int64_t pos_lo, pos_hi;
  const uint16_t *merge_src;
  int64_t merge_stride;
  const uint32_t *merge_bits;
  int64_t bits_stride;      // words between consecutive rows' bitmasks (0 = shared)
  const uint16_t *pinv_log; // [batch][pinv_stride] or null
  int64_t pinv_stride;
  int pinv_val;             // R = 16: pinv_log holds alpha^pinv (values), multiplied without tables
  const uint16_t *log_tab, *exp_tab;
  uint32_t mord;            // 2^r - 1
  int vec;  // 16-byte vector accesses allowed
  int al4;  // 4-byte aligned rows
};

struct PassParams {
  // raw_tma: the raw input tiles arrive by TMA through tm_in, a 3-D view
  // {8 symbols (16 B), 16-byte chunks, rows} of the row-major input, as
  // chunk-major [chunk][row][16 B] shared-memory tiles (R = 16, row layout,
  // tile = positions 32t .. 32t+31)
  alignas(64) CUtensorMap tm_in;
  // merge_tma: the decode's survivor source (raw_out.merge_src) for position
  // chunks 0-1 of each output tile arrives by TMA (tm_merge, same view as
  // tm_in) into the spare 32 KB of shared memory while the tile computes
  alignas(64) CUtensorMap tm_merge;
  int raw_tma, merge_tma;
  // raw_bulk: packet-layout raw input tiles (R = 16, tile = 32 consecutive
  // positions, window aligned to 32): each position's 1024 lanes are one
  // contiguous 2 KB run, fetched by a 1-D bulk copy into [position][lane]
  int raw_bulk;
  uint32_t taps;         // reduction polynomial & (2^R - 1) (runtime-polynomial instances)
  int nops;
  PassOp ops[MAXOPS];
  int nrounds;
  PassRound rounds[MAXROUNDS];
  int npre, npost;        // per-position scalings before / after the rounds
  PassOp pre[MAXSCALE], post[MAXSCALE];
  int tpb;               // tile bits
  int gbit[TPB_MAX];     // tile bit m -> global position bit
  int lgH;               // positions in the buffers = 2^lgH
  int nnb;               // non-tile bits
  int nbit[16];          // non-tile bit i -> global position bit
  uint32_t ins_mask[TPB_MAX];  // (1 << g) - 1 for the tile bits g, ascending: tile base =
                               // tile index with a zero inserted at each g
  int lgnt;              // log2 of the tiles per group (lgH - tpb)
  int64_t batch;
  int ngroups;           // 1024-lane batch groups
  int64_t pkt;           // stripe-group size in batch lanes (table rows), 0 = none
  int in_mode, out_mode;
  const uint4 *bs_in;    // BS buffers: block (g, pos) = 32*R words at ((g << lgH) + pos) * 8R uint4
  uint4 *bs_out;
  RawIO raw_in, raw_out;
  const uint16_t *w_hat;
  uint32_t w_hat_off[17];
  uint4 *gt_out;         // gather epilogue: partial derivative sums over the tile bits
  int gt_lgH;
  int dbg;  // experiments only: 1 = skip global I/O, 2 = skip butterflies
};

// XOR-gather step of the formal derivative (derivative.py:60-70) over a set
// of position bits, lanes over positions (no factor is involved, except the
// optional constant-multiplied special bit):
//   T[j] = T_in[j] + sum_{m != sb, bit m of j clear} y[j | 2^bits[m]]
//                  + c * (y[j] + y[j | 2^bits[sb]])   (if sb >= 0, bit clear)
// for j < 2^lgH_out.  One CTA per (tile, group, lane-word).
constexpr int GMAXB = 11;
constexpr size_t GATHER_SMEM_MAX = 96 * 1024;  // 2 CTAs per SM
// largest tile (1 CTA per SM): two lane-words per CTA, so every 16-byte chunk
// read shares its 32-byte sector with the neighbouring lane-word's
constexpr size_t GATHER_SMEM_CAP = 200 * 1024;
struct GatherParams {
  uint32_t taps;  // reduction polynomial & (2^R - 1) (runtime-polynomial instances)
  int nbits;
  int bits[GMAXB];
  int sb;                // the special (top) position bit, not a tile bit, or -1
  uint32_t c;            // constant for the special bit
  int lgH_in, lgH_out;
  int nnb;
  int nbit[16];
  int lwpc;              // log2 lane-words per CTA (0..5)
  // summed bits that are NOT tile bits: the partner y[j | 2^dbits[i]] of every
  // output with that bit clear streams from global memory (the tile then has
  // fewer positions and more lane-words: longer contiguous runs per position)
  int ndirect;
  int dbits[4];
  const uint4 *y;
  const uint4 *t_in;     // may be null
  uint4 *t_out;
};
struct FwhtParams {
  uint32_t *data;        // [nvec][2^lgn]
  int64_t nvec;
  int lgn, b0, tb;       // this pass covers bits [b0, b0 + tb)
  uint32_t mod;
  const uint32_t *bits;  // indicator input (bitmask) when non-null
  const uint32_t *bits_e;  // erasure bitmask for the decode epilogue
  const uint32_t *post_mul;  // multiply by post_mul[j] mod after the pass
  // epilogue (locator): loc = exp[x], log = x
  const uint16_t *exp;
  uint16_t *loc_out, *log_out;
  // per-codeword decode epilogue (rs.py:130-134, 141-148): phi = rx * Pi_bar
  // on survivors (0 on erasures) and pinv_log = -log Pi' on erased j < k
  const uint16_t *rx;
  int64_t rx_stride;
  const uint16_t *log;
  uint16_t *phi;
  uint16_t *pinv_log;
  uint32_t k;
};

// Small-codeword GF(2^8) codec (lch_small.cu): one CTA per codeword.
struct Small8Params {
  int mode;                 // 0 encode (power-of-two k), 1 decode (any k)
  int k, lg_k, max_h;
  int64_t batch;
  const uint16_t *in;       // message [batch][k] or received [batch][256]
  int64_t in_stride;
  uint16_t *out;            // parity [batch][256 - k] or message [batch][k]
  int64_t out_stride;
  const uint32_t *bits;     // decode: erasure bitmask words, 8 per pattern
  int64_t bits_stride;      // 0 = one shared pattern
  const uint16_t *log, *exp, *w_hat, *b_prod, *b_prod_inv;
  const uint32_t *fwht_log;
  uint8_t hs[256 * 8];      // encode: W^_i(blk * k) per parity block and level
};
cudaError_t launch_small8(const Small8Params &p, cudaStream_t s);

template <int R, uint32_t POLY>
cudaError_t launch_pass(const PassParams &p, int ngroups, cudaStream_t s);
size_t gather_smem_bytes(int R, const GatherParams &p);
template <int R, uint32_t POLY>
cudaError_t launch_gather(const GatherParams &p, int ngroups, cudaStream_t s);
cudaError_t launch_fwht(const FwhtParams &p, cudaStream_t s);
// whole r = 16 locator per pattern (bits, post_mul = FWHT(log), exp, and the
// loc/log or decode epilogue fields of FwhtParams)
cudaError_t launch_locator16(const FwhtParams &p, cudaStream_t s);
cudaError_t launch_decode_rows(const uint16_t *logs, const uint32_t *bits, const uint16_t *exp,
                               uint32_t m, uint32_t n, uint32_t k, uint16_t *pi_row,
                               uint16_t *pinv, int64_t np, cudaStream_t s);
// out = a ^ b (or a when b is null) over positions [0, len) of `batch` lanes,
// row (pkt = 0, strides = row strides) or packet layout (strides = positions
// per stripe group); out may alias a or b.
cudaError_t launch_xor_views(uint16_t *out, int64_t so, const uint16_t *a, int64_t sa,
                             const uint16_t *b, int64_t sb, int64_t batch, int64_t len, int64_t pkt,
                             cudaStream_t s);
// full[r][j] = rank[j] >= 0 ? comp[r][rank[j]] : 0 (survivor rows -> n-wide rows)
cudaError_t launch_expand_rows(const uint16_t *comp, int64_t comp_stride, const int32_t *rank, uint16_t *full,
                               int64_t n, int64_t rows, cudaStream_t s);
// packets: full[g][j][P] = rank[g*rank_stride + j] >= 0 ? comp[g][rank][P] : 0
cudaError_t launch_expand_packets(const uint16_t *comp, int64_t comp_pos, const int32_t *rank,
                                  int64_t rank_stride, uint16_t *full, int64_t n, int64_t pkt, int64_t groups,
                                  cudaStream_t s);
struct WPrime {
  uint32_t w[16];  // W'_l (derivative.py:80-82)
  int r;
  uint32_t poly;
};
cudaError_t launch_derivative_direct(const uint16_t *in, uint16_t *out, int64_t batch, int64_t stride,
                                     int lg_h, const WPrime &wp, cudaStream_t s);
cudaError_t launch_pointwise_mul(const uint16_t *a, const uint16_t *b, uint16_t *out, int64_t count,
                                 const uint16_t *log, const uint16_t *exp, uint32_t m, cudaStream_t s);
cudaError_t launch_stripes_to_packets(const uint8_t *bytes, int64_t len, int w, int64_t k, int64_t S,
                                      uint16_t *pk, int64_t P, cudaStream_t s);
cudaError_t launch_packets_to_stripes(const uint16_t *pk, int64_t P, int64_t k, int w, uint8_t *bytes,
                                      int64_t len, cudaStream_t s);
cudaError_t launch_payload_packets(const uint8_t *pay, uint16_t *pk, int64_t rows, int64_t S, int64_t P,
                                   int w, int to_packets, uint8_t *pay_out, const uint16_t *pk_in,
                                   cudaStream_t s);
cudaError_t launch_gen_packets(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                               uint32_t mask, uint16_t *out, int64_t npos, int64_t pkt,
                               cudaStream_t s);
cudaError_t launch_gen_symbols(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                               uint32_t mask, uint16_t *out, int64_t row_stride,
                               cudaStream_t s);
cudaError_t launch_gen_keys(uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                            int64_t *keys, cudaStream_t s);
cudaError_t launch_count_bits(const uint32_t *bits, int64_t npatterns, int words,
                              int64_t *counts, cudaStream_t s);

size_t pass_smem_bytes(int R, int tpb, bool raw);

}  // namespace lch
