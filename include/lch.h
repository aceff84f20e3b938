/*
 * lch.h -- C ABI of the B200 (sm_100a) Lin-Chung-Han transform + RS(2^r, k)
 * erasure codec.  Implemented by paper_1404_3458_b200/csrc (liblch.so).
 *
 * The reference (`binfec`, pure Python) exposes this path as a Python module
 * API with no FFI layer; each entry point below names the reference function
 * it replaces.  Python binds them with ctypes (paper_1404_3458_b200/_lib.py);
 * INTEGRATION.md shows the binding a binfec maintainer would add.
 *
 * Conventions
 *  - Symbols are uint16 for r = 8 and r = 16 (batch.py:33,116).  Element i of
 *    the field is the integer i, so field addition is XOR (field.py:1-13).
 *  - Row-major batches: element (b, j) at ptr[b * row_stride + j]
 *    (row_stride in elements, >= the row length).  Packet-major batches
 *    (packet_len P > 0): element (g, j, s) of stripe group g, position j,
 *    packet symbol s at ptr[(g * n_pos + j) * P + s]; batch = groups * P,
 *    P a multiple of 1024, pointers 16-byte aligned, and the stride
 *    arguments give n_pos (positions per stripe group).  Lane g * P + s of a
 *    stripe group is an ordinary codeword (shard j = symbol j of every
 *    stripe, shardfile.py:16-20,129-140).
 *  - All data pointers are DEVICE pointers unless the name says host_.
 *    `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous with respect to the host unless stated otherwise.
 *  - Return 0 on success or a negative LCH_E* code; lch_strerror() names it.
 *    The Python shim maps LCH_EINVAL -> ValueError, LCH_ETOOMANY ->
 *    TooManyErasuresError(ValueError) (rs.py:30-31,121-123), LCH_EZERODIV ->
 *    ZeroDivisionError (field.py:83-84).
 *  - There is no CPU fallback: without a CUDA device every compute entry point
 *    returns LCH_ECUDA.
 *  - A context uploads its tables to the device current at its first compute
 *    call and stays bound to it (calls with another current device return
 *    LCH_EINVAL); use one context per GPU.
 */
#ifndef LCH_H
#define LCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCH_OK 0
#define LCH_EINVAL -1      /* ValueError */
#define LCH_ETOOMANY -2    /* TooManyErasuresError */
#define LCH_ENOTPRIM -3    /* ValueError("not primitive") from build_tables */
#define LCH_ECUDA -4       /* CUDA runtime failure / no device */
#define LCH_ENOMEM -5
#define LCH_EUNSUPPORTED -6
#define LCH_EZERODIV -7

typedef struct lch_ctx lch_ctx;

/* Version string of the library build. */
const char *lch_version(void);
const char *lch_strerror(int code);

/* Build field + basis tables on the host and upload them.
 * Replaces field.tables_for / build_tables (field.py:100-135),
 * basis.build_basis_tables (basis.py:135-137) and walsh._fwht_of_log
 * (walsh.py:64-74).  max_h = 2^max_lg_h (<= 2^r). */
int lch_init(int r, uint32_t poly, int max_lg_h, lch_ctx **out);
/* As lch_init with the log/exp tables built from the generator alpha (an
 * element index, FieldParams.alpha_index, field.py:31-49); LCH_ENOTPRIM when
 * alpha does not generate GF(2^r)*.  lch_init uses alpha = 2 (the polynomial
 * x).  Any primitive reduction polynomial is accepted; the two reference
 * defaults run specialised kernels, others the runtime-taps instances. */
int lch_init_alpha(int r, uint32_t poly, uint32_t alpha, int max_lg_h, lch_ctx **out);
void lch_destroy(lch_ctx *ctx);

/* Host copies of the tables (any pointer may be NULL).  Sizes: log[2^r],
 * exp[2^r - 1], w_hat[max_h - 1] (level i at offset max_h - (max_h >> i)),
 * w_prime[r], b_prod[max_h], b_prod_inv[max_h], fwht_log[2^r] (uint32),
 * w_on_basis[r*r], w_norm[r].  Mirrors FieldTables/BasisTables attributes. */
int lch_get_tables(const lch_ctx *ctx, uint16_t *host_log, uint16_t *host_exp,
                   uint16_t *host_w_hat, uint16_t *host_w_prime,
                   uint16_t *host_b_prod, uint16_t *host_b_prod_inv,
                   uint32_t *host_fwht_log, uint16_t *host_w_on_basis,
                   uint16_t *host_w_norm);

/* Batched transform Psi_h^shift, in place on a row-major or packet-major
 * batch.  Replaces transform.forward/_forward_inplace (transform.py:69-76,
 * 102-140) and BatchCodec._forward_inplace (batch.py:65-81). */
int lch_forward(lch_ctx *ctx, uint16_t *data, int64_t batch, int64_t row_stride,
                int lg_h, uint32_t shift, int64_t packet_len, void *stream);
/* (Psi_h^shift)^-1 in place.  Replaces transform.inverse/_inverse_inplace
 * (transform.py:79-86, 143-175) and BatchCodec._inverse_inplace (batch.py:83-99). */
int lch_inverse(lch_ctx *ctx, uint16_t *data, int64_t batch, int64_t row_stride,
                int lg_h, uint32_t shift, int64_t packet_len, void *stream);
/* Formal derivative in the basis, out-of-place (in != out, same strides).
 * Replaces derivative.derivative_fast (derivative.py:46-77) and
 * BatchCodec._derivative (batch.py:101-106). */
int lch_derivative(lch_ctx *ctx, const uint16_t *in, uint16_t *out, int64_t batch,
                   int64_t row_stride, int lg_h, int64_t packet_len, void *stream);

/* Formal derivative by the direct formula out[j] = sum_{l : bit l of j clear}
 * W'_l * in[j + 2^l] (derivative.derivative_direct, derivative.py:26-43):
 * an independent check of lch_derivative, row layout only, in != out. */
int lch_derivative_direct(lch_ctx *ctx, const uint16_t *in, uint16_t *out, int64_t batch,
                          int64_t row_stride, int lg_h, void *stream);

/* In-place Walsh-Hadamard transform over Z_modulus of `batch` vectors of
 * length 2^lg_n (uint32 residues).  Replaces walsh.fwht (walsh.py:42-61). */
int lch_fwht(lch_ctx *ctx, uint32_t *data, int64_t batch, int lg_n, uint32_t modulus,
             void *stream);

/* Erasure-locator values for `npatterns` erasure bitmasks (2^r bits each,
 * bit j of word j/32 set = position j erased).  loc_out[p][j] = Pi_bar(j) for
 * survivors, Pi'(j) for erased positions (walsh.locator_values,
 * walsh.py:77-115).  log_out (optional, uint16 [npatterns][2^r]) receives the
 * log-domain values.  Validation (walsh.py:85-96) is the caller's job: each
 * pattern must erase >= 1 and <= 2^r - 1 positions. */
int lch_locator(lch_ctx *ctx, const uint32_t *erasure_bits, int64_t npatterns,
                uint16_t *loc_out, uint16_t *log_out, void *stream);

/* Systematic RS(2^r, 2^lg_k) encode.  msg: [batch][k] (row_stride_in);
 * parity: [batch][n-k] (row_stride_out), parity block i-1 (shift i*k) at
 * columns [(i-1)k, ik).  Replaces rs.encode (rs.py:85-96) and
 * BatchCodec.encode (batch.py:110-124); the message columns of the reference's
 * codeword are the input itself (systematic), so callers that want [batch][n]
 * pass parity = codeword + k with row_stride_out = n.  Packet-major when
 * packet_len > 0 (msg: [groups][k][P], parity: [groups][n-k][P]). */
int lch_encode(lch_ctx *ctx, const uint16_t *msg, int64_t row_stride_in,
               uint16_t *parity, int64_t row_stride_out, int64_t batch, int lg_k,
               int64_t packet_len, void *stream);

/* Erasure decode.  rx: [batch][n] (row_stride_in), values at erased
 * positions ignored; erasure_bits: one bitmask (shared = 1) or one per row
 * (shared = 0); out: [batch][k] (row_stride_out).  Returns LCH_ETOOMANY when a
 * pattern erases more than n - k positions; an empty pattern is a copy.
 * Replaces rs.decode (rs.py:99-149) and BatchCodec.decode (batch.py:126-153).
 * Packet layout: see lch_decode_k (shared = 0 means one pattern per group).
 * host_counts (optional): per-pattern erasure counts if the caller already
 * knows them (skips a device->host read). */
int lch_decode(lch_ctx *ctx, const uint16_t *rx, int64_t row_stride_in,
               const uint32_t *erasure_bits, int shared, uint16_t *out,
               int64_t row_stride_out, int64_t batch, int lg_k, int64_t packet_len,
               const int64_t *host_counts, void *stream);

/* General-k systematic RS(2^r, k) encode, 1 <= k <= 2^r.
 * The codeword is the evaluation at omega_0..omega_(n-1) of the unique
 * polynomial of degree < k through the message at omega_0..omega_(k-1)
 * (novel-basis interpolation).  For power-of-two k this is lch_encode
 * (rs.encode, rs.py:85-96); otherwise the default is a recursive systematic
 * encoder over the binary expansion of k (fused power-of-two encode plans
 * and XORs); LCH_ENCODE_BY_DECODE=1 selects the
 * erasure-decode formulation instead (E = [k, n), the reference's decode
 * algorithm rs.py:125-148; same codeword, kept as a cross-check).  Layouts
 * as lch_encode; in packet layout the strides count positions per stripe
 * group. */
int lch_encode_k(lch_ctx *ctx, const uint16_t *msg, int64_t stride_in, uint16_t *parity,
                 int64_t stride_out, int64_t batch, int64_t k, int64_t packet_len,
                 void *stream);

/* General-k erasure decode (rs.decode, rs.py:99-149 with the power-of-two
 * restriction of rs.py:43-44 lifted): recovers positions [0, k) from any
 * <= n - k erasures.  Row layout: shared = 1 (one pattern) or 0 (one per
 * row).  Packet layout: shared = 1 (one pattern) or 0 (one pattern
 * per stripe group, erasure_bits [batch / packet_len][2^r / 32]). */
int lch_decode_k(lch_ctx *ctx, const uint16_t *rx, int64_t stride_in,
                 const uint32_t *erasure_bits, int shared, uint16_t *out, int64_t stride_out,
                 int64_t batch, int64_t k, int64_t packet_len, const int64_t *host_counts,
                 void *stream);

/* Host-buffer codec (the reference's host-array API, batch.py:110-153):
 * inputs and outputs in host memory (page-locked for full overlap).  The
 * batch streams through the GPU in chunks of `chunk` rows (codewords, or
 * stripe groups when packet_len > 0; 0 = ~64 MiB per chunk): host->device
 * copies, kernels and device->host copies of neighbouring chunks overlap on
 * three streams.  The kernels and the OUTPUT buffers are ordered on `stream`
 * like the device entry points.  Host INPUT buffers must hold their data when
 * the call is made (like the arrays handed to the reference's BatchCodec):
 * their copies start right away, so they overlap the tail of an earlier call
 * still in flight on the same context (the device slots and page-locked
 * staging persist in the context; lch_release_host_buffers frees them).
 * lch_set_host_ordering(ctx, 1) restores stream-ordered reads of the inputs
 * (for callers that fill them by earlier work on `stream`).  Layouts and
 * semantics as lch_encode_k / lch_decode_k; erasure counts are taken from the
 * host bitmasks (no device round trip). */
int lch_encode_host(lch_ctx *ctx, const uint16_t *host_msg, int64_t stride_in,
                    uint16_t *host_parity, int64_t stride_out, int64_t batch, int64_t k,
                    int64_t packet_len, int64_t chunk, void *stream);
int lch_decode_host(lch_ctx *ctx, const uint16_t *host_rx, int64_t stride_in,
                    const uint32_t *host_bits, int shared, uint16_t *host_out,
                    int64_t stride_out, int64_t batch, int64_t k, int64_t packet_len,
                    int64_t chunk, void *stream);

/* stream_ordered != 0: the host-buffer entry points read their host inputs in
 * stream order (after the work already queued on `stream`); 0 (default): at
 * the call. */
int lch_set_host_ordering(lch_ctx *ctx, int stream_ordered);
/* Bytes the host-buffer entry points have queued for host->device and
 * device->host copies since the context was created (bench accounting: a
 * shared-pattern decode sends a chunk compacted or as it is). */
int lch_host_copy_bytes(lch_ctx *ctx, uint64_t *h2d_bytes, uint64_t *d2h_bytes);
/* Waits for the device and frees the pipeline's persistent device slots and
 * page-locked staging buffers (they are re-created on demand). */
int lch_release_host_buffers(lch_ctx *ctx);

/* Host helper of the decode pipeline: row r of host_out = the survivors
 * (bit j of host_bits clear) of row r of host_rx, in order (multi-threaded,
 * AVX-512 VBMI2 compress-store when available).  No device involved. */
int lch_compact_rows(lch_ctx *ctx, const uint16_t *host_rx, int64_t stride,
                     const uint32_t *host_bits, int64_t n, int64_t rows, uint16_t *host_out,
                     int64_t out_stride);

/* Device scratch budget per call (bytes, default 4 GiB): batches whose
 * bit-sliced intermediates exceed it are processed in lane chunks. */
int lch_set_scratch_limit(lch_ctx *ctx, uint64_t bytes);

/* out[i] = a[i] * b[i] in GF(2^r) (the pointwise step of transform.poly_mul,
 * transform.py:204-205); out may alias a or b. */
int lch_pointwise_mul(lch_ctx *ctx, const uint16_t *a, const uint16_t *b, uint16_t *out,
                      int64_t count, void *stream);

/* Shard-file layouts (reference shardfile.py:16-20,109-140).  A file of
 * `len` bytes is stripes [S][k] of r/8-byte little-endian symbols, zero
 * padded (S = ceil(len / (k r/8))); shard j holds symbol j of every stripe.
 * The codec's packet layout with one stripe group and lanes = stripes,
 * packets [positions][packet_len] (packet_len >= S, lanes >= S zero), is the
 * shard layout:
 *   lch_stripes_to_packets   file bytes -> message packets [k][packet_len]
 *   lch_packets_to_stripes   message packets -> file bytes (cut to len)
 *   lch_payload_to_packets   shard payloads [rows][S * r/8] -> packets
 *   lch_packets_to_payload   packets -> shard payloads
 * All pointers are device pointers. */
int lch_stripes_to_packets(lch_ctx *ctx, const uint8_t *file, int64_t len, int r, int64_t k,
                           uint16_t *packets, int64_t packet_len, void *stream);
int lch_packets_to_stripes(lch_ctx *ctx, const uint16_t *packets, int64_t packet_len, int r,
                           int64_t k, uint8_t *file, int64_t len, void *stream);
int lch_payload_to_packets(lch_ctx *ctx, const uint8_t *payload, int64_t rows, int64_t stripes,
                           int r, uint16_t *packets, int64_t packet_len, void *stream);
int lch_packets_to_payload(lch_ctx *ctx, const uint16_t *packets, int64_t packet_len, int64_t rows,
                           int64_t stripes, int r, uint8_t *payload, void *stream);

/* Seeded counter-based inputs (oracle/lch_oracle.c orc_key):
 * out[b][j] = key(seed, cw0 + b, j) & (2^r - 1), row-major with row_stride. */
int lch_gen_symbols(lch_ctx *ctx, uint64_t seed, uint64_t cw0, int64_t batch,
                    int64_t len, uint16_t *out, int64_t row_stride, void *stream);
/* Packet-major seeded inputs: lane b = g * packet_len + s holds codeword
 * cw0 + b, so out[(g * n_pos + j) * packet_len + s] = key(seed, cw0 + b, j)
 * & (2^r - 1) for j < len (batch = groups * packet_len). */
int lch_gen_packets(lch_ctx *ctx, uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                    uint16_t *out, int64_t n_pos, int64_t packet_len, void *stream);
/* keys[b][j] = key(seed, cw0 + b, j) >> 1 (int64, for the erasure selection). */
int lch_gen_keys(lch_ctx *ctx, uint64_t seed, uint64_t cw0, int64_t batch, int64_t len,
                 int64_t *keys, void *stream);

/* Kernel launches issued by this context since creation (bench accounting). */
int64_t lch_launch_count(const lch_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
