/*
 * lch_oracle.h -- CPU restatement of the reference algorithm (TEST INFRASTRUCTURE).
 *
 * This header and lch_oracle.c are the parity oracle for the B200 codec.  They
 * restate, in plain C, the arithmetic of the reference package `binfec`
 * (/root/reference/pkg/src/binfec, pure Python): every function cites the
 * reference file:line it follows.  Only tests/, __graft_entry__.smoke() and
 * bench.py (its cpu_baseline leg and the `--impl reference` arm) may load the
 * compiled oracle; the product library (liblch.so) never links or calls it.
 *
 * Parity pin: the oracle is checked against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py imports /root/reference in the
 * build container) and against the reference's own known-answer values
 * (tests/test_oracle_golden.py).
 */
#ifndef LCH_ORACLE_H
#define LCH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_EINVAL -1          /* ValueError in the reference */
#define ORC_ETOOMANY -2        /* TooManyErasuresError */
#define ORC_ENOTPRIM -3        /* non-primitive / reducible polynomial */
#define ORC_ENOMEM -4

typedef struct orc_ctx orc_ctx;

/* field.py:100-135 + basis.py:34-91 + walsh.py:69-74: build every table. */
int orc_create(int r, uint32_t poly, uint32_t max_h, orc_ctx **out);
void orc_destroy(orc_ctx *c);

/* table export (copies); sizes: log[2^r], exp[2^r-1], w_hat[max_h-1] (level i
 * at offset max_h - (max_h >> i)), w_prime[r], b_prod[max_h], b_prod_inv[max_h],
 * fwht_log[2^r], w_on_basis[r*r], w_norm[r] */
void orc_tables(const orc_ctx *c, uint16_t *log, uint16_t *exp, uint16_t *w_hat,
                uint16_t *w_prime, uint16_t *b_prod, uint16_t *b_prod_inv,
                uint32_t *fwht_log, uint16_t *w_on_basis, uint16_t *w_norm);

uint32_t orc_mul(const orc_ctx *c, uint32_t a, uint32_t b);
uint32_t orc_eval_w_hat(const orc_ctx *c, int i, uint32_t x);

/* transform.py:102-175 (in place, length h, shift < 2^r). */
int orc_forward(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift);
int orc_inverse(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift);
/* derivative.py:46-77 */
int orc_derivative(const orc_ctx *c, const uint16_t *in, uint16_t *out, uint32_t h);
/* walsh.py:42-61 (in place, any modulus) */
int orc_fwht(uint32_t *data, uint32_t n, uint32_t modulus);
/* walsh.py:77-115: mixed[j] = log-domain locator value for every position;
 * erased is a 0/1 byte mask of length 2^r. */
int orc_locator_logs(const orc_ctx *c, const uint8_t *erased, uint32_t *mixed);

/* rs.py:85-96: codeword[n] = message || parity blocks */
int orc_encode(const orc_ctx *c, uint32_t k, const uint16_t *msg, uint16_t *codeword);
/* rs.py:99-149: out[k]; erased is a 0/1 byte mask of length n */
int orc_decode(const orc_ctx *c, uint32_t k, const uint16_t *received,
               const uint8_t *erased, uint16_t *out);

/* General k, composed from the reference primitives:
 * recover every erased position (rs.py:125-148 evaluated on all of E),
 * systematic encode = erasure-decode of E = [k, n), decode = positions [0, k). */
int orc_recover_all(const orc_ctx *c, const uint16_t *received, const uint8_t *erased,
                    uint16_t *full);
int orc_encode_any(const orc_ctx *c, uint32_t k, const uint16_t *msg, uint16_t *codeword);
int orc_decode_any(const orc_ctx *c, uint32_t k, const uint16_t *received,
                   const uint8_t *erased, uint16_t *out);

/* Batched drivers with a thread pool over codewords (CPU baseline). */
int orc_encode_batch(const orc_ctx *c, uint32_t k, const uint16_t *msg,
                     uint16_t *parity, int64_t batch, int nthreads);
int orc_decode_batch(const orc_ctx *c, uint32_t k, const uint16_t *received,
                     const uint8_t *erased, int shared_pattern, uint16_t *out,
                     int64_t batch, int nthreads);
int orc_encode_any_batch(const orc_ctx *c, uint32_t k, const uint16_t *msg,
                         uint16_t *parity, int64_t batch, int nthreads);
int orc_decode_any_batch(const orc_ctx *c, uint32_t k, const uint16_t *received,
                         const uint8_t *erased, int shared_pattern, uint16_t *out,
                         int64_t batch, int nthreads);
int orc_transform_batch(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift,
                        int inverse, int64_t batch, int nthreads);

/* Seeded counter-based inputs (identical on the GPU, csrc/lch_gen.cu). */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_key(uint64_t seed, uint64_t cw, uint64_t pos);
void orc_gen_symbols(uint64_t seed, int r, uint64_t cw0, int64_t ncw, uint32_t len,
                     uint16_t *out);
/* erased[cw][pos] = 1 for the `count` positions with the smallest
 * (orc_key(seed, cw, pos) >> 1, pos); cw index = cw0 + row (or 0 for shared). */
void orc_gen_erasures(uint64_t seed, uint32_t n, uint32_t count, uint64_t cw0,
                      int64_t ncw, uint8_t *erased);

#ifdef __cplusplus
}
#endif
#endif
