/*
 * lch_oracle.c -- CPU restatement of the reference `binfec` hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see lch_oracle.h).  Loaded by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py for the CPU
 * baseline / reference arm.  Never linked into liblch.so.
 *
 * Citations "file.py:N" refer to /root/reference/pkg/src/binfec/file.py.
 */
#include "lch_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

struct orc_ctx {
    int r;
    uint32_t poly, order, m; /* m = 2^r - 1 (field.py:66-67) */
    uint32_t max_h;
    int levels;
    uint16_t *log, *exp;     /* field.py:56-69 */
    uint16_t w_on_basis[16][16];
    uint16_t w_norm[16], inv_norm[16];
    uint16_t *w_hat;         /* flat; level i at w_hat_off[i] */
    uint32_t w_hat_off[17];
    uint16_t w_prime[16];
    uint16_t *b_prod, *b_prod_inv;
    uint32_t *fwht_log;      /* walsh.py:64-74 (cached FWHT of the log table) */
};

/* field.py:138-150 (_mul_slow): carry-less multiply reduced bit by bit. */
static uint32_t mul_slow(uint32_t a, uint32_t b, uint32_t poly, int r) {
    uint32_t top = 1u << r, p = 0;
    while (b) {
        if (b & 1) p ^= a;
        b >>= 1;
        a <<= 1;
        if (a & top) a ^= poly;
    }
    return p;
}

/* field.py:75-79 */
uint32_t orc_mul(const orc_ctx *c, uint32_t a, uint32_t b) {
    if (a == 0 || b == 0) return 0;
    return c->exp[((uint32_t)c->log[a] + c->log[b]) % c->m];
}

/* field.py:81-85 (caller guarantees a != 0) */
static uint32_t f_inv(const orc_ctx *c, uint32_t a) {
    return c->exp[(c->m - c->log[a]) % c->m];
}

/* basis.py:95-105: W_i(x) by linearity over the bits of x */
static uint32_t eval_w(const orc_ctx *c, int i, uint32_t x) {
    uint32_t acc = 0;
    for (int b = 0; x; ++b, x >>= 1)
        if (x & 1) acc ^= c->w_on_basis[i][b];
    return acc;
}

/* basis.py:107-109 */
uint32_t orc_eval_w_hat(const orc_ctx *c, int i, uint32_t x) {
    return orc_mul(c, eval_w(c, i, x), c->inv_norm[i]);
}

int orc_fwht(uint32_t *data, uint32_t n, uint32_t modulus) {
    /* walsh.py:42-61: (x, y) -> ((x+y) mod q, (x-y) mod q), levels ascending */
    if (n & (n - 1)) return ORC_EINVAL;
    for (uint32_t half = 1; half < n; half <<= 1) {
        uint32_t step = half << 1;
        for (uint32_t cst = 0; cst < n; cst += step)
            for (uint32_t j = cst; j < cst + half; ++j) {
                uint64_t x = data[j], y = data[j + half];
                data[j] = (uint32_t)((x + y) % modulus);
                data[j + half] = (uint32_t)((x + modulus - (y % modulus)) % modulus);
            }
    }
    return ORC_OK;
}

int orc_create(int r, uint32_t poly, uint32_t max_h, orc_ctx **out) {
    *out = NULL;
    /* field.py:41-49 (FieldParams validation) */
    if (r != 8 && r != 16) return ORC_EINVAL;
    if ((poly >> r) != 1) return ORC_EINVAL; /* bit_length must be r + 1 */
    /* basis.py:35-38 */
    if (max_h < 1 || (max_h & (max_h - 1)) || max_h > (1u << r)) return ORC_EINVAL;

    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    if (!c) return ORC_ENOMEM;
    c->r = r;
    c->poly = poly;
    c->order = 1u << r;
    c->m = c->order - 1;
    c->max_h = max_h;
    c->levels = 0;
    while ((1u << c->levels) < max_h) c->levels++;
    c->log = (uint16_t *)malloc(sizeof(uint16_t) * c->order);
    c->exp = (uint16_t *)malloc(sizeof(uint16_t) * c->order);
    c->w_hat = (uint16_t *)malloc(sizeof(uint16_t) * (max_h > 1 ? max_h - 1 : 1));
    c->b_prod = (uint16_t *)malloc(sizeof(uint16_t) * max_h);
    c->b_prod_inv = (uint16_t *)malloc(sizeof(uint16_t) * max_h);
    c->fwht_log = (uint32_t *)malloc(sizeof(uint32_t) * c->order);
    if (!c->log || !c->exp || !c->w_hat || !c->b_prod || !c->b_prod_inv || !c->fwht_log) {
        orc_destroy(c);
        return ORC_ENOMEM;
    }

    /* field.py:100-129: powers of alpha = x (index 2), primitivity check */
    int32_t *lg = (int32_t *)malloc(sizeof(int32_t) * c->order);
    if (!lg) { orc_destroy(c); return ORC_ENOMEM; }
    for (uint32_t i = 0; i < c->order; ++i) lg[i] = -1;
    uint32_t val = 1;
    for (uint32_t i = 0; i < c->m; ++i) {
        if (lg[val] != -1) { free(lg); orc_destroy(c); return ORC_ENOTPRIM; }
        c->exp[i] = (uint16_t)val;
        lg[val] = (int32_t)i;
        val = mul_slow(val, 2, poly, r);
    }
    if (val != 1) { free(lg); orc_destroy(c); return ORC_ENOTPRIM; }
    lg[0] = 0; /* field.py:128 */
    for (uint32_t i = 0; i < c->order; ++i) c->log[i] = (uint16_t)lg[i];
    c->exp[c->m] = 1; /* padding entry, never read by the reference indices */
    free(lg);

    /* basis.py:46-53: w_on_basis rows via W_{i+1}(x) = W_i(x)(W_i(x) + W_i(v_i)) */
    for (int b = 0; b < r; ++b) c->w_on_basis[0][b] = (uint16_t)(1u << b);
    for (int i = 0; i + 1 < r; ++i) {
        uint32_t nrm = c->w_on_basis[i][i];
        for (int b = 0; b < r; ++b) {
            uint32_t t = c->w_on_basis[i][b];
            c->w_on_basis[i + 1][b] = (uint16_t)orc_mul(c, t, t ^ nrm);
        }
    }
    /* basis.py:57-61 */
    for (int i = 0; i < r; ++i) {
        c->w_norm[i] = c->w_on_basis[i][i];
        if (c->w_norm[i] == 0) { orc_destroy(c); return ORC_EINVAL; }
        c->inv_norm[i] = (uint16_t)f_inv(c, c->w_norm[i]);
    }
    /* basis.py:63-69: w_hat[i][b] = W^_i(b * 2^(i+1)), h-1 entries in total */
    uint32_t off = 0;
    for (int i = 0; i < c->levels; ++i) {
        c->w_hat_off[i] = off;
        uint32_t cnt = max_h >> (i + 1);
        for (uint32_t b = 0; b < cnt; ++b)
            c->w_hat[off + b] = (uint16_t)orc_eval_w_hat(c, i, b << (i + 1));
        off += cnt;
    }
    c->w_hat_off[c->levels] = off;
    /* basis.py:71-82: W'_l from the running log-sum of elements 1..2^l-1 */
    uint64_t acc = 0;
    for (int l = 0; l < r; ++l) {
        c->w_prime[l] = (uint16_t)orc_mul(c, c->exp[acc % c->m], c->inv_norm[l]);
        if (l < r - 1)
            for (uint32_t j = 1u << l; j < (1u << (l + 1)); ++j) acc += c->log[j];
    }
    /* basis.py:84-91: subset products over the set bits */
    c->b_prod[0] = 1;
    for (uint32_t i = 1; i < max_h; ++i) {
        uint32_t low = i & (~i + 1);
        c->b_prod[i] = (uint16_t)orc_mul(c, c->b_prod[i ^ low], c->w_prime[__builtin_ctz(low)]);
    }
    for (uint32_t i = 0; i < max_h; ++i) c->b_prod_inv[i] = (uint16_t)f_inv(c, c->b_prod[i]);
    /* walsh.py:69-74: FWHT of the log table mod 2^r - 1 */
    for (uint32_t i = 0; i < c->order; ++i) c->fwht_log[i] = c->log[i];
    orc_fwht(c->fwht_log, c->order, c->m);

    *out = c;
    return ORC_OK;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    free(c->log); free(c->exp); free(c->w_hat); free(c->b_prod);
    free(c->b_prod_inv); free(c->fwht_log);
    free(c);
}

void orc_tables(const orc_ctx *c, uint16_t *log, uint16_t *exp, uint16_t *w_hat,
                uint16_t *w_prime, uint16_t *b_prod, uint16_t *b_prod_inv,
                uint32_t *fwht_log, uint16_t *w_on_basis, uint16_t *w_norm) {
    if (log) memcpy(log, c->log, sizeof(uint16_t) * c->order);
    if (exp) memcpy(exp, c->exp, sizeof(uint16_t) * c->m);
    if (w_hat && c->max_h > 1) memcpy(w_hat, c->w_hat, sizeof(uint16_t) * (c->max_h - 1));
    if (w_prime) memcpy(w_prime, c->w_prime, sizeof(uint16_t) * c->r);
    if (b_prod) memcpy(b_prod, c->b_prod, sizeof(uint16_t) * c->max_h);
    if (b_prod_inv) memcpy(b_prod_inv, c->b_prod_inv, sizeof(uint16_t) * c->max_h);
    if (fwht_log) memcpy(fwht_log, c->fwht_log, sizeof(uint32_t) * c->order);
    if (w_on_basis)
        for (int i = 0; i < c->r; ++i)
            for (int b = 0; b < c->r; ++b) w_on_basis[i * c->r + b] = c->w_on_basis[i][b];
    if (w_norm) memcpy(w_norm, c->w_norm, sizeof(uint16_t) * c->r);
}

/* transform.py:60-66 */
static int check_size(const orc_ctx *c, uint32_t h, uint32_t shift) {
    if (h < 1 || (h & (h - 1))) return ORC_EINVAL;
    if (h > c->max_h) return ORC_EINVAL;
    if (shift >= c->order) return ORC_EINVAL;
    return ORC_OK;
}

static int lg2(uint32_t h) { int l = 0; while ((1u << l) < h) ++l; return l; }

/* transform.py:102-140: levels lg h - 1 .. 0, (u, v) -> (u + f v, u + f v + v) */
int orc_forward(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift) {
    int rc = check_size(c, h, shift);
    if (rc) return rc;
    int levels = lg2(h);
    for (int i = levels - 1; i >= 0; --i) {
        uint32_t half = 1u << i, step = half << 1;
        const uint16_t *hat = c->w_hat + c->w_hat_off[i];
        uint32_t hat_shift = shift ? orc_eval_w_hat(c, i, shift) : 0;
        int64_t zero_c = (shift < h && !(shift & (step - 1))) ? (int64_t)shift : -1;
        for (uint32_t cst = 0; cst < h; cst += step) {
            if ((int64_t)cst == zero_c) {
                for (uint32_t j = cst; j < cst + half; ++j) a[j + half] ^= a[j];
                continue;
            }
            uint32_t f = hat[cst >> (i + 1)] ^ hat_shift;
            if (f) {
                uint32_t lf = c->log[f];
                for (uint32_t j = cst; j < cst + half; ++j) {
                    uint32_t v = a[j + half], u;
                    if (v) {
                        u = a[j] ^ c->exp[(c->log[v] + lf) % c->m];
                        a[j] = (uint16_t)u;
                    } else {
                        u = a[j];
                    }
                    a[j + half] = (uint16_t)(u ^ v);
                }
            } else {
                for (uint32_t j = cst; j < cst + half; ++j) a[j + half] ^= a[j];
            }
        }
    }
    return ORC_OK;
}

/* transform.py:143-175: levels 0 .. lg h - 1, v <- u + v, u <- u + f v */
int orc_inverse(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift) {
    int rc = check_size(c, h, shift);
    if (rc) return rc;
    int levels = lg2(h);
    for (int i = 0; i < levels; ++i) {
        uint32_t half = 1u << i, step = half << 1;
        const uint16_t *hat = c->w_hat + c->w_hat_off[i];
        uint32_t hat_shift = shift ? orc_eval_w_hat(c, i, shift) : 0;
        int64_t zero_c = (shift < h && !(shift & (step - 1))) ? (int64_t)shift : -1;
        for (uint32_t cst = 0; cst < h; cst += step) {
            if ((int64_t)cst == zero_c) {
                for (uint32_t j = cst; j < cst + half; ++j) a[j + half] ^= a[j];
                continue;
            }
            uint32_t f = hat[cst >> (i + 1)] ^ hat_shift;
            if (f) {
                uint32_t lf = c->log[f];
                for (uint32_t j = cst; j < cst + half; ++j) {
                    uint32_t v = a[j] ^ a[j + half];
                    a[j + half] = (uint16_t)v;
                    if (v) a[j] ^= c->exp[(c->log[v] + lf) % c->m];
                }
            } else {
                for (uint32_t j = cst; j < cst + half; ++j) a[j + half] ^= a[j];
            }
        }
    }
    return ORC_OK;
}

/* derivative.py:46-77: scale by B_i, gather-XOR over the zero bits, scale by B_j^-1 */
int orc_derivative(const orc_ctx *c, const uint16_t *in, uint16_t *out, uint32_t h) {
    if (h < 1 || (h & (h - 1)) || h > c->max_h) return ORC_EINVAL;
    int levels = lg2(h);
    uint16_t *scaled = (uint16_t *)malloc(sizeof(uint16_t) * h);
    if (!scaled) return ORC_ENOMEM;
    for (uint32_t i = 0; i < h; ++i) scaled[i] = (uint16_t)orc_mul(c, in[i], c->b_prod[i]);
    /* the gather in the batch codec's order (batch.py:101-106): one pass per
     * level l over the destinations j with bit l clear, acc[j] ^= scaled[j + 2^l]
     * (derivative.py:60-70 sums the same terms per j) */
    memset(out, 0, sizeof(uint16_t) * h);
    for (int l = 0; l < levels; ++l) {
        uint32_t step = 1u << l;
        for (uint32_t blk = 0; blk < h; blk += 2 * step)
            for (uint32_t j = blk; j < blk + step; ++j) out[j] ^= scaled[j + step];
    }
    for (uint32_t j = 0; j < h; ++j)
        out[j] = out[j] ? (uint16_t)orc_mul(c, out[j], c->b_prod_inv[j]) : 0;
    free(scaled);
    return ORC_OK;
}

/* walsh.py:77-115: indicator FWHT, pointwise product with FWHT(log), FWHT */
int orc_locator_logs(const orc_ctx *c, const uint8_t *erased, uint32_t *mixed) {
    uint32_t n = c->order, cnt = 0;
    for (uint32_t j = 0; j < n; ++j) cnt += erased[j] ? 1 : 0;
    if (cnt == 0) return ORC_EINVAL;        /* walsh.py:85-86 */
    if (cnt > n - 1) return ORC_EINVAL;     /* walsh.py:92-93 */
    for (uint32_t j = 0; j < n; ++j) mixed[j] = erased[j] ? 1 : 0;
    orc_fwht(mixed, n, c->m);
    for (uint32_t j = 0; j < n; ++j)
        mixed[j] = (uint32_t)(((uint64_t)mixed[j] * c->fwht_log[j]) % c->m);
    orc_fwht(mixed, n, c->m);
    return ORC_OK;
}

/* rs.py:85-96 (+ rs.py:159-163 table checks) */
int orc_encode(const orc_ctx *c, uint32_t k, const uint16_t *msg, uint16_t *codeword) {
    uint32_t n = c->order;
    if (k < 1 || (k & (k - 1)) || k > n) return ORC_EINVAL; /* rs.py:41-46 */
    if (c->max_h < k) return ORC_EINVAL;                     /* rs.py:162-163 */
    uint16_t *coeffs = (uint16_t *)malloc(sizeof(uint16_t) * k);
    if (!coeffs) return ORC_ENOMEM;
    memcpy(coeffs, msg, sizeof(uint16_t) * k);
    int rc = orc_inverse(c, coeffs, k, 0);
    if (rc) { free(coeffs); return rc; }
    memcpy(codeword, msg, sizeof(uint16_t) * k);
    for (uint32_t i = 1; i < n / k; ++i) {
        uint16_t *blk = codeword + (size_t)i * k;
        memcpy(blk, coeffs, sizeof(uint16_t) * k);
        rc = orc_forward(c, blk, k, i * k);
        if (rc) break;
    }
    free(coeffs);
    return rc;
}

/* rs.py:99-149.  shared_logs (optional): the locator residues of this erasure
 * pattern evaluated by the caller -- BatchCodec.decode evaluates the locator
 * once per shared erasure set (batch.py:126-139), not once per row. */
static int decode_with_logs(const orc_ctx *c, uint32_t k, const uint16_t *received,
                            const uint8_t *erased, const uint32_t *shared_logs, uint16_t *out) {
    uint32_t n = c->order;
    if (k < 1 || (k & (k - 1)) || k > n) return ORC_EINVAL;
    if (c->max_h < k) return ORC_EINVAL;
    uint32_t cnt = 0;
    for (uint32_t j = 0; j < n; ++j) cnt += erased[j] ? 1 : 0;
    if (cnt == 0) { memcpy(out, received, sizeof(uint16_t) * k); return ORC_OK; } /* rs.py:119-120 */
    if (cnt > n - k) return ORC_ETOOMANY;                                          /* rs.py:121-123 */
    if (c->max_h < n) return ORC_EINVAL; /* n-point inverse needs the capacity (transform.py:63-64) */
    uint32_t *own = shared_logs ? NULL : (uint32_t *)malloc(sizeof(uint32_t) * n);
    const uint32_t *mixed = shared_logs ? shared_logs : own;
    uint16_t *phi = (uint16_t *)malloc(sizeof(uint16_t) * n);
    uint16_t *dc = (uint16_t *)malloc(sizeof(uint16_t) * n);
    if (!mixed || !phi || !dc) { free(own); free(phi); free(dc); return ORC_ENOMEM; }
    int rc = own ? orc_locator_logs(c, erased, own) : ORC_OK;
    if (!rc) {
        /* rs.py:130-134: phi = received * pi_bar on survivors, 0 on erasures */
        for (uint32_t j = 0; j < n; ++j)
            phi[j] = erased[j] ? 0 : (uint16_t)orc_mul(c, received[j], c->exp[mixed[j]]);
        rc = orc_inverse(c, phi, n, 0);                    /* rs.py:136 */
        if (!rc) rc = orc_derivative(c, phi, dc, n);       /* rs.py:137 */
        if (!rc) rc = orc_forward(c, dc, n, 0);            /* rs.py:138 */
        if (!rc) {
            memcpy(out, received, sizeof(uint16_t) * k);   /* rs.py:140 */
            for (uint32_t j = 0; j < k; ++j) {
                if (!erased[j]) continue;
                uint32_t prime = c->exp[mixed[j]];
                out[j] = (uint16_t)orc_mul(c, dc[j], f_inv(c, prime)); /* rs.py:141-148 */
            }
        }
    }
    free(own); free(phi); free(dc);
    return rc;
}

int orc_decode(const orc_ctx *c, uint32_t k, const uint16_t *received,
               const uint8_t *erased, uint16_t *out) {
    return decode_with_logs(c, k, received, erased, NULL, out);
}

/* General k: the reference's decode algorithm (rs.py:125-148)
 * without the power-of-two restriction of rs.py:43-44, evaluated at every
 * erased position.  full[n] = received with each erased j replaced by
 * Phi^d(j) / Pi'(j).  Phi = f * Pi has degree < k + |E| <= n, so the n-point
 * transforms recover f at the erasures for any k. */
static int recover_all_with_logs(const orc_ctx *c, const uint16_t *received, const uint8_t *erased,
                                 const uint32_t *shared_logs, uint16_t *full) {
    uint32_t n = c->order;
    if (c->max_h < n) return ORC_EINVAL;
    uint32_t cnt = 0;
    for (uint32_t j = 0; j < n; ++j) cnt += erased[j] ? 1 : 0;
    memcpy(full, received, sizeof(uint16_t) * n);
    if (cnt == 0) return ORC_OK;
    if (cnt == n) return ORC_EINVAL; /* walsh.py:92-93: at least one survivor */
    uint32_t *own = shared_logs ? NULL : (uint32_t *)malloc(sizeof(uint32_t) * n);
    const uint32_t *mixed = shared_logs ? shared_logs : own;
    uint16_t *phi = (uint16_t *)malloc(sizeof(uint16_t) * n);
    uint16_t *dc = (uint16_t *)malloc(sizeof(uint16_t) * n);
    if (!mixed || !phi || !dc) { free(own); free(phi); free(dc); return ORC_ENOMEM; }
    int rc = own ? orc_locator_logs(c, erased, own) : ORC_OK;
    if (!rc) {
        for (uint32_t j = 0; j < n; ++j)
            phi[j] = erased[j] ? 0 : (uint16_t)orc_mul(c, received[j], c->exp[mixed[j]]);
        rc = orc_inverse(c, phi, n, 0);
        if (!rc) rc = orc_derivative(c, phi, dc, n);
        if (!rc) rc = orc_forward(c, dc, n, 0);
        if (!rc)
            for (uint32_t j = 0; j < n; ++j)
                if (erased[j]) full[j] = (uint16_t)orc_mul(c, dc[j], f_inv(c, c->exp[mixed[j]]));
    }
    free(own); free(phi); free(dc);
    return rc;
}

int orc_recover_all(const orc_ctx *c, const uint16_t *received, const uint8_t *erased,
                    uint16_t *full) {
    return recover_all_with_logs(c, received, erased, NULL, full);
}

/* Systematic encode for any 1 <= k <= n: erasure-decode E = [k, n) from the
 * message (fact iii: equals orc_encode for power-of-two k). */
int orc_encode_any(const orc_ctx *c, uint32_t k, const uint16_t *msg, uint16_t *codeword) {
    uint32_t n = c->order;
    if (k < 1 || k > n) return ORC_EINVAL;
    uint16_t *rx = (uint16_t *)calloc(n, sizeof(uint16_t));
    uint8_t *e = (uint8_t *)calloc(n, 1);
    if (!rx || !e) { free(rx); free(e); return ORC_ENOMEM; }
    memcpy(rx, msg, sizeof(uint16_t) * k);
    for (uint32_t j = k; j < n; ++j) e[j] = 1;
    int rc = orc_recover_all(c, rx, e, codeword);
    free(rx); free(e);
    return rc;
}

/* Decode for any 1 <= k <= n: out[k] = positions [0, k) of the recovered word. */
static int decode_any_with_logs(const orc_ctx *c, uint32_t k, const uint16_t *received,
                                const uint8_t *erased, const uint32_t *shared_logs, uint16_t *out) {
    uint32_t n = c->order;
    if (k < 1 || k > n) return ORC_EINVAL;
    uint32_t cnt = 0;
    for (uint32_t j = 0; j < n; ++j) cnt += erased[j] ? 1 : 0;
    if (cnt > n - k) return ORC_ETOOMANY;
    uint16_t *full = (uint16_t *)malloc(sizeof(uint16_t) * n);
    if (!full) return ORC_ENOMEM;
    int rc = recover_all_with_logs(c, received, erased, shared_logs, full);
    if (!rc) memcpy(out, full, sizeof(uint16_t) * k);
    free(full);
    return rc;
}

int orc_decode_any(const orc_ctx *c, uint32_t k, const uint16_t *received,
                   const uint8_t *erased, uint16_t *out) {
    return decode_any_with_logs(c, k, received, erased, NULL, out);
}

/* ------------------------------------------------------------------------ */
/* batched drivers (thread pool over codewords)                              */

typedef struct {
    const orc_ctx *c;
    int op;                 /* 0 encode, 1 decode, 2 transform */
    uint32_t k, h, shift;
    int inverse, shared;
    const uint16_t *in;
    uint16_t *out;
    uint16_t *inout;
    const uint8_t *erased;
    const uint32_t *shared_logs; /* op 1, shared pattern: locator residues of the batch */
    int64_t begin, end;
    int rc;
} job_t;

static void *run_job(void *arg) {
    job_t *j = (job_t *)arg;
    const orc_ctx *c = j->c;
    uint32_t n = c->order;
    j->rc = ORC_OK;
    uint16_t *cw = NULL;
    if (j->op == 0 || j->op == 3) cw = (uint16_t *)malloc(sizeof(uint16_t) * n);
    for (int64_t b = j->begin; b < j->end && j->rc == ORC_OK; ++b) {
        if (j->op == 0) {
            j->rc = orc_encode(c, j->k, j->in + b * j->k, cw);
            memcpy(j->out + b * (int64_t)(n - j->k), cw + j->k, sizeof(uint16_t) * (n - j->k));
        } else if (j->op == 3) {
            j->rc = orc_encode_any(c, j->k, j->in + b * j->k, cw);
            memcpy(j->out + b * (int64_t)(n - j->k), cw + j->k, sizeof(uint16_t) * (n - j->k));
        } else if (j->op == 1 || j->op == 4) {
            const uint8_t *e = j->erased + (j->shared ? 0 : b * (int64_t)n);
            j->rc = j->op == 1 ? decode_with_logs(c, j->k, j->in + b * (int64_t)n, e, j->shared_logs,
                                                  j->out + b * j->k)
                               : decode_any_with_logs(c, j->k, j->in + b * (int64_t)n, e, j->shared_logs,
                                                      j->out + b * j->k);
        } else {
            uint16_t *a = j->inout + b * (int64_t)j->h;
            j->rc = j->inverse ? orc_inverse(c, a, j->h, j->shift) : orc_forward(c, a, j->h, j->shift);
        }
    }
    free(cw);
    return NULL;
}

static int run_pool(job_t proto, int64_t batch, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    if (batch < nthreads) nthreads = (int)(batch > 0 ? batch : 1);
    pthread_t th[512];
    job_t jobs[512];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].begin = batch * t / nthreads;
        jobs[t].end = batch * (t + 1) / nthreads;
        if (nthreads == 1) run_job(&jobs[t]);
        else pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    int rc = ORC_OK;
    for (int t = 0; t < nthreads; ++t) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    return rc;
}

/* Decode drivers.  One shared erasure set: the locator runs once for the
 * batch, as BatchCodec.decode does (batch.py:126-139); degenerate erasure
 * counts keep the per-row checks. */
static int run_decode_pool(job_t p, int64_t batch, int nthreads) {
    uint32_t *logs = NULL;
    if (p.shared && batch > 1) {
        uint32_t n = p.c->order, cnt = 0;
        for (uint32_t j = 0; j < n; ++j) cnt += p.erased[j] ? 1 : 0;
        if (cnt > 0 && cnt < n && cnt <= n - p.k && p.k >= 1 && p.k <= n) {
            logs = (uint32_t *)malloc(sizeof(uint32_t) * n);
            if (!logs) return ORC_ENOMEM;
            int rc = orc_locator_logs(p.c, p.erased, logs);
            if (rc) { free(logs); return rc; }
            p.shared_logs = logs;
        }
    }
    int rc = run_pool(p, batch, nthreads);
    free(logs);
    return rc;
}

int orc_encode_batch(const orc_ctx *c, uint32_t k, const uint16_t *msg,
                     uint16_t *parity, int64_t batch, int nthreads) {
    job_t p;
    memset(&p, 0, sizeof(p));
    p.c = c; p.op = 0; p.k = k; p.in = msg; p.out = parity;
    return run_pool(p, batch, nthreads);
}

int orc_decode_batch(const orc_ctx *c, uint32_t k, const uint16_t *received,
                     const uint8_t *erased, int shared_pattern, uint16_t *out,
                     int64_t batch, int nthreads) {
    job_t p;
    memset(&p, 0, sizeof(p));
    p.c = c; p.op = 1; p.k = k; p.in = received; p.out = out;
    p.erased = erased; p.shared = shared_pattern;
    return run_decode_pool(p, batch, nthreads);
}

int orc_encode_any_batch(const orc_ctx *c, uint32_t k, const uint16_t *msg,
                         uint16_t *parity, int64_t batch, int nthreads) {
    job_t p;
    memset(&p, 0, sizeof(p));
    p.c = c; p.op = 3; p.k = k; p.in = msg; p.out = parity;
    return run_pool(p, batch, nthreads);
}

int orc_decode_any_batch(const orc_ctx *c, uint32_t k, const uint16_t *received,
                         const uint8_t *erased, int shared_pattern, uint16_t *out,
                         int64_t batch, int nthreads) {
    job_t p;
    memset(&p, 0, sizeof(p));
    p.c = c; p.op = 4; p.k = k; p.in = received; p.out = out;
    p.erased = erased; p.shared = shared_pattern;
    return run_decode_pool(p, batch, nthreads);
}

int orc_transform_batch(const orc_ctx *c, uint16_t *a, uint32_t h, uint32_t shift,
                        int inverse, int64_t batch, int nthreads) {
    job_t p;
    memset(&p, 0, sizeof(p));
    p.c = c; p.op = 2; p.h = h; p.shift = shift; p.inverse = inverse; p.inout = a;
    return run_pool(p, batch, nthreads);
}

/* ------------------------------------------------------------------------ */
/* seeded inputs; mirrored bit-for-bit by csrc/lch_gen.cu        */

#define GAMMA 0x9E3779B97F4A7C15ull

uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_key(uint64_t seed, uint64_t cw, uint64_t pos) {
    uint64_t s = orc_mix64(seed + GAMMA);
    return orc_mix64(s + ((cw << 32) | pos) * GAMMA);
}

void orc_gen_symbols(uint64_t seed, int r, uint64_t cw0, int64_t ncw, uint32_t len,
                     uint16_t *out) {
    uint64_t mask = (1ull << r) - 1;
    for (int64_t b = 0; b < ncw; ++b)
        for (uint32_t j = 0; j < len; ++j)
            out[b * (int64_t)len + j] = (uint16_t)(orc_key(seed, cw0 + (uint64_t)b, j) & mask);
}

typedef struct { uint64_t key; uint32_t pos; } kp_t;

static int kp_cmp(const void *a, const void *b) {
    const kp_t *x = (const kp_t *)a, *y = (const kp_t *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

void orc_gen_erasures(uint64_t seed, uint32_t n, uint32_t count, uint64_t cw0,
                      int64_t ncw, uint8_t *erased) {
    kp_t *kp = (kp_t *)malloc(sizeof(kp_t) * n);
    for (int64_t b = 0; b < ncw; ++b) {
        uint8_t *e = erased + b * (int64_t)n;
        for (uint32_t j = 0; j < n; ++j) {
            kp[j].key = orc_key(seed, cw0 + (uint64_t)b, j) >> 1;
            kp[j].pos = j;
        }
        qsort(kp, n, sizeof(kp_t), kp_cmp);
        memset(e, 0, n);
        for (uint32_t t = 0; t < count && t < n; ++t) e[kp[t].pos] = 1;
    }
    free(kp);
}
