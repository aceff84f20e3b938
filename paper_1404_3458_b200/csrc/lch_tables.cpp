// Host-side table construction (see lch_tables.h for the reference citations).
#include "lch_tables.h"

#include "../../include/lch.h"

namespace lch {

namespace {
// Shift-and-xor product reduced by the field polynomial; only used while the
// log/exp tables are being generated (field.py:138-150 plays the same role).
uint32_t clmul_reduce(uint32_t a, uint32_t b, uint32_t poly, int r) {
  const uint32_t top = 1u << r;
  uint32_t acc = 0;
  for (; b; b >>= 1) {
    if (b & 1) acc ^= a;
    a <<= 1;
    if (a & top) a ^= poly;
  }
  return acc;
}
}  // namespace

uint32_t Tables::eval_w(int i, uint32_t x) const {
  // W_i is F_2-linear (basis.py:95-105): XOR of W_i(v_b) over the set bits of x
  uint32_t acc = 0;
  for (int b = 0; x; ++b, x >>= 1)
    if (x & 1) acc ^= w_on_basis[i * r + b];
  return acc;
}

void fwht_host(std::vector<uint32_t> &a, uint32_t mod) {
  const size_t n = a.size();
  for (size_t half = 1; half < n; half <<= 1)
    for (size_t c = 0; c < n; c += 2 * half)
      for (size_t j = c; j < c + half; ++j) {
        const uint64_t x = a[j] % mod, y = a[j + half] % mod;
        a[j] = uint32_t((x + y) % mod);
        a[j + half] = uint32_t((x + mod - y) % mod);
      }
}

int build_tables(int r, uint32_t poly, uint32_t max_h, Tables &t, uint32_t alpha) {
  if (r != 8 && r != 16) return LCH_EINVAL;               // field.py:42-43
  if ((poly >> r) != 1u) return LCH_EINVAL;               // degree check, field.py:44-47
  if (max_h < 1 || (max_h & (max_h - 1)) || max_h > (1u << r)) return LCH_EINVAL;  // basis.py:35-38
  if (alpha == 0 || alpha >= (1u << r)) return LCH_EINVAL;                            // field.py:48-49

  t.r = r;
  t.poly = poly;
  t.alpha = alpha;
  t.order = 1u << r;
  t.m = t.order - 1;
  t.max_h = max_h;
  t.levels = 0;
  while ((1u << t.levels) < max_h) ++t.levels;

  // log/exp: walk the powers of alpha (x by default); a repeat before 2^r - 1
  // steps (or not returning to 1) means alpha does not generate the group
  // (polynomial not primitive, or alpha not a generator; field.py:116-133).
  t.log.assign(t.order, 0);
  t.exp.assign(t.order, 0);
  std::vector<uint8_t> seen(t.order, 0);
  uint32_t val = 1;
  for (uint32_t e = 0; e < t.m; ++e) {
    if (seen[val]) return LCH_ENOTPRIM;
    seen[val] = 1;
    t.exp[e] = uint16_t(val);
    t.log[val] = uint16_t(e);
    val = clmul_reduce(val, alpha, poly, r);
  }
  if (val != 1) return LCH_ENOTPRIM;
  t.log[0] = 0;        // log(0) := 0 convention; zero operands are branched on
  t.exp[t.m] = 1;      // alpha^m = 1: lets device code index exp[s] for s <= m

  // W_i(v_b): row 0 is the identity map, W_{i+1}(x) = W_i(x) (W_i(x) + W_i(v_i))
  t.w_on_basis.assign(size_t(r) * r, 0);
  for (int b = 0; b < r; ++b) t.w_on_basis[b] = uint16_t(1u << b);
  for (int i = 0; i + 1 < r; ++i) {
    const uint32_t nrm = t.w_on_basis[i * r + i];
    for (int b = 0; b < r; ++b) {
      const uint32_t w = t.w_on_basis[i * r + b];
      t.w_on_basis[(i + 1) * r + b] = uint16_t(t.mul(w, w ^ nrm));
    }
  }
  t.w_norm.resize(r);
  t.inv_norm.resize(r);
  for (int i = 0; i < r; ++i) {
    t.w_norm[i] = t.w_on_basis[i * r + i];
    if (!t.w_norm[i]) return LCH_EINVAL;
    t.inv_norm[i] = uint16_t(t.inv(t.w_norm[i]));
  }

  // butterfly factors for block starts: level i holds max_h >> (i+1) entries
  t.w_hat.assign(max_h > 1 ? max_h - 1 : 0, 0);
  t.w_hat_off.assign(t.levels + 1, 0);
  uint32_t off = 0;
  for (int i = 0; i < t.levels; ++i) {
    t.w_hat_off[i] = off;
    for (uint32_t b = 0; b < (max_h >> (i + 1)); ++b)
      t.w_hat[off + b] = uint16_t(t.eval_w_hat(i, b << (i + 1)));
    off += max_h >> (i + 1);
  }
  t.w_hat_off[t.levels] = off;

  // W'_l = (prod of nonzero elements below 2^l) / W_l(v_l), via a log-sum
  t.w_prime.resize(r);
  uint64_t logsum = 0;
  for (int l = 0; l < r; ++l) {
    t.w_prime[l] = uint16_t(t.mul(t.exp[logsum % t.m], t.inv_norm[l]));
    if (l + 1 < r)
      for (uint32_t j = 1u << l; j < (2u << l); ++j) logsum += t.log[j];
  }

  // B_i = prod over set bits j of i of W'_j, and inverses
  t.b_prod.assign(max_h, 1);
  t.b_prod_inv.assign(max_h, 1);
  for (uint32_t i = 1; i < max_h; ++i) {
    const uint32_t low = i & (0u - i);
    t.b_prod[i] = uint16_t(t.mul(t.b_prod[i ^ low], t.w_prime[__builtin_ctz(low)]));
  }
  for (uint32_t i = 0; i < max_h; ++i) t.b_prod_inv[i] = uint16_t(t.inv(t.b_prod[i]));

  // cached FWHT of the log table (log[0] = 0 entry included)
  t.fwht_log.assign(t.log.begin(), t.log.end());
  fwht_host(t.fwht_log, t.m);
  return LCH_OK;
}

}  // namespace lch
