// Host-side field + basis tables for the LCH transform (product code).
//
// Restated from the reference's definitions (not from the oracle):
//   field.py:100-135  log/exp by powers of alpha = x, primitivity check
//   basis.py:34-109   W_i on the basis, normalisers, w_hat factors (h-1 total),
//                     W'_l, subset products B_i and inverses
//   walsh.py:64-74    FWHT of the log table mod 2^r - 1
#pragma once

#include <cstdint>
#include <vector>

namespace lch {

struct Tables {
  int r = 0;
  uint32_t poly = 0;
  uint32_t alpha = 2;    // generator the log/exp tables are built from (field.py:31-39)
  uint32_t order = 0;   // 2^r
  uint32_t m = 0;       // 2^r - 1
  uint32_t max_h = 0;
  int levels = 0;       // lg max_h
  std::vector<uint16_t> log;        // [order], log[0] = 0
  std::vector<uint16_t> exp;        // [order]; exp[m] = exp[0] = 1 (wrap entry)
  std::vector<uint16_t> w_on_basis; // [r*r]
  std::vector<uint16_t> w_norm;     // [r]
  std::vector<uint16_t> inv_norm;   // [r]
  std::vector<uint16_t> w_hat;      // [max_h - 1], level i at w_hat_off[i]
  std::vector<uint32_t> w_hat_off;  // [levels + 1]
  std::vector<uint16_t> w_prime;    // [r]
  std::vector<uint16_t> b_prod;     // [max_h]
  std::vector<uint16_t> b_prod_inv; // [max_h]
  std::vector<uint32_t> fwht_log;   // [order]

  uint32_t mul(uint32_t a, uint32_t b) const {
    if (!a || !b) return 0;
    return exp[(uint32_t(log[a]) + log[b]) % m];
  }
  uint32_t inv(uint32_t a) const { return exp[(m - log[a]) % m]; }
  uint32_t eval_w(int i, uint32_t x) const;
  uint32_t eval_w_hat(int i, uint32_t x) const { return mul(eval_w(i, x), inv_norm[i]); }
};

// Returns 0 or a negative LCH_E* code (lch.h).
int build_tables(int r, uint32_t poly, uint32_t max_h, Tables &t, uint32_t alpha = 2);

// In-place FWHT over Z_mod (host helper used for the cached FWHT(log)).
void fwht_host(std::vector<uint32_t> &a, uint32_t mod);

}  // namespace lch
