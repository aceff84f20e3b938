"""Subspace vanishing polynomials and the LCH basis tables (drop-in for
binfec.basis, basis.py:1-137).

The tables come from the native builder (csrc/lch_tables.cpp, restating
basis.py:34-91); the GPU context that runs the transforms is owned here, one
per (field, max_h).
"""

from __future__ import annotations

from . import _lib
from .field import FieldTables


class BasisTables:
    """Precomputed factors for transforms up to max_h points (basis.py:31-109)."""

    def __init__(self, ft: FieldTables, max_h: int):
        if max_h < 1 or max_h & (max_h - 1):
            raise ValueError(f"max_h must be a power of two, got {max_h}")
        if max_h > ft.order:
            raise ValueError(f"max_h={max_h} exceeds field size {ft.order}")
        self.ft = ft
        self.max_h = max_h
        self.levels = max_h.bit_length() - 1
        r = ft.r
        self.ctx = _lib.Context(r, ft.params.reduction_poly, self.levels, ft.params.alpha_index)
        t = self.ctx.tables()
        self._np = t
        self.w_on_basis: list[list[int]] = [[int(x) for x in row] for row in t["w_on_basis"]]
        self.w_norm: list[int] = [int(x) for x in t["w_norm"]]
        self.inv_norm: list[int] = [ft.inv(w) for w in self.w_norm]
        flat = [int(x) for x in t["w_hat"]]
        self.w_hat: list[list[int]] = []
        off = 0
        for i in range(self.levels):
            cnt = max_h >> (i + 1)
            self.w_hat.append(flat[off:off + cnt])
            off += cnt
        self.w_prime: list[int] = [int(x) for x in t["w_prime"]]
        self.b_prod: list[int] = [int(x) for x in t["b_prod"]]
        self.b_prod_inv: list[int] = [int(x) for x in t["b_prod_inv"]]

    def eval_w(self, i: int, x: int) -> int:
        """W_i(x) via linearity (basis.py:95-105)."""
        row = self.w_on_basis[i]
        acc = 0
        b = 0
        while x:
            if x & 1:
                acc ^= row[b]
            x >>= 1
            b += 1
        return acc

    def eval_w_hat(self, i: int, j: int) -> int:
        """Normalised factor W_i(j) / W_i(v_i) (basis.py:107-109)."""
        return self.ft.mul(self.eval_w(i, j), self.inv_norm[i])


def build_basis_tables(ft: FieldTables, max_h: int) -> BasisTables:
    """basis.py:135-137."""
    return BasisTables(ft, max_h)
