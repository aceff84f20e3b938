"""Formal derivative in the LCH basis (drop-in for binfec.derivative,
derivative.py:1-82), executed on the GPU: scale by B_i, gather-XOR over the
zero bits of j, scale by B_j^-1.

derivative_direct (derivative.py:26-43) runs the direct per-coefficient
formula in its own kernel (lch_derivative_direct), an independent path.
"""

from __future__ import annotations

from . import _lib
from .basis import BasisTables
from .transform import CoeffVec, OpCounter


def run_derivative(bt: BasisTables, src, dst) -> None:
    """dst = D(src) for CUDA int16 tensors [batch, h] (uint16 bits)."""
    batch, h = src.shape
    assert dst.shape == src.shape and dst.stride(0) == src.stride(0)
    lg = h.bit_length() - 1
    _lib.check(_lib.lib.lch_derivative(bt.ctx.handle, src.data_ptr(), dst.data_ptr(), batch,
                                       src.stride(0), lg, 0, _lib.stream_ptr()), "derivative")


def _check(bt: BasisTables, h: int) -> None:
    if h < 1 or h & (h - 1):
        raise ValueError(f"transform size must be a power of two, got {h}")
    if h > bt.max_h:
        raise ValueError(f"transform size {h} exceeds table capacity {bt.max_h}")


def derivative_fast(bt: BasisTables, coeffs: CoeffVec,
                    ops: OpCounter | None = None) -> CoeffVec:
    d = list(coeffs.data)
    h = len(d)
    _check(bt, h)
    _lib.require_cuda()
    src = _lib.to_device_u16(d).view(1, h)
    dst = _lib.torch_mod().empty_like(src)
    run_derivative(bt, src, dst)
    out = [int(x) for x in _lib.to_host_u16(dst)[0]]
    if ops is not None:
        # derivative.py:57-58,71-76: h scaling muls, one mul per nonzero output,
        # (terms - 1) adds per output with terms = #{l : bit l of j clear}
        levels = h.bit_length() - 1
        ops.muls += h + sum(1 for x in out if x)
        ops.adds += sum(max(levels - bin(j).count("1") - 1, 0) for j in range(h))
    return CoeffVec(out)


def derivative_direct(bt: BasisTables, coeffs: CoeffVec) -> CoeffVec:
    """out[j] = sum over clear bits l of j of W'_l * d[j + 2^l] (derivative.py:26-43)."""
    d = list(coeffs.data)
    h = len(d)
    _check(bt, h)
    _lib.require_cuda()
    src = _lib.to_device_u16(d).view(1, h)
    dst = _lib.torch_mod().empty_like(src)
    _lib.check(_lib.lib.lch_derivative_direct(bt.ctx.handle, src.data_ptr(), dst.data_ptr(), 1, h,
                                              h.bit_length() - 1, _lib.stream_ptr()), "derivative")
    return CoeffVec([int(x) for x in _lib.to_host_u16(dst)[0]])


def w_prime_const(bt: BasisTables, l: int) -> int:
    return bt.w_prime[l]
