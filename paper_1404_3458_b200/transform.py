"""The h-point LCH transform and its inverse (drop-in for binfec.transform,
transform.py:1-206), executed by the sm_100a pass kernels through liblch.

OpCounter totals are filled from the closed form of the butterfly schedule
the reference instruments (transform.py:118-140, 159-175): per level, every
block costs 2*half adds and half muls, except the block whose start equals
the shift, which costs half adds and no muls.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .basis import BasisTables


@dataclass
class CoeffVec:
    """Basis-domain coefficients; length must be a power of two."""

    data: list[int]

    def __len__(self) -> int:
        return len(self.data)


@dataclass
class EvalVec:
    """Evaluations at points indexed c ^ shift, c = 0..h-1."""

    data: list[int]
    shift: int = 0

    def __len__(self) -> int:
        return len(self.data)


@dataclass
class OpCounter:
    """Running totals of field additions and multiplications."""

    adds: int = 0
    muls: int = 0


def _check_size(bt: BasisTables, h: int, shift: int) -> None:
    # transform.py:60-66
    if h < 1 or h & (h - 1):
        raise ValueError(f"transform size must be a power of two, got {h}")
    if h > bt.max_h:
        raise ValueError(f"transform size {h} exceeds table capacity {bt.max_h}")
    if not 0 <= shift < bt.ft.order:
        raise ValueError(f"shift {shift} outside field of size {bt.ft.order}")


def transform_op_counts(h: int, shift: int, order: int) -> tuple[int, int]:
    """(adds, muls) the reference's schedule executes for one h-point transform."""
    adds = muls = 0
    levels = h.bit_length() - 1
    for i in range(levels):
        half = 1 << i
        step = half << 1
        blocks = h // step
        zero = 1 if (shift < h and not shift & (step - 1)) else 0
        adds += (blocks - zero) * 2 * half + zero * half
        muls += (blocks - zero) * half
    return adds, muls


def run_transform(bt: BasisTables, dev, shift: int, inverse: bool) -> None:
    """In-place batched transform of a CUDA int16 tensor [batch, h] (uint16 bits)."""
    batch, h = dev.shape
    lg = h.bit_length() - 1
    fn = _lib.lib.lch_inverse if inverse else _lib.lib.lch_forward
    _lib.check(fn(bt.ctx.handle, dev.data_ptr(), batch, dev.stride(0), lg, shift, 0,
                  _lib.stream_ptr()), "inverse" if inverse else "forward")


def _one(bt: BasisTables, data: list[int], shift: int, inverse: bool) -> list[int]:
    _lib.require_cuda()
    dev = _lib.to_device_u16(data).view(1, len(data))
    run_transform(bt, dev, shift, inverse)
    return [int(x) for x in _lib.to_host_u16(dev)[0]]


def forward(bt: BasisTables, coeffs: CoeffVec, shift: int = 0,
            ops: OpCounter | None = None) -> EvalVec:
    """Transform coefficients into evaluations at points c ^ shift (transform.py:69-76)."""
    h = len(coeffs.data)
    _check_size(bt, h, shift)
    out = _one(bt, list(coeffs.data), shift, False)
    if ops is not None:
        a, m = transform_op_counts(h, shift, bt.ft.order)
        ops.adds += a
        ops.muls += m
    return EvalVec(out, shift)


def inverse(bt: BasisTables, evals: EvalVec, ops: OpCounter | None = None) -> CoeffVec:
    """Recover the coefficients whose forward transform is `evals` (transform.py:79-86)."""
    h = len(evals.data)
    _check_size(bt, h, evals.shift)
    out = _one(bt, list(evals.data), evals.shift, True)
    if ops is not None:
        a, m = transform_op_counts(h, evals.shift, bt.ft.order)
        ops.adds += a
        ops.muls += m
    return CoeffVec(out)


def forward_counted(bt: BasisTables, coeffs: CoeffVec,
                    shift: int = 0) -> tuple[EvalVec, OpCounter]:
    ops = OpCounter()
    return forward(bt, coeffs, shift, ops), ops


def inverse_counted(bt: BasisTables, evals: EvalVec) -> tuple[CoeffVec, OpCounter]:
    ops = OpCounter()
    return inverse(bt, evals, ops), ops


def degree(coeffs: CoeffVec) -> int | None:
    """Largest index with a nonzero coefficient (transform.py:178-186)."""
    for j in range(len(coeffs.data) - 1, -1, -1):
        if coeffs.data[j]:
            return j
    return None


def poly_mul(bt: BasisTables, a: CoeffVec, b: CoeffVec) -> CoeffVec:
    """Product via 2h-point transforms (transform.py:189-206)."""
    h = len(a.data)
    if len(b.data) != h:
        raise ValueError("poly_mul operands must have equal length")
    h2 = 2 * h
    if h2 > bt.max_h:
        raise ValueError(f"product size {h2} exceeds table capacity {bt.max_h}")
    _lib.require_cuda()
    # both operands zero-extended to 2h, forward, pointwise product, inverse:
    # all on the device, one copy in and one out
    dev = _lib.to_device_u16([list(a.data) + [0] * h, list(b.data) + [0] * h])
    run_transform(bt, dev, 0, False)
    _lib.check(_lib.lib.lch_pointwise_mul(bt.ctx.handle, dev[0].data_ptr(), dev[1].data_ptr(),
                                          dev[0].data_ptr(), h2, _lib.stream_ptr()), "poly_mul")
    pd = dev[0:1]
    run_transform(bt, pd, 0, True)
    return CoeffVec([int(x) for x in _lib.to_host_u16(pd)[0]])
