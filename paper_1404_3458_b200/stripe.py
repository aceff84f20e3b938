"""Storage-stripe codec (config 5): packet-major stripe groups, any k.

A stripe group holds n = 2^r positions; position j is a packet of P symbols
(P a multiple of 1024; 2048 uint16 = 4 KiB in the storage workload) and the
transform / code act symbol-wise across the packet, so lane s of a group is an
ordinary RS(n, k) codeword.  This is the reference's shard layout: shard j =
symbol j of every stripe (shardfile.py:16-20,129-140), with the stripes of the
reference's `bytes_to_stripes` (shardfile.py:109-122) becoming the P lanes.

Device layout: tensors [groups, positions, P] (CUDA int16/uint16, contiguous),
lane b = g * P + s.  Power-of-two k follows rs.encode / BatchCodec exactly
(rs.py:85-96, batch.py:110-153).  Other k (k/n = 3/4, 15/16: rejected by the
reference's CodeParams, rs.py:43-44) use the interpolation code of SURVEY H6:
the codeword is the evaluation of the degree < k polynomial through the
message at positions 0..k-1, computed by erasure-decoding E = [k, n).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .basis import BasisTables


def _check_packets(t, P: int, what: str):
    torch = _lib.torch_mod()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dim() == 3):
        raise ValueError(f"{what}: expected a CUDA tensor [groups, positions, packet_len]")
    if t.dtype not in (torch.int16, torch.uint16):
        raise ValueError(f"{what}: expected int16/uint16 symbols")
    if t.shape[2] != P or not t.is_contiguous():
        raise ValueError(f"{what}: expected contiguous [groups, positions, {P}]")
    return t.view(torch.int16)


class StripeCodec:
    """RS(2^r, k) over packet-major stripe groups, 1 <= k <= 2^r."""

    def __init__(self, bt: BasisTables, k: int, packet_len: int = 2048):
        n = 1 << bt.ft.r
        if not 1 <= k <= n:
            raise ValueError(f"k={k} outside [1, {n}]")
        if packet_len <= 0 or packet_len % 1024:
            raise ValueError(f"packet_len {packet_len} must be a positive multiple of 1024")
        if bt.max_h < n and k & (k - 1):
            raise ValueError("non-power-of-two k needs n-point basis tables")
        self.bt, self.k, self.n, self.P = bt, k, n, packet_len

    @property
    def ctx(self):
        return self.bt.ctx

    def encode_into(self, msg, parity) -> None:
        """msg [G, k, P] -> parity [G, n-k, P] (positions k..n-1)."""
        m = _check_packets(msg, self.P, "msg")
        p = _check_packets(parity, self.P, "parity")
        if m.shape[1] != self.k or p.shape[1] != self.n - self.k or p.shape[0] != m.shape[0]:
            raise ValueError("shape mismatch: msg [G, k, P], parity [G, n-k, P]")
        _lib.check(_lib.lib.lch_encode_k(self.ctx.handle, m.data_ptr(), self.k, p.data_ptr(),
                                         self.n - self.k, m.shape[0] * self.P, self.k, self.P,
                                         _lib.stream_ptr()), "encode")

    def encode(self, msg):
        torch = _lib.torch_mod()
        parity = torch.empty((msg.shape[0], self.n - self.k, self.P), dtype=torch.int16,
                             device=msg.device)
        self.encode_into(msg, parity)
        return parity

    def decode_into(self, rx, erased, out, counts=None) -> None:
        """rx [G, n, P] (erased packets ignored) -> out [G, k, P].

        erased: int32 bitmask words [n/32] (one pattern for every group) or
        [G, n/32] (one pattern per stripe group); see gen.mask_to_bits.
        """
        r = _check_packets(rx, self.P, "rx")
        o = _check_packets(out, self.P, "out")
        if r.shape[1] != self.n or o.shape[1] != self.k or o.shape[0] != r.shape[0]:
            raise ValueError("shape mismatch: rx [G, n, P], out [G, k, P]")
        shared = 1 if erased.dim() == 1 else 0
        cnt = None
        if counts is not None:
            vals = [int(counts)] if shared else [int(x) for x in counts]
            cnt = (ctypes.c_int64 * len(vals))(*vals)
        _lib.check(_lib.lib.lch_decode_k(self.ctx.handle, r.data_ptr(), self.n,
                                         erased.contiguous().data_ptr(), shared, o.data_ptr(),
                                         self.k, r.shape[0] * self.P, self.k, self.P, cnt,
                                         _lib.stream_ptr()), "decode")

    def decode(self, rx, erased, counts=None):
        torch = _lib.torch_mod()
        out = torch.empty((rx.shape[0], self.k, self.P), dtype=torch.int16, device=rx.device)
        self.decode_into(rx, erased, out, counts)
        return out

    # -- symbol-wise transforms over packets (transform.py:69-86, derivative.py:46)

    def forward_inplace(self, a, shift: int = 0) -> None:
        self._transform(a, shift, False)

    def inverse_inplace(self, a, shift: int = 0) -> None:
        self._transform(a, shift, True)

    def _transform(self, a, shift: int, inverse: bool) -> None:
        t = _check_packets(a, self.P, "data")
        h = t.shape[1]
        if h < 1 or h & (h - 1):
            raise ValueError(f"transform size {h} is not a power of two")
        fn = _lib.lib.lch_inverse if inverse else _lib.lib.lch_forward
        _lib.check(fn(self.ctx.handle, t.data_ptr(), t.shape[0] * self.P, h, h.bit_length() - 1,
                      shift, self.P, _lib.stream_ptr()), "transform")

    def derivative(self, a):
        torch = _lib.torch_mod()
        t = _check_packets(a, self.P, "data")
        h = t.shape[1]
        if h < 1 or h & (h - 1):
            raise ValueError(f"transform size {h} is not a power of two")
        out = torch.empty_like(t)
        _lib.check(_lib.lib.lch_derivative(self.ctx.handle, t.data_ptr(), out.data_ptr(),
                                           t.shape[0] * self.P, h, h.bit_length() - 1, self.P,
                                           _lib.stream_ptr()), "derivative")
        return out


def set_scratch_limit(bt: BasisTables, nbytes: int) -> None:
    """Device scratch budget per call; larger batches run in lane chunks."""
    _lib.check(_lib.lib.lch_set_scratch_limit(bt.ctx.handle, int(nbytes)), "scratch limit")
