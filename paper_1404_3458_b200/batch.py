"""Whole-batch codec (drop-in for binfec.batch.BatchCodec, batch.py:1-153).

Rows are independent codewords (stripes).  The reference applies one
butterfly schedule to a (stripes x n) numpy matrix; here the matrix is moved
to HBM once and the fused sm_100a pipelines process all rows at once, 1024
codewords per CTA (one bit-plane word per thread lane).

Inputs may be numpy arrays (host; results come back as numpy uint16) or CUDA
tensors (zero-copy; results stay on the device, dtype int16 carrying the
uint16 bit patterns, or torch.uint16 if given that).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import TooManyErasuresError
from .basis import BasisTables
from .derivative import run_derivative
from .rs import CodeParams, decode_device, decode_host, encode_device, encode_host
from .transform import run_transform


def _is_torch(a) -> bool:
    try:
        import torch
        return isinstance(a, torch.Tensor)
    except Exception:
        return False


class BatchCodec:
    """Matrix encoder/decoder for one (CodeParams, BasisTables) pair."""

    def __init__(self, cp: CodeParams, bt: BasisTables):
        if bt.ft.r != cp.r:
            raise ValueError(f"basis tables built for r={bt.ft.r}, code needs r={cp.r}")
        if bt.max_h < cp.n:
            raise ValueError(f"basis tables capacity {bt.max_h} below n={cp.n}")
        self.cp = cp
        self.bt = bt
        self.ft = bt.ft

    # -- device helpers ------------------------------------------------------

    @staticmethod
    def _dev(a):
        _lib.require_cuda()
        if _is_torch(a):
            t = _lib.to_device_u16(a)
            return t if t.dim() == 2 else t.view(1, -1)
        arr = np.asarray(a)
        if arr.ndim != 2:
            raise ValueError("expected a 2-D (stripes x symbols) matrix")
        return _lib.to_device_u16(arr.astype(np.uint16, copy=False))

    @staticmethod
    def _back(like, dev):
        if _is_torch(like):
            import torch
            return dev.view(torch.uint16) if like.dtype == torch.uint16 else dev
        return _lib.to_host_u16(dev)

    # -- transforms on matrices (columns = codeword positions) ---------------

    def _forward_inplace(self, a, shift: int) -> None:
        """batch.py:65-81 (mutates `a`)."""
        self._inplace(a, shift, False)

    def _inverse_inplace(self, a, shift: int) -> None:
        """batch.py:83-99 (mutates `a`)."""
        self._inplace(a, shift, True)

    def _inplace(self, a, shift: int, inverse: bool) -> None:
        h = a.shape[1]
        if h < 1 or h & (h - 1) or h > self.bt.max_h:
            raise ValueError(f"transform size {h} invalid for table capacity {self.bt.max_h}")
        if not 0 <= shift < self.ft.order:
            raise ValueError(f"shift {shift} outside field of size {self.ft.order}")
        if _is_torch(a) and a.is_cuda and a.dtype in (_lib.torch_mod().int16,
                                                        _lib.torch_mod().uint16):
            t = a.view(_lib.torch_mod().int16)
            run_transform(self.bt, t, shift, inverse)
            return
        dev = self._dev(a)
        run_transform(self.bt, dev, shift, inverse)
        res = self._back(a, dev)
        a[...] = res

    def _derivative(self, a):
        """batch.py:101-106."""
        dev = self._dev(a)
        out = _lib.torch_mod().empty_like(dev)
        run_derivative(self.bt, dev, out)
        return self._back(a, out)

    # -- public API ------------------------------------------------------------

    def encode(self, messages):
        """Encode a (stripes x k) message matrix into (stripes x n) (batch.py:110-124).

        Host (numpy) matrices stream through the GPU in overlapped chunks
        (lch_encode_host); CUDA tensors are encoded in place on the device."""
        cp = self.cp
        s, width = messages.shape
        if width != cp.k:
            raise ValueError(f"message width {width} != k={cp.k}")
        if not _is_torch(messages):
            _lib.require_cuda()
            msg = np.ascontiguousarray(np.asarray(messages).astype(np.uint16, copy=False))
            out = np.empty((s, cp.n), np.uint16)
            out[:, :cp.k] = msg
            if cp.n > cp.k and s > 0:
                encode_host(cp, self.bt, msg, out[:, cp.k:])
                _lib.torch_mod().cuda.current_stream().synchronize()
            return out
        torch = _lib.torch_mod()
        md = self._dev(messages)
        out = torch.empty((s, cp.n), dtype=torch.int16, device="cuda")
        out[:, :cp.k].copy_(md)
        if cp.n > cp.k and s > 0:
            encode_device(cp, self.bt, md, out[:, cp.k:])
        return self._back(messages, out)

    def decode_patterns(self, received, erased_masks):
        """Extension: one erasure pattern per row (rs.decode row by row, config 4b).

        erased_masks: bool/uint8 array [stripes, n] (True = erased).  Rows may
        erase 0..n-k positions; more raises TooManyErasuresError.
        """
        cp = self.cp
        n, k = cp.n, cp.k
        if received.shape[1] != n:
            raise ValueError(f"received width {received.shape[1]} != n={n}")
        torch = _lib.torch_mod()
        rd = self._dev(received)
        if _is_torch(erased_masks) and erased_masks.is_cuda:
            # device masks: packed on the device; the library counts the
            # erasures of each pattern itself (and reports too many)
            m = erased_masks.bool()
            if tuple(m.shape) != (rd.shape[0], n):
                raise ValueError("erased_masks must be [stripes, n]")
            from .gen import mask_to_bits
            bits = mask_to_bits(m).contiguous()
            counts = None
        else:
            # host masks: bit-pack and count on the host, one upload
            mh = erased_masks.numpy() if _is_torch(erased_masks) else np.asarray(erased_masks)
            mh = mh.astype(bool, copy=False)
            if mh.shape != (rd.shape[0], n):
                raise ValueError("erased_masks must be [stripes, n]")
            counts = np.count_nonzero(mh, axis=1).tolist()
            if any(c > n - k for c in counts):
                raise TooManyErasuresError(f"{max(counts)} erasures exceed repair capacity {n - k}")
            packed = np.packbits(mh, axis=1, bitorder="little").view(np.uint32)
            bits = _lib.to_device_u32(np.ascontiguousarray(packed))
        out = torch.empty((rd.shape[0], k), dtype=torch.int16, device="cuda")
        if rd.shape[0] > 0:
            decode_device(cp, self.bt, rd, bits, out, counts)
        return self._back(received, out)

    def decode(self, received, erased: set[int]):
        """Recover the (stripes x k) messages; erased columns are ignored (batch.py:126-153)."""
        cp = self.cp
        n, k = cp.n, cp.k
        if received.shape[1] != n:
            raise ValueError(f"received width {received.shape[1]} != n={n}")
        erased = set(int(e) for e in erased)
        for e in erased:
            if not 0 <= e < n:
                raise ValueError(f"erasure position {e} outside field of size {n}")
        if len(erased) > n - k:
            raise TooManyErasuresError(f"{len(erased)} erasures exceed repair capacity {n - k}")
        if not _is_torch(received):
            rx = np.ascontiguousarray(np.asarray(received).astype(np.uint16, copy=False))
            if not erased:
                return rx[:, :k].copy()
            _lib.require_cuda()
            out = np.empty((rx.shape[0], k), np.uint16)
            if rx.shape[0] > 0:
                decode_host(cp, self.bt, rx, _lib.bitmask_from_positions(n, erased), out)
                _lib.torch_mod().cuda.current_stream().synchronize()
            return out
        rd = self._dev(received)
        if not erased:
            return self._back(received, rd[:, :k].contiguous())
        torch = _lib.torch_mod()
        bits = _lib.to_device_u32(_lib.bitmask_from_positions(n, erased))
        out = torch.empty((rd.shape[0], k), dtype=torch.int16, device="cuda")
        if rd.shape[0] > 0:
            decode_device(cp, self.bt, rd, bits, out, len(erased))
        return self._back(received, out)
