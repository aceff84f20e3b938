"""Erasure-locator evaluation via Walsh-Hadamard transforms (drop-in for
binfec.walsh, walsh.py:1-115).  The FWHTs over Z_{2^r-1}, the pointwise
product with FWHT(log) and the final exp[] run on the GPU (fwht_kernel).
"""

from __future__ import annotations

from collections.abc import Iterable
from dataclasses import dataclass

import numpy as np

from . import _lib
from .field import FieldTables

ResidueVec = list[int]


@dataclass
class LocatorValues:
    """pi_bar[j] at survivors, pi_prime[j] at erased positions (walsh.py:29-39)."""

    pi_bar: dict[int, int]
    pi_prime: dict[int, int]


_FWHT_CTX = None


def _fwht_ctx() -> "_lib.Context":
    global _FWHT_CTX
    if _FWHT_CTX is None:
        _FWHT_CTX = _lib.Context(8, 0x11D, 0)
    return _FWHT_CTX


def fwht(data: ResidueVec, modulus: int) -> ResidueVec:
    """In-place Walsh-Hadamard transform over Z_modulus (walsh.py:42-61)."""
    n = len(data)
    if n & (n - 1):
        raise ValueError(f"length must be a power of two, got {n}")
    if n == 0:
        return data
    if not 0 < modulus < (1 << 32):
        raise NotImplementedError("modulus must lie in [1, 2^32)")
    _lib.require_cuda()
    host = np.asarray([int(x) % modulus for x in data], dtype=np.uint32)
    dev = _lib.to_device_u32(host)
    _lib.check(_lib.lib.lch_fwht(_fwht_ctx().handle, dev.data_ptr(), 1, n.bit_length() - 1,
                                 modulus, _lib.stream_ptr()), "fwht")
    out = dev.cpu().numpy().view(np.uint32)
    data[:] = [int(x) for x in out]
    return data


def _fwht_of_log(ft: FieldTables) -> list[int]:
    """Cached FWHT of the log table (walsh.py:64-74); built by the native table builder."""
    cached = getattr(ft, "_fwht_log_list", None)
    if cached is None:
        cached = [int(x) for x in ft._np["fwht_log"]]
        ft._fwht_log_list = cached
    return cached


def locator_values_device(ft: FieldTables, bits_dev, npatterns: int = 1):
    """Raw device call: locator values [npatterns, 2^r] (uint16 bits in int16)."""
    torch = _lib.torch_mod()
    n = ft.order
    loc = torch.empty((npatterns, n), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_locator(ft._ctx.handle, bits_dev.data_ptr(), npatterns,
                                    loc.data_ptr(), None, _lib.stream_ptr()), "locator")
    return loc


def locator_values(ft: FieldTables, erasures: Iterable[int]) -> LocatorValues:
    """Locator values for an erasure set, all positions at once (walsh.py:77-115)."""
    positions = list(erasures)
    erased = set(positions)
    if not erased:
        raise ValueError("erasure set must not be empty")
    if len(erased) != len(positions):
        raise ValueError("duplicate erasure positions")
    n = ft.order
    if len(erased) > n - 1:
        raise ValueError("erasure set must leave at least one survivor")
    for e in erased:
        if not 0 <= e < n:
            raise ValueError(f"erasure position {e} outside field of size {n}")
    _lib.require_cuda()
    bits = _lib.to_device_u32(_lib.bitmask_from_positions(n, erased))
    loc = _lib.to_host_u16(locator_values_device(ft, bits))[0]
    pi_bar: dict[int, int] = {}
    pi_prime: dict[int, int] = {}
    for j in range(n):
        if j in erased:
            pi_prime[j] = int(loc[j])
        else:
            pi_bar[j] = int(loc[j])
    return LocatorValues(pi_bar, pi_prime)
