"""Seeded synthetic inputs on the device.

symbol(seed, cw, pos) = key(seed, cw, pos) & (2^r - 1) and the erasure set
of a codeword = the `count` positions with the smallest (key >> 1, pos),
key = SplitMix64-style mix (csrc/lch_kernels.cu key_d; identical to the
oracle's orc_key and the pure-Python restatement in tests/golden_util.py).
"""

from __future__ import annotations

import numpy as np

from . import _lib


def symbols(ctx, seed: int, cw0: int, batch: int, length: int):
    torch = _lib.torch_mod()
    t = torch.empty((batch, length), dtype=torch.int16, device="cuda")
    if batch and length:
        _lib.check(_lib.lib.lch_gen_symbols(ctx.handle, seed, cw0, batch, length, t.data_ptr(),
                                            length, _lib.stream_ptr()), "gen_symbols")
    return t


def packets(ctx, seed: int, cw0: int, groups: int, length: int, packet_len: int):
    """[groups, length, P] packet-major symbols; lane g * P + s = codeword cw0 + g * P + s,
    so lane s of group g equals row g * P + s of `symbols`."""
    torch = _lib.torch_mod()
    t = torch.empty((groups, length, packet_len), dtype=torch.int16, device="cuda")
    if groups and length:
        _lib.check(_lib.lib.lch_gen_packets(ctx.handle, seed, cw0, groups * packet_len, length,
                                            t.data_ptr(), length, packet_len, _lib.stream_ptr()),
                   "gen_packets")
    return t


def erasure_masks(ctx, seed: int, n: int, count: int, cw0: int, batch: int):
    """Bool tensor [batch, n]: True at erased positions."""
    torch = _lib.torch_mod()
    keys = torch.empty((batch, n), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib.lch_gen_keys(ctx.handle, seed, cw0, batch, n, keys.data_ptr(),
                                     _lib.stream_ptr()), "gen_keys")
    order = torch.sort(keys, dim=1, stable=True).indices  # ties broken by position
    mask = torch.zeros((batch, n), dtype=torch.bool, device="cuda")
    mask.scatter_(1, order[:, :count], True)
    return mask


def mask_to_bits(mask) -> "object":
    """Bool [batch, n] -> packed uint32 bitmask words [batch, n/32] (int32 storage)."""
    torch = _lib.torch_mod()
    b, n = mask.shape
    m = mask.view(b, n // 32, 32).to(torch.int64)
    w = (m << torch.arange(32, device=mask.device, dtype=torch.int64)).sum(dim=2)
    return torch.where(w >= (1 << 31), w - (1 << 32), w).to(torch.int32)


def mask_to_bits_host(mask: np.ndarray) -> np.ndarray:
    return _lib.bitmask_from_positions(mask.shape[-1], np.nonzero(mask)[0])
