"""ctypes binding of liblch.so (include/lch.h) + device-buffer plumbing.

The product path has no CPU fallback: every compute call goes through the
CUDA library; without a CUDA device the library returns LCH_ECUDA and the
shim raises RuntimeError.  If the shared object is missing, importing the
package raises ImportError (build it with `python __graft_entry__.py` or
`python -m paper_1404_3458_b200.build`).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("LCH_SO_PATH") or os.path.join(_HERE, "_build", "liblch.so")

LCH_OK = 0
LCH_EINVAL = -1
LCH_ETOOMANY = -2
LCH_ENOTPRIM = -3
LCH_ECUDA = -4
LCH_ENOMEM = -5
LCH_EUNSUPPORTED = -6
LCH_EZERODIV = -7


class TooManyErasuresError(ValueError):
    """More erasures than the code can repair (above n - k); rs.py:30-31."""


def _load() -> ctypes.CDLL:
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"liblch.so not built ({SO_PATH}); run `python -m paper_1404_3458_b200.build`")
    L = ctypes.CDLL(SO_PATH)
    P = ctypes.c_void_p
    i32, u32, i64, u64 = ctypes.c_int, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64
    sig = {
        "lch_version": ([], ctypes.c_char_p),
        "lch_strerror": ([i32], ctypes.c_char_p),
        "lch_init": ([i32, u32, i32, ctypes.POINTER(P)], i32),
        "lch_init_alpha": ([i32, u32, u32, i32, ctypes.POINTER(P)], i32),
        "lch_destroy": ([P], None),
        "lch_get_tables": ([P] + [P] * 9, i32),
        "lch_forward": ([P, P, i64, i64, i32, u32, i64, P], i32),
        "lch_inverse": ([P, P, i64, i64, i32, u32, i64, P], i32),
        "lch_derivative": ([P, P, P, i64, i64, i32, i64, P], i32),
        "lch_fwht": ([P, P, i64, i32, u32, P], i32),
        "lch_locator": ([P, P, i64, P, P, P], i32),
        "lch_encode": ([P, P, i64, P, i64, i64, i32, i64, P], i32),
        "lch_decode": ([P, P, i64, P, i32, P, i64, i64, i32, i64, P, P], i32),
        "lch_encode_k": ([P, P, i64, P, i64, i64, i64, i64, P], i32),
        "lch_decode_k": ([P, P, i64, P, i32, P, i64, i64, i64, i64, P, P], i32),
        "lch_set_scratch_limit": ([P, u64], i32),
        "lch_set_host_ordering": ([P, i32], i32),
        "lch_release_host_buffers": ([P], i32),
        "lch_host_copy_bytes": ([P, P, P], i32),
        "lch_compact_rows": ([P, P, i64, P, i64, i64, P, i64], i32),
        "lch_encode_host": ([P, P, i64, P, i64, i64, i64, i64, i64, P], i32),
        "lch_decode_host": ([P, P, i64, P, i32, P, i64, i64, i64, i64, i64, P], i32),
        "lch_gen_symbols": ([P, u64, u64, i64, i64, P, i64, P], i32),
        "lch_gen_packets": ([P, u64, u64, i64, i64, P, i64, i64, P], i32),
        "lch_pointwise_mul": ([P, P, P, P, i64, P], i32),
        "lch_derivative_direct": ([P, P, P, i64, i64, i32, P], i32),
        "lch_stripes_to_packets": ([P, P, i64, i32, i64, P, i64, P], i32),
        "lch_packets_to_stripes": ([P, P, i64, i32, i64, P, i64, P], i32),
        "lch_payload_to_packets": ([P, P, i64, i64, i32, P, i64, P], i32),
        "lch_packets_to_payload": ([P, P, i64, i64, i64, i32, P, P], i32),
        "lch_gen_keys": ([P, u64, u64, i64, i64, P, P], i32),
        "lch_launch_count": ([P], i64),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()


def check(rc: int, what: str = "") -> None:
    if rc == LCH_OK:
        return
    msg = lib.lch_strerror(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == LCH_ETOOMANY:
        raise TooManyErasuresError(msg)
    if rc in (LCH_EINVAL, LCH_ENOTPRIM):
        raise ValueError(msg)
    if rc == LCH_EZERODIV:
        raise ZeroDivisionError(msg)
    if rc == LCH_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


class Context:
    """One liblch context: tables for (r, poly) with capacity 2^max_lg_h."""

    def __init__(self, r: int, poly: int, max_lg_h: int, alpha: int = 2):
        h = ctypes.c_void_p()
        check(lib.lch_init_alpha(r, poly, alpha, max_lg_h, ctypes.byref(h)), "lch_init")
        self.handle = h
        self.r, self.poly, self.max_lg_h, self.alpha = r, poly, max_lg_h, alpha
        self.lock = threading.Lock()

    def __del__(self):
        try:
            if self.handle:
                lib.lch_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def tables(self) -> dict:
        r = self.r
        n, mh = 1 << r, 1 << self.max_lg_h
        out = dict(
            log=np.zeros(n, np.uint16), exp=np.zeros(n - 1, np.uint16),
            w_hat=np.zeros(max(mh - 1, 1), np.uint16), w_prime=np.zeros(r, np.uint16),
            b_prod=np.zeros(mh, np.uint16), b_prod_inv=np.zeros(mh, np.uint16),
            fwht_log=np.zeros(n, np.uint32), w_on_basis=np.zeros(r * r, np.uint16),
            w_norm=np.zeros(r, np.uint16))
        keys = ("log", "exp", "w_hat", "w_prime", "b_prod", "b_prod_inv", "fwht_log",
                "w_on_basis", "w_norm")
        check(lib.lch_get_tables(self.handle, *[out[k].ctypes.data for k in keys]))
        out["w_hat"] = out["w_hat"][: mh - 1]
        out["w_on_basis"] = out["w_on_basis"].reshape(r, r)
        return out


# ---------------------------------------------------------------------------
# device buffers (torch is the allocator/stream provider, not the compute)

def torch_mod():
    import torch
    return torch


def cuda_ok() -> bool:
    try:
        return torch_mod().cuda.is_available()
    except Exception:
        return False


def require_cuda() -> None:
    if not cuda_ok():
        raise RuntimeError("no CUDA device: the LCH codec runs only on the GPU (no CPU fallback)")


def stream_ptr() -> int:
    return torch_mod().cuda.current_stream().cuda_stream


def to_device_u16(a) -> "object":
    """Host array-like -> contiguous CUDA int16 tensor holding the uint16 bits."""
    torch = torch_mod()
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype == torch.uint16:
            t = t.view(torch.int16)
        elif t.dtype != torch.int16:
            t = t.to(torch.int32).to(torch.int16)
        return t.to("cuda").contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint16))
    return torch.from_numpy(arr.view(np.int16)).to("cuda")


def to_host_u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def ptr(t) -> int:
    return t.data_ptr()


def bitmask_from_positions(n: int, positions) -> np.ndarray:
    words = max(1, (n + 31) // 32)
    bits = np.zeros(words, np.uint32)
    pos = np.asarray(list(positions), dtype=np.int64)
    if pos.size:
        np.bitwise_or.at(bits, pos >> 5, (np.uint32(1) << (pos & 31).astype(np.uint32)))
    return bits


def to_device_u32(a) -> "object":
    torch = torch_mod()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return torch.from_numpy(arr.view(np.int32)).to("cuda")
