"""ctypes wrapper for the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

The oracle (lch_oracle.c) restates the reference `binfec` hot path in C with
file:line citations.  Only tests/, __graft_entry__.smoke() and bench.py (the
cpu_baseline leg and the `--impl reference` arm) import this module; the
product package `paper_1404_3458_b200` never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liblch_oracle.so")

ORC_OK, ORC_EINVAL, ORC_ETOOMANY, ORC_ENOTPRIM = 0, -1, -2, -3


def build() -> str:
    """Compile the oracle if its .so is missing or stale."""
    src = os.path.join(_HERE, "lch_oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, U16P, U32P, U8P = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
        i32, u32, i64, u64 = ctypes.c_int, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64
        L.orc_create.argtypes = [i32, u32, u32, ctypes.POINTER(P)]
        L.orc_destroy.argtypes = [P]
        L.orc_tables.argtypes = [P, U16P, U16P, U16P, U16P, U16P, U16P, U32P, U16P, U16P]
        L.orc_mul.argtypes = [P, u32, u32]
        L.orc_mul.restype = u32
        L.orc_eval_w_hat.argtypes = [P, i32, u32]
        L.orc_eval_w_hat.restype = u32
        for name in ("orc_forward", "orc_inverse"):
            getattr(L, name).argtypes = [P, U16P, u32, u32]
        L.orc_derivative.argtypes = [P, U16P, U16P, u32]
        L.orc_fwht.argtypes = [U32P, u32, u32]
        L.orc_locator_logs.argtypes = [P, U8P, U32P]
        L.orc_encode.argtypes = [P, u32, U16P, U16P]
        L.orc_decode.argtypes = [P, u32, U16P, U8P, U16P]
        L.orc_encode_batch.argtypes = [P, u32, U16P, U16P, i64, i32]
        L.orc_decode_batch.argtypes = [P, u32, U16P, U8P, i32, U16P, i64, i32]
        L.orc_transform_batch.argtypes = [P, U16P, u32, u32, i32, i64, i32]
        L.orc_recover_all.argtypes = [P, U16P, U8P, U16P]
        L.orc_encode_any.argtypes = [P, u32, U16P, U16P]
        L.orc_decode_any.argtypes = [P, u32, U16P, U8P, U16P]
        L.orc_encode_any_batch.argtypes = [P, u32, U16P, U16P, i64, i32]
        L.orc_decode_any_batch.argtypes = [P, u32, U16P, U8P, i32, U16P, i64, i32]
        L.orc_mix64.argtypes = [u64]
        L.orc_mix64.restype = u64
        L.orc_key.argtypes = [u64, u64, u64]
        L.orc_key.restype = u64
        L.orc_gen_symbols.argtypes = [u64, i32, u64, i64, u32, U16P]
        L.orc_gen_erasures.argtypes = [u64, u32, u32, u64, i64, U8P]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _check(rc: int) -> None:
    if rc == ORC_OK:
        return
    if rc == ORC_ETOOMANY:
        raise ValueError("too many erasures")
    raise ValueError(f"oracle error {rc}")


class Oracle:
    """One (r, poly, max_h) instance of the restated reference tables."""

    def __init__(self, r: int, poly: int | None = None, max_h: int | None = None):
        defaults = {8: 0x11D, 16: 0x1100B}
        self.r = r
        self.poly = defaults[r] if poly is None else poly
        self.n = 1 << r
        self.max_h = self.n if max_h is None else max_h
        h = ctypes.c_void_p()
        _check(lib().orc_create(r, self.poly, self.max_h, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                lib().orc_destroy(self._h)
        except Exception:
            pass

    def tables(self) -> dict:
        n, mh, r = self.n, self.max_h, self.r
        out = dict(
            log=np.zeros(n, np.uint16), exp=np.zeros(n - 1, np.uint16),
            w_hat=np.zeros(max(mh - 1, 1), np.uint16), w_prime=np.zeros(r, np.uint16),
            b_prod=np.zeros(mh, np.uint16), b_prod_inv=np.zeros(mh, np.uint16),
            fwht_log=np.zeros(n, np.uint32), w_on_basis=np.zeros(r * r, np.uint16),
            w_norm=np.zeros(r, np.uint16))
        lib().orc_tables(self._h, *[_p(out[k]) for k in (
            "log", "exp", "w_hat", "w_prime", "b_prod", "b_prod_inv", "fwht_log",
            "w_on_basis", "w_norm")])
        out["w_hat"] = out["w_hat"][: mh - 1]
        out["w_on_basis"] = out["w_on_basis"].reshape(r, r)
        return out

    def mul(self, a: int, b: int) -> int:
        return int(lib().orc_mul(self._h, a, b))

    def eval_w_hat(self, i: int, x: int) -> int:
        return int(lib().orc_eval_w_hat(self._h, i, x))

    def forward(self, a, shift: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(a, dtype=np.uint16).copy()
        _check(lib().orc_forward(self._h, _p(x), x.size, shift))
        return x

    def inverse(self, a, shift: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(a, dtype=np.uint16).copy()
        _check(lib().orc_inverse(self._h, _p(x), x.size, shift))
        return x

    def transform_batch(self, a: np.ndarray, shift: int, inverse: bool,
                        nthreads: int = 1) -> np.ndarray:
        x = np.ascontiguousarray(a, dtype=np.uint16).copy()
        _check(lib().orc_transform_batch(self._h, _p(x), x.shape[1], shift,
                                         int(inverse), x.shape[0], nthreads))
        return x

    def derivative(self, a) -> np.ndarray:
        x = np.ascontiguousarray(a, dtype=np.uint16)
        out = np.zeros_like(x)
        _check(lib().orc_derivative(self._h, _p(x), _p(out), x.size))
        return out

    def locator_logs(self, erased_mask) -> np.ndarray:
        e = np.ascontiguousarray(erased_mask, dtype=np.uint8)
        out = np.zeros(self.n, np.uint32)
        _check(lib().orc_locator_logs(self._h, _p(e), _p(out)))
        return out

    def encode(self, k: int, msg) -> np.ndarray:
        m = np.ascontiguousarray(msg, dtype=np.uint16)
        cw = np.zeros(self.n, np.uint16)
        _check(lib().orc_encode(self._h, k, _p(m), _p(cw)))
        return cw

    def decode(self, k: int, received, erased_mask) -> np.ndarray:
        rx = np.ascontiguousarray(received, dtype=np.uint16)
        e = np.ascontiguousarray(erased_mask, dtype=np.uint8)
        out = np.zeros(k, np.uint16)
        _check(lib().orc_decode(self._h, k, _p(rx), _p(e), _p(out)))
        return out

    def encode_batch(self, k: int, msgs: np.ndarray, nthreads: int = 1) -> np.ndarray:
        m = np.ascontiguousarray(msgs, dtype=np.uint16)
        par = np.zeros((m.shape[0], self.n - k), np.uint16)
        _check(lib().orc_encode_batch(self._h, k, _p(m), _p(par), m.shape[0], nthreads))
        return par

    def decode_batch(self, k: int, received: np.ndarray, erased: np.ndarray,
                     nthreads: int = 1) -> np.ndarray:
        rx = np.ascontiguousarray(received, dtype=np.uint16)
        e = np.ascontiguousarray(erased, dtype=np.uint8)
        shared = int(e.ndim == 1)
        out = np.zeros((rx.shape[0], k), np.uint16)
        _check(lib().orc_decode_batch(self._h, k, _p(rx), _p(e), shared, _p(out),
                                      rx.shape[0], nthreads))
        return out


    # -- general k: composition of the reference's primitives --

    def recover_all(self, received, erased_mask) -> np.ndarray:
        rx = np.ascontiguousarray(received, dtype=np.uint16)
        e = np.ascontiguousarray(erased_mask, dtype=np.uint8)
        out = np.zeros(self.n, np.uint16)
        _check(lib().orc_recover_all(self._h, _p(rx), _p(e), _p(out)))
        return out

    def encode_any(self, k: int, msg) -> np.ndarray:
        m = np.ascontiguousarray(msg, dtype=np.uint16)
        cw = np.zeros(self.n, np.uint16)
        _check(lib().orc_encode_any(self._h, k, _p(m), _p(cw)))
        return cw

    def decode_any(self, k: int, received, erased_mask) -> np.ndarray:
        rx = np.ascontiguousarray(received, dtype=np.uint16)
        e = np.ascontiguousarray(erased_mask, dtype=np.uint8)
        out = np.zeros(k, np.uint16)
        _check(lib().orc_decode_any(self._h, k, _p(rx), _p(e), _p(out)))
        return out

    def encode_any_batch(self, k: int, msgs: np.ndarray, nthreads: int = 1) -> np.ndarray:
        m = np.ascontiguousarray(msgs, dtype=np.uint16)
        par = np.zeros((m.shape[0], self.n - k), np.uint16)
        _check(lib().orc_encode_any_batch(self._h, k, _p(m), _p(par), m.shape[0], nthreads))
        return par

    def decode_any_batch(self, k: int, received: np.ndarray, erased: np.ndarray,
                         nthreads: int = 1) -> np.ndarray:
        rx = np.ascontiguousarray(received, dtype=np.uint16)
        e = np.ascontiguousarray(erased, dtype=np.uint8)
        shared = int(e.ndim == 1)
        out = np.zeros((rx.shape[0], k), np.uint16)
        _check(lib().orc_decode_any_batch(self._h, k, _p(rx), _p(e), shared, _p(out),
                                          rx.shape[0], nthreads))
        return out


def fwht(data, modulus: int) -> np.ndarray:
    x = np.ascontiguousarray(data, dtype=np.uint32).copy()
    _check(lib().orc_fwht(_p(x), x.size, modulus))
    return x


def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & (2**64 - 1)))


def gen_symbols(seed: int, r: int, cw0: int, ncw: int, length: int) -> np.ndarray:
    out = np.zeros((ncw, length), np.uint16)
    lib().orc_gen_symbols(seed, r, cw0, ncw, length, _p(out))
    return out


def gen_erasures(seed: int, n: int, count: int, cw0: int, ncw: int) -> np.ndarray:
    out = np.zeros((ncw, n), np.uint8)
    lib().orc_gen_erasures(seed, n, count, cw0, ncw, _p(out))
    return out
