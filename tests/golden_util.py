"""Helpers shared by the parity tests: golden fixtures + the input generator."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def load_r8() -> dict:
    with np.load(os.path.join(GOLDEN, "golden_r8.npz")) as z:
        return {k: z[k] for k in z.files}


def load_r16() -> dict:
    with open(os.path.join(GOLDEN, "golden_r16.json")) as fh:
        return json.load(fh)


def digest(a) -> str:
    a = np.asarray(a)
    dt = "<u4" if a.dtype == np.uint32 else "<u2"
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def check_digest(a, entry: dict) -> None:
    a = np.asarray(a).ravel()
    s = entry.get("sample")
    if s:
        got = [int(a[i]) for i in s["idx"]]
        assert got == s["val"], "sampled entries differ from the reference"
    assert digest(a) == entry["sha256"], "sha256 differs from the reference"


M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    """Pure-Python restatement of the SplitMix64 finaliser."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key(seed: int, cw: int, pos: int) -> int:
    s = mix64(seed + GAMMA)
    return mix64(s + (((cw << 32) | pos) * GAMMA))


def gen_symbols_py(seed: int, r: int, cw: int, length: int) -> list[int]:
    mask = (1 << r) - 1
    return [key(seed, cw, j) & mask for j in range(length)]


def gen_erasures_py(seed: int, n: int, count: int, cw: int) -> list[int]:
    order = sorted(range(n), key=lambda j: (key(seed, cw, j) >> 1, j))
    return sorted(order[:count])


def tr_cases(g: dict):
    """Yield (h, shift, input, fwd, inv, der) from golden_r8 transform cases."""
    off = 0
    for h, shift in g["tr_meta"]:
        h = int(h)
        sl = slice(off, off + h)
        yield h, int(shift), g["tr_in"][sl], g["tr_fwd"][sl], g["tr_inv"][sl], g["tr_der"][sl]
        off += h
