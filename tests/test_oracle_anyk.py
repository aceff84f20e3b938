"""General-k oracle (config 5 rates 3/4 and 15/16) pinned to
vectors composed from the reference's own primitives (tests/golden/
make_golden.py: locator_values, inverse, derivative_fast, forward)."""

import json
import os

import numpy as np

from golden_util import check_digest, load_r8
from oracle import oracle as O

G8 = load_r8()
HERE = os.path.dirname(os.path.abspath(__file__))


def test_anyk_r8_match_reference_composition(orc8):
    for k in (3, 100, 192, 240, 255):
        for m, cw, mask, rx in zip(G8[f"anyk{k}_msg"], G8[f"anyk{k}_cw"], G8[f"anyk{k}_mask"],
                                   G8[f"anyk{k}_rx"]):
            np.testing.assert_array_equal(orc8.encode_any(k, m), cw)
            np.testing.assert_array_equal(orc8.recover_all(rx, mask), cw)
            np.testing.assert_array_equal(orc8.decode_any(k, rx, mask), m)


def test_anyk_equals_rs_encode_for_power_of_two(orc8):
    """Fact (iii): encode-by-erasure-decode = rs.encode for power-of-two k."""
    for k in (1, 2, 4, 16, 64, 256):
        for m, cw in zip(G8[f"k{k}_msg"], G8[f"k{k}_cw"]):
            np.testing.assert_array_equal(orc8.encode_any(k, m), cw)


def test_anyk_mds_r8(orc8):
    rng = np.random.default_rng(3)
    for k in (5, 77, 130, 200):
        m = rng.integers(0, 256, k).astype(np.uint16)
        cw = orc8.encode_any(k, m)
        for _ in range(4):
            e = np.zeros(256, np.uint8)
            e[rng.choice(256, int(rng.integers(1, 256 - k + 1)), replace=False)] = 1
            rx = np.where(e == 1, rng.integers(0, 256, 256), cw).astype(np.uint16)
            np.testing.assert_array_equal(orc8.decode_any(k, rx, e), m)


def test_anyk_too_many(orc8):
    import pytest
    e = np.zeros(256, np.uint8)
    e[:57] = 1
    with pytest.raises(Exception):
        orc8.decode_any(200, np.zeros(256, np.uint16), e)


def test_anyk_r16_match_reference_composition(orc16):
    with open(os.path.join(HERE, "golden", "golden_r16_anyk.json")) as f:
        cases = json.load(f)
    n = 1 << 16
    for c in cases:
        k = c["k"]
        m = O.gen_symbols(c["seed"], 16, c["cw"], 1, k)[0]
        cw = orc16.encode_any(k, m)
        check_digest(cw[k:], c["parity"])
        mask = O.gen_erasures(c["erasure_seed"], n, n - k, 0, 1)[0]
        check_digest(np.nonzero(mask)[0].astype(np.uint32), {"sha256": c["pattern_sha256"]})
        junk = O.gen_symbols(c["junk_seed"], 16, 0, 1, n)[0]
        rx = np.where(mask == 1, junk, cw).astype(np.uint16)
        np.testing.assert_array_equal(orc16.decode_any(k, rx, mask), m)
        check_digest(orc16.decode_any(k, junk, mask), c["junk_out"])


def test_batch_decode_shared_locator_equals_per_row(orc8, orc16):
    """A shared erasure set evaluates the locator once per batch
    (batch.py:126-139); the result must equal the per-row decodes, for the
    power-of-two codec and the general-k composition, on non-codewords too."""
    for orc, r, ks in ((orc8, 8, (128, 100)), (orc16, 16, (1 << 15, 49152))):
        n = 1 << r
        for k in ks:
            mask = O.gen_erasures(77 + k, n, n - k, 0, 1)[0]
            junk = O.gen_symbols(78 + k, r, 0, 3, n)
            if k & (k - 1) == 0:
                a = orc.decode_batch(k, junk, mask, 2)
                b = np.stack([orc.decode(k, junk[i], mask) for i in range(3)])
                c = orc.decode_batch(k, junk, np.stack([mask] * 3), 2)
                np.testing.assert_array_equal(a, b)
                np.testing.assert_array_equal(a, c)
            a = orc.decode_any_batch(k, junk, mask, 2)
            b = np.stack([orc.decode_any(k, junk[i], mask) for i in range(3)])
            np.testing.assert_array_equal(a, b)

