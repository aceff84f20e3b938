"""CPU-side checks of the product library: the C ABI loads and exports every
declared symbol, the native tables equal the reference's (golden fixtures),
host logic (validation, op-count closed forms), and no CPU fallback exists."""

import re

import numpy as np
import pytest

from golden_util import check_digest, load_r8, load_r16

import paper_1404_3458_b200 as lch
from paper_1404_3458_b200 import _lib

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def declared_symbols():
    src = open(f"{ROOT}/include/lch.h").read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(lch_[a-z0-9_]+)\s*\(", src, re.M)))


def test_abi_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(_lib.lib, s), s


def test_tables_r8_equal_reference():
    g = load_r8()
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    np.testing.assert_array_equal(ft.log, g["tab_log"])
    np.testing.assert_array_equal(ft.exp, g["tab_exp"])
    np.testing.assert_array_equal([x for lvl in bt.w_hat for x in lvl], g["tab_w_hat"])
    np.testing.assert_array_equal(bt.w_prime, g["tab_w_prime"])
    np.testing.assert_array_equal(bt.b_prod, g["tab_b_prod"])
    np.testing.assert_array_equal(bt.b_prod_inv, g["tab_b_prod_inv"])
    np.testing.assert_array_equal(bt.w_on_basis, g["tab_w_on_basis"])
    from paper_1404_3458_b200.walsh import _fwht_of_log
    np.testing.assert_array_equal(_fwht_of_log(ft), g["tab_fwht_log"])


def test_tables_r16_equal_reference():
    g = load_r16()["tables"]
    ft = lch.tables_for(16)
    bt = lch.build_basis_tables(ft, 1 << 16)
    check_digest(np.asarray(ft.log, np.uint16), g["log"])
    check_digest(np.asarray(ft.exp, np.uint16), g["exp"])
    check_digest(np.asarray([x for lvl in bt.w_hat for x in lvl], np.uint16), g["w_hat"])
    check_digest(np.asarray(bt.b_prod, np.uint16), g["b_prod"])
    check_digest(np.asarray(bt.b_prod_inv, np.uint16), g["b_prod_inv"])
    check_digest(np.asarray(ft._np["fwht_log"], np.uint32), g["fwht_log"])


def test_field_semantics_and_errors():
    ft = lch.tables_for(8)
    assert ft.mul(2, 128) == 29 and ft.inv(2) == 142
    assert ft.add(6, 3) == 5
    with pytest.raises(ZeroDivisionError):
        ft.inv(0)
    with pytest.raises(ZeroDivisionError):
        ft.div(3, 0)
    with pytest.raises(ValueError, match="not primitive"):
        lch.build_tables(lch.FieldParams(r=8, reduction_poly=0x11B))
    with pytest.raises(ValueError):
        lch.FieldParams(r=12, reduction_poly=0x1053)
    with pytest.raises(ValueError):
        lch.build_basis_tables(ft, 3)
    with pytest.raises(ValueError):
        lch.build_basis_tables(ft, 512)


def test_basis_linearity_and_roots():
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    for i in range(8):
        for j in range(256):
            assert (bt.eval_w(i, j) == 0) == (j < (1 << i))
    assert sum(len(level) for level in bt.w_hat) == 255


def test_op_count_closed_forms():
    from paper_1404_3458_b200.transform import transform_op_counts
    for lg in range(1, 9):
        h = 1 << lg
        shift = h if h < 256 else 255
        assert transform_op_counts(h, shift, 256) == (h * lg, h // 2 * lg)
        assert transform_op_counts(h, 0, 256) == (h * lg - h + 1, h // 2 * lg - h + 1)
    assert transform_op_counts(8, 8, 256) == (24, 12)
    assert transform_op_counts(8, 0, 256) == (17, 5)
    assert transform_op_counts(1, 3, 256) == (0, 0)
    # Appendix B: encode r=16 (2^16, 2^15) = 458,753 muls and 950,273 adds
    a0, m0 = transform_op_counts(1 << 15, 0, 1 << 16)
    a1, m1 = transform_op_counts(1 << 15, 1 << 15, 1 << 16)
    assert (m0 + m1, a0 + a1) == (458753, 950273)


def test_validation_before_device():
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    with pytest.raises(ValueError):
        lch.forward(bt, lch.CoeffVec([1, 2, 3]), 0)
    with pytest.raises(ValueError):
        lch.forward(bt, lch.CoeffVec([0] * 512), 0)
    with pytest.raises(ValueError):
        lch.forward(bt, lch.CoeffVec([1, 2]), 256)
    with pytest.raises(ValueError):
        lch.CodeParams(8, 3)
    cp = lch.CodeParams(8, 128)
    with pytest.raises(lch.TooManyErasuresError):
        lch.decode(cp, bt, ft, [0] * 256, lch.ErasurePattern.of(256, range(129)))
    with pytest.raises(ValueError):
        lch.locator_values(ft, [])
    with pytest.raises(ValueError):
        lch.locator_values(ft, [3, 3])
    with pytest.raises(ValueError):
        lch.locator_values(ft, range(256))
    with pytest.raises(ValueError):
        lch.fwht([1, 2, 3], 255)
    # empty pattern is a copy (rs.py:119-120), no device needed
    assert lch.decode(cp, bt, ft, list(range(256)), lch.ErasurePattern.of(256, ())) == list(range(128))


def test_no_cpu_fallback():
    if _lib.cuda_ok():
        pytest.skip("has a GPU")
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    with pytest.raises(RuntimeError):
        lch.forward(bt, lch.CoeffVec([1, 2, 3, 4]), 0)
    with pytest.raises(RuntimeError):
        lch.encode(lch.CodeParams(8, 128), bt, [0] * 128)
    # the raw ABI refuses too (no device): LCH_ECUDA
    rc = _lib.lib.lch_forward(bt.ctx.handle, None, 1, 4, 2, 0, 0, None)
    assert rc == _lib.LCH_ECUDA


def test_general_k_and_packet_validation_before_device():
    """lch_encode_k / lch_decode_k / host pipeline argument checks run before
    any device access (so they hold on CPU-only hosts)."""
    import ctypes
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    h = bt.ctx.handle
    L = _lib.lib
    EINVAL = _lib.LCH_EINVAL
    buf = (ctypes.c_uint16 * 4096)()
    p = ctypes.addressof(buf)
    p16 = p + (16 - p % 16) % 16  # 16-byte aligned
    # k outside [1, n]
    assert L.lch_encode_k(h, p16, 256, p16, 256, 1, 0, 0, None) == EINVAL
    assert L.lch_encode_k(h, p16, 256, p16, 256, 1, 257, 0, None) == EINVAL
    # strides too small
    assert L.lch_encode_k(h, p16, 99, p16, 156, 1, 100, 0, None) == EINVAL
    assert L.lch_encode_k(h, p16, 100, p16, 155, 1, 100, 0, None) == EINVAL
    # packet_len not a multiple of 1024, batch not a multiple of packet_len, misaligned
    assert L.lch_encode_k(h, p16, 128, p16, 128, 1000, 128, 1000, None) == EINVAL
    assert L.lch_encode_k(h, p16, 128, p16, 128, 1500, 128, 1024, None) == EINVAL
    assert L.lch_encode_k(h, p16 + 2, 128, p16, 128, 1024, 128, 1024, None) == EINVAL
    # decode: k range, strides, missing bitmask
    assert L.lch_decode_k(h, p16, 256, p16, 1, p16, 128, 1, 0, 0, None, None) == EINVAL
    assert L.lch_decode_k(h, p16, 255, p16, 1, p16, 128, 1, 128, 0, None, None) == EINVAL
    assert L.lch_decode_k(h, p16, 256, None, 1, p16, 128, 1, 128, 0, None, None) == EINVAL
    # host pipeline
    assert L.lch_encode_host(h, None, 128, p16, 128, 1, 128, 0, 0, None) == EINVAL
    assert L.lch_decode_host(h, p16, 256, None, 1, p16, 128, 1, 128, 0, 0, None) == EINVAL
    assert L.lch_decode_host(h, p16, 256, p16, 1, p16, 128, 1, 128, 1000, 0, None) == EINVAL
    assert L.lch_set_scratch_limit(h, 0) == EINVAL
    with pytest.raises(ValueError):
        lch.StripeCodec(bt, 0, 1024)
    with pytest.raises(ValueError):
        lch.StripeCodec(bt, 128, 1000)


def test_host_pipeline_too_many_from_host_counts():
    """lch_decode_host counts erasures from the host bitmask (rs.py:121-123)
    before any device work."""
    import ctypes
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    bits = np.zeros(8, np.uint32)
    bits[:5] = 0xFFFFFFFF  # 160 erasures > n - k = 128
    rx = np.zeros((1, 256), np.uint16)
    out = np.zeros((1, 128), np.uint16)
    rc = _lib.lib.lch_decode_host(bt.ctx.handle, rx.ctypes.data, 256, bits.ctypes.data, 1,
                                  out.ctypes.data, 128, 1, 128, 0, 0, None)
    assert rc in (_lib.LCH_ETOOMANY, _lib.LCH_ECUDA)
    if not _lib.cuda_ok():
        # ensure_device() runs first on a CPU-only host
        assert rc == _lib.LCH_ECUDA
    with pytest.raises(Exception):
        lch.BatchCodec(lch.CodeParams(8, 128), bt).decode(rx, set(range(129)))


def test_host_compaction_of_survivors():
    """lch_compact_rows (host side of the decode pipeline): survivors in order,
    vector and scalar paths (n multiple of 32 or not)."""
    ft = lch.tables_for(8)
    bt = lch.build_basis_tables(ft, 256)
    rng = np.random.default_rng(4)
    for n in (256, 96, 40):
        rows = 37
        rx = rng.integers(0, 65536, (rows, n + 3)).astype(np.uint16)  # stride n + 3
        mask = rng.random(n) < 0.45
        bits = _lib.bitmask_from_positions(n, np.nonzero(mask)[0])
        surv = int((~mask).sum())
        out = np.zeros((rows, surv + 1), np.uint16)
        rc = _lib.lib.lch_compact_rows(bt.ctx.handle, rx.ctypes.data, n + 3, bits.ctypes.data, n, rows,
                                       out.ctypes.data, surv + 1)
        assert rc == _lib.LCH_OK
        np.testing.assert_array_equal(out[:, :surv], rx[:, :n][:, ~mask])
