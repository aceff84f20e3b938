"""GF(2^8) small-batch codec (one CTA per codeword, csrc/lch_small.cu) vs the
oracle, and vs the bit-sliced batched path on the same inputs."""

import os

import numpy as np
import pytest

from golden_util import load_r8
from oracle import oracle as O

pytestmark = pytest.mark.gpu
G8 = load_r8()


@pytest.fixture(scope="module")
def lch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_3458_b200 as m
    return m


@pytest.fixture(scope="module")
def bt8(lch):
    return lch.build_basis_tables(lch.tables_for(8), 256)


def host(t):
    from paper_1404_3458_b200 import _lib
    return _lib.to_host_u16(t)


def dev(a):
    from paper_1404_3458_b200 import _lib
    return _lib.to_device_u16(np.ascontiguousarray(a))


def bits_of(mask_rows):
    import torch
    from paper_1404_3458_b200.gen import mask_to_bits
    return mask_to_bits(torch.from_numpy(np.asarray(mask_rows, bool)).to("cuda")).contiguous()


def enc(bt8, msg, k):
    import torch
    from paper_1404_3458_b200 import _lib
    B = msg.shape[0]
    md = dev(msg)
    pd = torch.empty((B, 256 - k), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_encode_k(bt8.ctx.handle, md.data_ptr(), k, pd.data_ptr(), 256 - k, B, k, 0,
                                     _lib.stream_ptr()))
    return host(pd)


def dec(bt8, rx, mask, k, shared):
    import torch
    from paper_1404_3458_b200 import _lib
    B = rx.shape[0]
    bits = bits_of(mask if mask.ndim == 2 else mask[None, :])
    if shared:
        bits = bits[0]
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    rd = dev(rx)
    _lib.check(_lib.lib.lch_decode_k(bt8.ctx.handle, rd.data_ptr(), 256, bits.data_ptr(), int(shared),
                                     out.data_ptr(), k, B, k, 0, None, _lib.stream_ptr()))
    return host(out)


@pytest.mark.parametrize("k", [1, 2, 4, 8, 16, 32, 64, 128])
def test_small8_encode(lch, bt8, orc8, k):
    msg = O.gen_symbols(1404345801, 8, 0, 64, k)
    np.testing.assert_array_equal(enc(bt8, msg, k), orc8.encode_batch(k, msg, nthreads=8))


def test_small8_cfg1_golden(lch, bt8):
    """Config 1 exactly as the reference ran it (golden_r8.npz cfg1_*)."""
    msg, cw, mask = G8["cfg1_msg"], G8["cfg1_cw"], G8["cfg1_mask"].astype(bool)
    np.testing.assert_array_equal(enc(bt8, msg, 128), cw[:, 128:])
    rx = np.where(mask, 0, cw).astype(np.uint16)
    np.testing.assert_array_equal(dec(bt8, rx, mask, 128, False), msg)
    junk = np.stack([O.gen_symbols(1404345801 ^ 0x5A5A, 8, row, 1, 256)[0] for row in range(64)])
    np.testing.assert_array_equal(dec(bt8, junk, mask, 128, False), G8["cfg1_junk_dec"])


@pytest.mark.parametrize("k,count,shared", [(128, 128, False), (128, 128, True), (128, 3, False),
                                            (100, 156, False), (192, 64, True), (1, 255, False),
                                            (255, 1, False), (64, 0, False)])
def test_small8_decode(lch, bt8, orc8, k, count, shared):
    B = 300
    msg = O.gen_symbols(77 + k, 8, 0, B, k)
    cw = np.concatenate([msg, orc8.encode_any_batch(k, msg, nthreads=8)], axis=1)
    mask = O.gen_erasures(78 + count, 256, count, 0, 1 if shared else B).astype(bool)
    if shared:
        mask = mask[0]
    rx = np.where(np.broadcast_to(mask, cw.shape), 0xA5, cw).astype(np.uint16)
    out = dec(bt8, rx, mask, k, shared)
    np.testing.assert_array_equal(out, msg)
    # non-codeword input: every internal stage shows in the output
    junk = O.gen_symbols(79, 8, 0, B, 256)
    e = np.broadcast_to(mask, (B, 256)).astype(np.uint8)
    np.testing.assert_array_equal(dec(bt8, junk, mask, k, shared),
                                  orc8.decode_any_batch(k, junk, np.ascontiguousarray(e), nthreads=8))


def test_small8_matches_bitsliced_path(lch, bt8):
    B, k = 700, 128
    msg = O.gen_symbols(5, 8, 0, B, k)
    masks = O.gen_erasures(6, 256, 128, 0, B).astype(bool)
    junk = O.gen_symbols(7, 8, 0, B, 256)
    a_par, a_dec = enc(bt8, msg, k), dec(bt8, junk, masks, k, False)
    os.environ["LCH_NO_SMALL8"] = "1"
    try:
        b_par, b_dec = enc(bt8, msg, k), dec(bt8, junk, masks, k, False)
    finally:
        del os.environ["LCH_NO_SMALL8"]
    np.testing.assert_array_equal(a_par, b_par)
    np.testing.assert_array_equal(a_dec, b_dec)
