"""Randomised parity sweep: random shapes, strides, shifts, k, erasure counts
and layouts against the CPU oracle (r = 8, cheap enough to check every lane)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("seed", range(12))
def test_random_transform_shapes(lch, bt8, orc8, seed):
    import torch
    from paper_1404_3458_b200 import _lib
    rng = np.random.default_rng(seed)
    lg = int(rng.integers(1, 9))
    h = 1 << lg
    B = int(rng.integers(1, 3000))
    stride = h + int(rng.integers(0, 3)) * 8
    shift = int(rng.integers(0, 256)) & ~(h - 1) if rng.random() < 0.5 else int(rng.integers(0, 256))
    a = rng.integers(0, 256, (B, stride)).astype(np.uint16)
    d = dev(a)
    fn = _lib.lib.lch_inverse if seed % 2 else _lib.lib.lch_forward
    _lib.check(fn(bt8.ctx.handle, d.data_ptr(), B, stride, lg, shift, 0, _lib.stream_ptr()))
    got = host(d)
    want = a.copy()
    want[:, :h] = orc8.transform_batch(np.ascontiguousarray(a[:, :h]), shift, bool(seed % 2), nthreads=8)
    np.testing.assert_array_equal(got, want)  # columns beyond h untouched


@pytest.mark.parametrize("seed", range(12))
def test_random_codec(lch, bt8, orc8, seed):
    import torch
    from paper_1404_3458_b200 import _lib
    from paper_1404_3458_b200.gen import mask_to_bits
    rng = np.random.default_rng(100 + seed)
    k = int(rng.integers(1, 256))
    B = int(rng.choice([int(rng.integers(1, 900)), int(rng.integers(1024, 3000))]))
    n = 256
    msg = rng.integers(0, 256, (B, k)).astype(np.uint16)
    md = dev(msg)
    pd = torch.empty((B, n - k), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_encode_k(bt8.ctx.handle, md.data_ptr(), k, pd.data_ptr(), n - k, B, k, 0,
                                     _lib.stream_ptr()))
    par = host(pd)
    np.testing.assert_array_equal(par, orc8.encode_any_batch(k, msg, nthreads=8))
    cw = np.concatenate([msg, par], axis=1)
    shared = bool(rng.random() < 0.5) or k > 128
    cnt = int(rng.integers(0, n - k + 1))
    masks = np.zeros((1 if shared else B, n), bool)
    for row in masks:
        row[rng.choice(n, cnt, replace=False)] = True
    rx = np.where(np.broadcast_to(masks, cw.shape), rng.integers(0, 256, cw.shape), cw).astype(np.uint16)
    bits = mask_to_bits(torch.from_numpy(masks).to("cuda")).contiguous()
    if shared:
        bits = bits[0]
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_decode_k(bt8.ctx.handle, dev(rx).data_ptr(), n, bits.data_ptr(), int(shared),
                                     out.data_ptr(), k, B, k, 0, None, _lib.stream_ptr()))
    np.testing.assert_array_equal(host(out), msg)


def test_per_codeword_decode_in_lane_chunks(lch, bt8, orc8):
    """A scratch budget below the batch splits per-codeword decodes into lane
    chunks (phi, -log Pi' and the bit-sliced intermediates are per codeword)."""
    import torch
    from paper_1404_3458_b200 import _lib
    from paper_1404_3458_b200.gen import mask_to_bits
    from paper_1404_3458_b200.stripe import set_scratch_limit
    n, k, B = 256, 100, 3000
    rng = np.random.default_rng(9)
    msg = rng.integers(0, 256, (B, k)).astype(np.uint16)
    cw = np.concatenate([msg, orc8.encode_any_batch(k, msg, nthreads=8)], axis=1)
    masks = np.zeros((B, n), bool)
    for row in masks:
        row[rng.choice(n, int(rng.integers(0, n - k + 1)), replace=False)] = True
    rx = np.where(masks, 7, cw).astype(np.uint16)
    bits = mask_to_bits(torch.from_numpy(masks).to("cuda")).contiguous()
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    try:
        set_scratch_limit(bt8, 1 << 20)
        _lib.check(_lib.lib.lch_decode_k(bt8.ctx.handle, dev(rx).data_ptr(), n, bits.data_ptr(), 0,
                                         out.data_ptr(), k, B, k, 0, None, _lib.stream_ptr()))
    finally:
        set_scratch_limit(bt8, 4 << 30)
    np.testing.assert_array_equal(host(out), msg)
