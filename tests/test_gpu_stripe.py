"""GPU parity for the storage-stripe path (config 5): packet-major layout,
per-stripe-group erasure patterns, general k, lane chunking.

Lane s of stripe group g is codeword g * P + s; every check compares those
lanes with the CPU oracle (oracle/lch_oracle.c), bit-exact.  For power-of-two
k the oracle is the reference's own algorithm (pinned by the golden vectors);
for other k it is the composition of the reference primitives (orc_encode_any
/ orc_decode_any), which equals rs.encode at power-of-two k (fact iii, checked
on the CPU in test_oracle_anyk.py).
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEED = 1404345805


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


@pytest.fixture(scope="module")
def bt16(lch):
    return lch.build_basis_tables(lch.tables_for(16), 1 << 16)


def host(t):
    from paper_1404_3458_b200 import _lib
    return _lib.to_host_u16(t)


def dev(a):
    from paper_1404_3458_b200 import _lib
    return _lib.to_device_u16(np.ascontiguousarray(a))


def lanes(p):
    """[G, npos, P] -> [G * P, npos] (lane-major rows)."""
    G, npos, P = p.shape
    return np.ascontiguousarray(p.transpose(0, 2, 1).reshape(G * P, npos))


def packets(rows, P):
    """[G * P, npos] -> [G, npos, P]."""
    B, npos = rows.shape
    return np.ascontiguousarray(rows.reshape(B // P, P, npos).transpose(0, 2, 1))


def group_patterns(n, count, G, seed):
    """bool [G, n]: the `count` erased positions of each stripe group (§8d)."""
    return O.gen_erasures(seed, n, count, 0, G).astype(bool)


def bits_of(mask_rows):
    from paper_1404_3458_b200.gen import mask_to_bits
    import torch
    return mask_to_bits(torch.from_numpy(mask_rows).to("cuda")).contiguous()


def corrupt(rx_packets, mask, seed):
    """Garbage at erased packets (the decoder must ignore it)."""
    rng = np.random.default_rng(seed)
    out = rx_packets.copy()
    G = out.shape[0]
    for g in range(G):
        m = mask[g] if mask.ndim == 2 else mask
        out[g, m, :] = rng.integers(0, 1 << 16, size=(int(m.sum()), out.shape[2]),
                                    dtype=np.uint16) & np.uint16(0xFFFF)
    return out


# ---------------------------------------------------------------------------

def test_gen_packets_match_rows(lch, bt16):
    from paper_1404_3458_b200 import gen
    t = gen.packets(bt16.ctx, SEED, 5, 2, 300, 1024)
    np.testing.assert_array_equal(lanes(host(t)), O.gen_symbols(SEED, 16, 5, 2048, 300))


@pytest.mark.parametrize("lg,shift", [(1, 0), (5, 0), (6, 64), (10, 0), (16, 0), (16, 12345)])
def test_packet_transforms_r16(lch, bt16, orc16, lg, shift):
    import torch
    from paper_1404_3458_b200.transform import run_transform
    from paper_1404_3458_b200 import gen
    P, G, h = 1024, 1, 1 << lg
    sc = lch.StripeCodec(bt16, 1 << 15, P)
    a = gen.packets(bt16.ctx, SEED + lg, 0, G, h, P)
    rows = lanes(host(a))
    # row-layout GPU path (itself checked against the oracle) on the same lanes
    rt = dev(rows)
    run_transform(bt16, rt, shift, False)
    fwd_rows = host(rt)
    sc.forward_inplace(a, shift)
    np.testing.assert_array_equal(lanes(host(a)), fwd_rows)
    for b in (0, 1, 511, 1023):
        np.testing.assert_array_equal(fwd_rows[b], orc16.forward(rows[b], shift))
    sc.inverse_inplace(a, shift)
    np.testing.assert_array_equal(lanes(host(a)), rows)
    d = sc.derivative(a)
    for b in (0, 7, 1023):
        np.testing.assert_array_equal(lanes(host(d))[b], orc16.derivative(rows[b]))
    torch.cuda.synchronize()


@pytest.mark.parametrize("k", [1, 16, 128, 3, 100, 192, 240, 255])
def test_packet_encode_r8(lch, bt8, orc8, k):
    from paper_1404_3458_b200 import gen
    P, G, n = 1024, 2, 256
    sc = lch.StripeCodec(bt8, k, P)
    msg = gen.packets(bt8.ctx, SEED, 0, G, k, P)
    par = sc.encode(msg)
    want = orc8.encode_any_batch(k, lanes(host(msg)), nthreads=8)
    np.testing.assert_array_equal(lanes(host(par)), want)
    if k & (k - 1) == 0:  # the reference's own encoder (rs.encode)
        np.testing.assert_array_equal(want, orc8.encode_batch(k, lanes(host(msg)), nthreads=8))


@pytest.mark.parametrize("k,count,shared", [(128, 128, True), (128, 128, False), (128, 77, False),
                                            (192, 64, False), (100, 156, True), (100, 150, False),
                                            (1, 255, False), (255, 1, True)])
def test_packet_decode_r8(lch, bt8, orc8, k, count, shared):
    from paper_1404_3458_b200 import gen
    P, G, n = 1024, 2, 256
    sc = lch.StripeCodec(bt8, k, P)
    msg = gen.packets(bt8.ctx, SEED + k, 0, G, k, P)
    par = sc.encode(msg)
    cw = np.concatenate([host(msg), host(par)], axis=1)
    mask = group_patterns(n, count, 1 if shared else G, SEED + count)
    if shared:
        mask = mask[0]
    rx = corrupt(cw, mask, count)
    bits = bits_of(mask[None, :] if shared else mask)
    if shared:
        bits = bits[0]
    out = sc.decode(dev(rx), bits)
    np.testing.assert_array_equal(host(out), host(msg))
    # oracle on the same received lanes
    rxl = lanes(rx)
    e = np.repeat(np.repeat(mask[None, :], G, axis=0) if shared else mask, P, axis=0).astype(np.uint8)
    np.testing.assert_array_equal(lanes(host(out)), orc8.decode_any_batch(k, rxl, e, nthreads=8))


def test_packet_decode_too_many(lch, bt8):
    from paper_1404_3458_b200 import gen
    import torch
    P, G = 1024, 2
    sc = lch.StripeCodec(bt8, 192, P)
    rx = gen.packets(bt8.ctx, SEED, 0, G, 256, P)
    mask = group_patterns(256, 64, G, 3)
    mask[1, np.nonzero(~mask[1])[0][0]] = True  # group 1: 65 > n - k
    with pytest.raises(lch.TooManyErasuresError):
        sc.decode(rx, bits_of(mask))
    torch.cuda.synchronize()


@pytest.mark.parametrize("k", [100, 192, 240])
def test_row_general_k_r8(lch, bt8, orc8, k):
    """lch_encode_k / lch_decode_k on row-major batches (shared + per-row)."""
    import torch
    from paper_1404_3458_b200 import _lib
    n, B = 256, 1500
    msg = O.gen_symbols(SEED, 8, 0, B, k)
    md = dev(msg)
    pd = torch.empty((B, n - k), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_encode_k(bt8.ctx.handle, md.data_ptr(), k, pd.data_ptr(), n - k, B, k,
                                     0, _lib.stream_ptr()))
    par = host(pd)
    np.testing.assert_array_equal(par, orc8.encode_any_batch(k, msg, nthreads=8))
    cw = np.concatenate([msg, par], axis=1)
    for shared in ((True, False) if k <= 128 else (True,)):
        mask = O.gen_erasures(SEED + 1, n, n - k, 0, 1 if shared else B).astype(bool)
        rx = cw.copy()
        rx[np.broadcast_to(mask, rx.shape)] = 0xBEEF & 0xFF
        bits = bits_of(mask)
        if shared:
            bits = bits[0]
        out = torch.empty((B, k), dtype=torch.int16, device="cuda")
        _lib.check(_lib.lib.lch_decode_k(bt8.ctx.handle, dev(rx).data_ptr(), n, bits.data_ptr(),
                                         int(shared), out.data_ptr(), k, B, k, 0, None,
                                         _lib.stream_ptr()))
        np.testing.assert_array_equal(host(out), msg)


@pytest.mark.parametrize("k", [1 << 15, 49152, 61440])
def test_packet_r16_storage_codes(lch, bt16, orc16, k):
    """Config 5's three rates on two stripe groups of 1024-symbol packets."""
    import torch
    from paper_1404_3458_b200 import gen
    P, G, n = 1024, 2, 1 << 16
    sc = lch.StripeCodec(bt16, k, P)
    msg = gen.packets(bt16.ctx, SEED + 7, 0, G, k, P)
    par = sc.encode(msg)
    mh, ph = host(msg), host(par)
    sample = [0, 1, 1023, 1024, 1500, 2047]
    ml = lanes(mh)
    pl = lanes(ph)
    for b in sample:
        np.testing.assert_array_equal(pl[b], orc16.encode_any(k, ml[b])[k:])
    if k == 1 << 15:
        for b in sample[:2]:
            np.testing.assert_array_equal(pl[b], orc16.encode(k, ml[b])[k:])
    cw = np.concatenate([mh, ph], axis=1)
    del ml, pl
    mask = group_patterns(n, n - k, G, SEED + 9)
    rx = corrupt(cw, mask, 5)
    out = sc.decode(dev(rx), bits_of(mask))
    oh = host(out)
    np.testing.assert_array_equal(oh, mh)  # every lane recovers its message
    rl = lanes(rx)
    ol = lanes(oh)
    for b in (0, 1024, 2047):
        g = b // P
        np.testing.assert_array_equal(ol[b], orc16.decode_any(k, rl[b], mask[g].astype(np.uint8)))
    torch.cuda.synchronize()


def test_chunked_equals_unchunked(lch, bt16):
    """A scratch budget far below the batch forces lane chunks; results match."""
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.stripe import set_scratch_limit
    P, G, k, n = 1024, 4, 49152, 1 << 16
    sc = lch.StripeCodec(bt16, k, P)
    msg = gen.packets(bt16.ctx, SEED + 3, 0, G, k, P)
    mask = group_patterns(n, 5000, G, 11)
    bits = bits_of(mask)
    try:
        ref_par = host(sc.encode(msg))
        set_scratch_limit(bt16, 1 << 20)  # one stripe group per chunk
        par = host(sc.encode(msg))
        np.testing.assert_array_equal(par, ref_par)
        cw = dev(np.concatenate([host(msg), par], axis=1))
        out = host(sc.decode(cw, bits))
        np.testing.assert_array_equal(out, host(msg))
        a = gen.packets(bt16.ctx, SEED, 0, G, 1 << 12, P)
        a0 = host(a)
        sc.forward_inplace(a, 4096)
        f_chunk = host(a)
        set_scratch_limit(bt16, 4 << 30)
        b = dev(a0)
        sc.forward_inplace(b, 4096)
        np.testing.assert_array_equal(f_chunk, host(b))
    finally:
        set_scratch_limit(bt16, 4 << 30)


@pytest.mark.parametrize("r,k,B", [(8, 100, 1500), (8, 200, 2048), (16, 49152, 1024), (16, 40000, 1024)])
def test_general_encoder_equals_encode_by_decode(lch, bt8, bt16, r, k, B):
    """The recursive systematic encoder and the erasure-decode encoder give the
    same codeword (both are the degree < k interpolant)."""
    import os
    import torch
    from paper_1404_3458_b200 import _lib
    bt = bt8 if r == 8 else bt16
    n = 1 << r
    msg = dev(O.gen_symbols(SEED + k, r, 0, B, k))
    outs = []
    for env in (None, "1"):
        if env:
            os.environ["LCH_ENCODE_BY_DECODE"] = env
        try:
            par = torch.empty((B, n - k), dtype=torch.int16, device="cuda")
            _lib.check(_lib.lib.lch_encode_k(bt.ctx.handle, msg.data_ptr(), k, par.data_ptr(), n - k, B, k,
                                             0, _lib.stream_ptr()))
            outs.append(host(par))
        finally:
            os.environ.pop("LCH_ENCODE_BY_DECODE", None)
    np.testing.assert_array_equal(outs[0], outs[1])
    if r == 16:
        m0 = host(msg)[0]
        np.testing.assert_array_equal(outs[0][0], O.Oracle(16).encode_any(k, m0)[k:])


@pytest.mark.parametrize("k", [192, 240])
def test_row_per_codeword_general_k_above_half(lch, bt8, orc8, k):
    """Per-row patterns with k > n/2 (unfolded decode schedule), B >= 1024 so the
    bit-sliced path runs."""
    import torch
    from paper_1404_3458_b200 import _lib
    n, B = 256, 1100
    msg = O.gen_symbols(SEED + 3 * k, 8, 0, B, k)
    cw = np.concatenate([msg, orc8.encode_any_batch(k, msg, nthreads=8)], axis=1)
    masks = O.gen_erasures(SEED + 5, n, n - k, 0, B).astype(bool)
    junk = O.gen_symbols(SEED + 6, 8, 0, B, n)
    for rx, want in ((np.where(masks, 0x33, cw).astype(np.uint16), msg),
                     (junk, orc8.decode_any_batch(k, junk, masks.astype(np.uint8), nthreads=8))):
        out = torch.empty((B, k), dtype=torch.int16, device="cuda")
        bits = bits_of(masks)
        _lib.check(_lib.lib.lch_decode_k(bt8.ctx.handle, dev(rx).data_ptr(), n, bits.data_ptr(), 0,
                                         out.data_ptr(), k, B, k, 0, None, _lib.stream_ptr()))
        np.testing.assert_array_equal(host(out), want)
