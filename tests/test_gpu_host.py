"""Host-buffer pipeline (lch_encode_host / lch_decode_host): chunked H2D /
kernel / D2H overlap must give exactly the device-path results, which are
themselves pinned to the oracle (test_gpu_parity.py, test_gpu_stripe.py)."""

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


@pytest.fixture(scope="module")
def bt16(lch):
    return lch.build_basis_tables(lch.tables_for(16), 1 << 16)


def pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.int16, pin_memory=True)
    t.numpy().view(np.uint16)[...] = a
    return t


@pytest.mark.parametrize("chunk", [0, 1, 7, 700])
def test_encode_decode_host_r8(lch, bt8, orc8, chunk):
    import torch
    from paper_1404_3458_b200.rs import decode_host, encode_host
    cp = lch.CodeParams(8, 128)
    B = 1500
    msg = O.gen_symbols(11, 8, 0, B, 128)
    hm = pinned(msg)
    hp = torch.empty((B, 128), dtype=torch.int16, pin_memory=True)
    encode_host(cp, bt8, hm, hp, chunk)
    torch.cuda.synchronize()
    par = hp.numpy().view(np.uint16)
    np.testing.assert_array_equal(par, orc8.encode_batch(128, msg, nthreads=8))
    cw = np.concatenate([msg, par], axis=1)
    # shared pattern
    mask = O.gen_erasures(12, 256, 128, 0, 1)[0].astype(bool)
    rx = cw.copy()
    rx[:, mask] = 0x55
    out = torch.empty((B, 128), dtype=torch.int16, pin_memory=True)
    from paper_1404_3458_b200._lib import bitmask_from_positions
    hrx = pinned(rx)
    decode_host(cp, bt8, hrx, bitmask_from_positions(256, np.nonzero(mask)[0]), out, chunk)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.numpy().view(np.uint16), msg)
    # per-codeword patterns
    masks = O.gen_erasures(13, 256, 128, 0, B).astype(bool)
    rx = np.where(masks, 0x77, cw).astype(np.uint16)
    bits = np.stack([bitmask_from_positions(256, np.nonzero(m)[0]) for m in masks])
    out2 = torch.empty((B, 128), dtype=torch.int16, pin_memory=True)
    hrx2 = pinned(rx)
    decode_host(cp, bt8, hrx2, bits, out2, chunk)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out2.numpy().view(np.uint16), msg)


def test_batchcodec_numpy_paths(lch, bt8, orc8):
    cp = lch.CodeParams(8, 64)
    codec = lch.BatchCodec(cp, bt8)
    msg = O.gen_symbols(21, 8, 0, 300, 64)
    cw = codec.encode(msg)
    assert isinstance(cw, np.ndarray) and cw.shape == (300, 256)
    np.testing.assert_array_equal(cw[:, :64], msg)
    np.testing.assert_array_equal(cw[:, 64:], orc8.encode_batch(64, msg, nthreads=8))
    erased = set(range(0, 256, 2)) | {1, 3, 5}
    rx = cw.copy()
    rx[:, sorted(erased)] = 0
    np.testing.assert_array_equal(codec.decode(rx, erased), msg)
    with pytest.raises(lch.TooManyErasuresError):
        codec.decode(rx, set(range(193)))


def test_host_r16_matches_device(lch, bt16):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, decode_host, encode_device, encode_host
    cp = lch.CodeParams(16, 1 << 15)
    B, K, N = 600, 1 << 15, 1 << 16
    dmsg = gen.symbols(bt16.ctx, 5, 0, B, K)
    dpar = torch.empty((B, K), dtype=torch.int16, device="cuda")
    encode_device(cp, bt16, dmsg, dpar)
    hm = dmsg.cpu().pin_memory()
    hp = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
    encode_host(cp, bt16, hm, hp, 128)
    torch.cuda.synchronize()
    assert torch.equal(hp, dpar.cpu())
    mask = gen.erasure_masks(bt16.ctx, 6, N, N - K, 0, 1)
    bits_d = gen.mask_to_bits(mask)[0].contiguous()
    rx = torch.cat([dmsg, dpar], dim=1)
    rx[:, mask[0]] = 0
    hout = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
    hrx = rx.cpu().pin_memory()  # kept alive until the stream is synchronised
    decode_host(cp, bt16, hrx, bits_d.cpu().numpy().view(np.uint32), hout, 200)
    torch.cuda.synchronize()
    assert torch.equal(hout, dmsg.cpu())


@pytest.mark.parametrize("k", [192, 100])
def test_packet_host_pipeline(lch, bt8, k):
    """Packet layout through the host pipeline (rows = stripe groups); k = 100
    erases > 40 % of the packets, so surviving packets are packed on the host."""
    import torch
    from paper_1404_3458_b200 import _lib, gen
    P, G, n = 1024, 5, 256
    sc = lch.StripeCodec(bt8, k, P)
    msg = gen.packets(bt8.ctx, 31, 0, G, k, P)
    par = sc.encode(msg)
    hm = msg.cpu().pin_memory()
    hp = torch.empty((G, n - k, P), dtype=torch.int16, pin_memory=True)
    _lib.check(_lib.lib.lch_encode_host(bt8.ctx.handle, hm.data_ptr(), k, hp.data_ptr(), n - k, G * P, k,
                                        P, 2, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(hp, par.cpu())
    masks = O.gen_erasures(32, n, n - k, 0, G).astype(bool)
    from paper_1404_3458_b200._lib import bitmask_from_positions
    bits = np.stack([bitmask_from_positions(n, np.nonzero(m)[0]) for m in masks])
    rx = torch.cat([hm, hp], dim=1)
    for g in range(G):
        rx[g, torch.from_numpy(masks[g])] = 0
    hout = torch.empty((G, k, P), dtype=torch.int16, pin_memory=True)
    hrx = rx.pin_memory()
    _lib.check(_lib.lib.lch_decode_host(bt8.ctx.handle, hrx.data_ptr(), n, bits.ctypes.data, 0,
                                        hout.data_ptr(), k, G * P, k, P, 2, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(hout, hm)


@pytest.mark.parametrize("count", [0, 1, 128])
def test_decode_host_edge_counts(lch, bt8, orc8, count):
    """Host pipeline with the survivor compaction: empty pattern (copy), a
    single erasure, and the maximum; a batch that is not a multiple of the chunk."""
    import torch
    from paper_1404_3458_b200._lib import bitmask_from_positions
    from paper_1404_3458_b200.rs import decode_host
    cp = lch.CodeParams(8, 128)
    B = 1300
    msg = O.gen_symbols(41, 8, 0, B, 128)
    cw = np.concatenate([msg, orc8.encode_batch(128, msg, nthreads=8)], axis=1)
    erased = np.sort(np.random.default_rng(count).choice(256, count, replace=False))
    rx = cw.copy()
    rx[:, erased] = 0xEE
    hrx = pinned(rx)
    out = torch.empty((B, 128), dtype=torch.int16, pin_memory=True)
    decode_host(cp, bt8, hrx, bitmask_from_positions(256, erased), out, 500)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.numpy().view(np.uint16), msg)


def test_back_to_back_decode_host_calls_keep_their_staging(lch, bt16):
    """Two decode_host calls on different buffers queued without a host sync
    in between (the survivor-compaction path reuses the context's page-locked
    staging slots): each must decode its own rows (lch_api.cu
    host_pipeline)."""
    import torch
    from paper_1404_3458_b200._lib import bitmask_from_positions
    from paper_1404_3458_b200.rs import decode_host, encode_host
    n, k, B = 1 << 16, 1 << 15, 96
    cp = lch.CodeParams(16, k)
    mask = O.gen_erasures(21, n, n - k, 0, 1)[0].astype(bool)
    bits = bitmask_from_positions(n, np.nonzero(mask)[0])
    rxs, outs, msgs = [], [], []
    for seed in (31, 32, 33):
        msg = O.gen_symbols(seed, 16, 0, B, k)
        hp = torch.empty((B, n - k), dtype=torch.int16, pin_memory=True)
        encode_host(cp, bt16, pinned(msg), hp)
        torch.cuda.synchronize()
        rx = np.concatenate([msg, hp.numpy().view(np.uint16)], axis=1)
        rx[:, mask] = 0
        rxs.append(pinned(rx))
        outs.append(torch.empty((B, k), dtype=torch.int16, pin_memory=True))
        msgs.append(msg)
    for hrx, out in zip(rxs, outs):
        decode_host(cp, bt16, hrx, bits, out, 8)  # chunks of 8 rows: many staging slots in flight
    torch.cuda.synchronize()
    for out, msg in zip(outs, msgs):
        np.testing.assert_array_equal(out.numpy().view(np.uint16), msg)


def test_interleaved_host_calls_overlap_across_calls(lch, bt16):
    """encode_host / decode_host queued alternately on different buffers with a
    single host sync at the end: the persistent pipeline slots let the copies
    of one call overlap the tail of the previous one, and every call must
    still produce its own result (slot reuse is ordered by the context's
    per-slot events across calls)."""
    import torch
    from paper_1404_3458_b200._lib import bitmask_from_positions
    from paper_1404_3458_b200.rs import decode_host, encode_host
    n, k, B = 1 << 16, 1 << 15, 2100
    cp = lch.CodeParams(16, k)
    mask = O.gen_erasures(22, n, n - k, 0, 1)[0].astype(bool)
    bits = bitmask_from_positions(n, np.nonzero(mask)[0])
    msgs = [O.gen_symbols(seed, 16, 0, B, k) for seed in (51, 52, 53)]
    hmsgs = [pinned(m) for m in msgs]
    refs = []
    for hm in hmsgs:  # reference parity, one call at a time
        hp = torch.empty((B, n - k), dtype=torch.int16, pin_memory=True)
        encode_host(cp, bt16, hm, hp)
        torch.cuda.synchronize()
        refs.append(hp.numpy().view(np.uint16).copy())
    rxs = []
    for m, p in zip(msgs, refs):
        rx = np.concatenate([m, p], axis=1)
        rx[:, mask] = 0xABCD
        rxs.append(pinned(rx))
    pars = [torch.empty((B, n - k), dtype=torch.int16, pin_memory=True) for _ in msgs]
    outs = [torch.empty((B, k), dtype=torch.int16, pin_memory=True) for _ in msgs]
    for chunk in (0, 300):
        for t in pars + outs:
            t.zero_()
        for hm, hp, hrx, out in zip(hmsgs, pars, rxs, outs):
            encode_host(cp, bt16, hm, hp, chunk)
            decode_host(cp, bt16, hrx, bits, out, chunk)
        torch.cuda.synchronize()
        for m, p, hp, out in zip(msgs, refs, pars, outs):
            np.testing.assert_array_equal(hp.numpy().view(np.uint16), p)
            np.testing.assert_array_equal(out.numpy().view(np.uint16), m)
    # one sampled row against the oracle
    orc = O.Oracle(16)
    np.testing.assert_array_equal(refs[1][7], orc.encode(k, msgs[1][7])[k:])


def test_stream_ordered_host_inputs(lch, bt16):
    """lch_set_host_ordering(ctx, 1): a call may read a host buffer that an
    earlier call on the same stream is still writing (parity of the parity,
    chained without a host sync); released buffers are re-created on demand."""
    import torch
    from paper_1404_3458_b200 import _lib
    from paper_1404_3458_b200.rs import encode_device, encode_host
    n, k, B = 1 << 16, 1 << 15, 1500
    cp = lch.CodeParams(16, k)
    msg = O.gen_symbols(61, 16, 0, B, k)
    hm = pinned(msg)
    p1 = torch.zeros((B, k), dtype=torch.int16, pin_memory=True)
    p2 = torch.zeros((B, k), dtype=torch.int16, pin_memory=True)
    h = bt16.ctx.handle
    _lib.check(_lib.lib.lch_release_host_buffers(h))
    _lib.check(_lib.lib.lch_set_host_ordering(h, 1))
    try:
        encode_host(cp, bt16, hm, p1, 256)
        encode_host(cp, bt16, p1, p2, 256)
        torch.cuda.synchronize()
    finally:
        _lib.check(_lib.lib.lch_set_host_ordering(h, 0))
    d1 = torch.empty((B, k), dtype=torch.int16, device="cuda")
    d2 = torch.empty((B, k), dtype=torch.int16, device="cuda")
    encode_device(cp, bt16, hm.cuda(), d1)
    encode_device(cp, bt16, d1, d2)
    torch.cuda.synchronize()
    assert torch.equal(p1, d1.cpu())
    assert torch.equal(p2, d2.cpu())


@pytest.mark.parametrize("mode", ["all", "alt", "none", "auto"])
def test_decode_host_compaction_modes(lch, bt16, mode, monkeypatch):
    """Shared-pattern decode_host with the survivors compacted on the host for
    all / every other / no / automatically chosen chunks (LCH_COMPACT): the
    same output in every mode, non-codeword rows included."""
    import torch
    from paper_1404_3458_b200._lib import bitmask_from_positions
    from paper_1404_3458_b200.rs import decode_host
    n, k, B = 1 << 16, 1 << 15, 700
    cp = lch.CodeParams(16, k)
    mask = O.gen_erasures(71, n, n - k, 0, 1)[0].astype(bool)
    bits = bitmask_from_positions(n, np.nonzero(mask)[0])
    rx = O.gen_symbols(72, 16, 0, B, n)  # arbitrary received words (not codewords)
    hrx = pinned(rx)
    monkeypatch.setenv("LCH_COMPACT", mode)
    out = torch.zeros((B, k), dtype=torch.int16, pin_memory=True)
    decode_host(cp, bt16, hrx, bits, out, 96)
    torch.cuda.synchronize()
    got = out.numpy().view(np.uint16)
    orc = O.Oracle(16)
    for r in (0, 95, 96, 191, B - 1):
        np.testing.assert_array_equal(got[r], orc.decode(k, rx[r], mask.astype(np.uint8)))
    monkeypatch.setenv("LCH_COMPACT", "all")
    ref = torch.zeros((B, k), dtype=torch.int16, pin_memory=True)
    decode_host(cp, bt16, hrx, bits, ref, 0)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
