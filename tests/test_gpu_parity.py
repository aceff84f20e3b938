"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle, which is
itself pinned to the reference (test_oracle_golden.py).  Integer/byte work:
the bar is bit-exact equality."""

import numpy as np
import pytest

from golden_util import check_digest, load_r8, load_r16, tr_cases
from oracle import oracle as O

pytestmark = pytest.mark.gpu

G8 = load_r8()
G16 = load_r16()


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


def dev(a):
    from paper_1404_3458_b200 import _lib
    return _lib.to_device_u16(a)


def host(t):
    from paper_1404_3458_b200 import _lib
    return _lib.to_host_u16(t)


def gen(bt, seed, cw0, batch, length):
    import torch
    from paper_1404_3458_b200 import _lib
    t = torch.empty((batch, length), dtype=torch.int16, device="cuda")
    _lib.check(_lib.lib.lch_gen_symbols(bt.ctx.handle, seed, cw0, batch, length, t.data_ptr(),
                                        length, _lib.stream_ptr()))
    return t


def sample_rows(batch, extra=()):
    rows = {0, 1, 31, 32, 1023, batch - 1} | set(extra)
    rng = np.random.default_rng(batch)
    rows |= set(rng.choice(batch, size=min(12, batch), replace=False).tolist())
    return sorted(r for r in rows if 0 <= r < batch)


def test_gen_symbols_match_oracle(lch, bt16):
    t = gen(bt16, 1404345803, 7, 5, 1000)
    np.testing.assert_array_equal(host(t), O.gen_symbols(1404345803, 16, 7, 5, 1000))


def test_transforms_r8_golden_single(lch, bt8):
    for h, shift, d, fwd, inv, der in tr_cases(G8):
        d = [int(x) for x in d]
        assert lch.forward(bt8, lch.CoeffVec(d), shift).data == fwd.tolist()
        assert lch.inverse(bt8, lch.EvalVec(d, shift)).data == inv.tolist()
        assert lch.derivative_fast(bt8, lch.CoeffVec(d)).data == der.tolist()


@pytest.mark.parametrize("lg", range(1, 9))
def test_transforms_r8_batched_vs_oracle(lch, bt8, orc8, lg):
    from paper_1404_3458_b200.transform import run_transform
    from paper_1404_3458_b200.derivative import run_derivative
    h = 1 << lg
    B = 2100  # three 1024-lane groups, the last one partial
    x = gen(bt8, 11 + lg, 0, B, h)
    ref_in = host(x)
    for shift in sorted({0, h % 256, 77, 255}):
        y = x.clone()
        run_transform(bt8, y, shift, False)
        np.testing.assert_array_equal(host(y), orc8.transform_batch(ref_in, shift, False, 8))
        z = x.clone()
        run_transform(bt8, z, shift, True)
        np.testing.assert_array_equal(host(z), orc8.transform_batch(ref_in, shift, True, 8))
    d = x.clone()
    run_derivative(bt8, x, d)
    got = host(d)
    for r in sample_rows(B):
        np.testing.assert_array_equal(got[r], orc8.derivative(ref_in[r]))


@pytest.mark.parametrize("lg", [1, 3, 5, 6, 10, 15, 16])
def test_transforms_r16_vs_oracle(lch, bt16, orc16, lg):
    from paper_1404_3458_b200.transform import run_transform
    from paper_1404_3458_b200.derivative import run_derivative
    h = 1 << lg
    B = 1030 if lg >= 10 else 2100
    x = gen(bt16, 1404345802, 100 + lg, B, h)
    ref_in = host(x)
    rows = sample_rows(B)
    for shift in (0, 12345 % (1 << 16), h % (1 << 16)):
        y = x.clone()
        run_transform(bt16, y, shift, False)
        got = host(y)
        for r in rows:
            np.testing.assert_array_equal(got[r], orc16.forward(ref_in[r], shift), err_msg=f"row {r}")
        # full-batch round trip on the device
        run_transform(bt16, y, shift, True)
        np.testing.assert_array_equal(host(y), ref_in)
    z = x.clone()
    run_transform(bt16, z, 0, True)
    got = host(z)
    for r in rows:
        np.testing.assert_array_equal(got[r], orc16.inverse(ref_in[r], 0))
    d = x.clone()
    run_derivative(bt16, x, d)
    got = host(d)
    for r in rows[:6]:
        np.testing.assert_array_equal(got[r], orc16.derivative(ref_in[r]))


def test_transforms_r16_golden(lch, bt16):
    from paper_1404_3458_b200.transform import run_transform
    from paper_1404_3458_b200.derivative import run_derivative
    for c in G16["transform"]:
        x = gen(bt16, c["seed"], c["cw"], 1, c["h"])
        y = x.clone()
        run_transform(bt16, y, c["shift"], False)
        check_digest(host(y)[0], c["fwd"])
        y = x.clone()
        run_transform(bt16, y, c["shift"], True)
        check_digest(host(y)[0], c["inv"])
        d = x.clone()
        run_derivative(bt16, x, d)
        check_digest(host(d)[0], c["der"])


@pytest.mark.parametrize("k", [1, 2, 4, 16, 32, 64, 128, 256])
def test_encode_r8_all_k_vs_oracle(lch, bt8, orc8, k):
    cp = lch.CodeParams(8, k)
    codec = lch.BatchCodec(cp, bt8)
    msgs = O.gen_symbols(1404345801, 8, 0, 1500, k)
    enc = codec.encode(msgs)
    assert enc.shape == (1500, 256)
    np.testing.assert_array_equal(enc[:, :k], msgs)
    if k < 256:
        np.testing.assert_array_equal(enc[:, k:], orc8.encode_batch(k, msgs, 8))


def test_encode_r8_golden(lch, bt8):
    cp = lch.CodeParams(8, 128)
    for m, cw in zip(G8["cfg1_msg"], G8["cfg1_cw"]):
        assert lch.encode(cp, bt8, [int(x) for x in m]).symbols == cw.tolist()
    for k in (1, 2, 4, 16, 64, 256):
        enc = lch.BatchCodec(lch.CodeParams(8, k), bt8).encode(G8[f"k{k}_msg"])
        np.testing.assert_array_equal(enc, G8[f"k{k}_cw"])


def test_encode_r16_vs_oracle(lch, bt16, orc16):
    import torch
    from paper_1404_3458_b200.rs import encode_device
    k = 1 << 15
    cp = lch.CodeParams(16, k)
    B = 1100
    msg = gen(bt16, 1404345803, 0, B, k)
    par = torch.empty((B, k), dtype=torch.int16, device="cuda")
    encode_device(cp, bt16, msg, par)
    got, m = host(par), host(msg)
    for c in G16["encode"]:
        check_digest(got[c["cw"]], c["parity"])
    for r in sample_rows(B):
        np.testing.assert_array_equal(got[r], orc16.encode(k, m[r])[k:], err_msg=f"row {r}")


@pytest.mark.parametrize("lgk", [4, 8, 12, 14])
def test_encode_r16_small_k_vs_oracle(lch, bt16, orc16, lgk):
    k = 1 << lgk
    codec = lch.BatchCodec(lch.CodeParams(16, k), bt16)
    msgs = O.gen_symbols(lgk, 16, 0, 33, k)
    enc = codec.encode(msgs)
    for r in (0, 17, 32):
        np.testing.assert_array_equal(enc[r], orc16.encode(k, msgs[r]))


def test_decode_r16_shared_vs_oracle(lch, bt16, orc16):
    import torch
    from paper_1404_3458_b200 import _lib
    from paper_1404_3458_b200.rs import decode_device, encode_device
    n, k = 1 << 16, 1 << 15
    cp = lch.CodeParams(16, k)
    d = G16["decode"]
    mask = O.gen_erasures(d["erasure_seed"], n, d["count"], d["erasure_cw"], 1)[0]
    bits = _lib.to_device_u32(_lib.bitmask_from_positions(n, np.nonzero(mask)[0]))
    B = 1100
    # (a) true codewords: decode must return the message for every row
    msg = gen(bt16, 1404345803, 0, B, k)
    cw = torch.empty((B, n), dtype=torch.int16, device="cuda")
    cw[:, :k].copy_(msg)
    encode_device(cp, bt16, msg, cw[:, k:])
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    decode_device(cp, bt16, cw, bits, out)
    np.testing.assert_array_equal(host(out), host(msg))
    # (b) non-codewords: output is a deterministic function of every stage
    junk = gen(bt16, d["junk_seed"], 0, B, n)
    decode_device(cp, bt16, junk, bits, out)
    got, jh = host(out), host(junk)
    check_digest(got[0], d["junk_out"])
    for r in sample_rows(B)[:6]:
        np.testing.assert_array_equal(got[r], orc16.decode(k, jh[r], mask), err_msg=f"row {r}")


def test_decode_r16_batch_k256_golden(lch, bt16):
    c = G16["batch_k256"]
    codec = lch.BatchCodec(lch.CodeParams(16, 256), bt16)
    msgs = O.gen_symbols(c["msg_seed"], 16, 0, 3, 256)
    enc = codec.encode(msgs)
    check_digest(enc, {"sha256": c["enc_sha256"]})
    mask = O.gen_erasures(c["erasure_seed"], 1 << 16, c["count"], 0, 1)[0]
    junk = O.gen_symbols(c["junk_seed"], 16, 0, 3, 1 << 16)
    out = codec.decode(junk, set(np.nonzero(mask)[0].tolist()))
    check_digest(out, {"sha256": c["junk_dec_sha256"], "sample": c["junk_dec_sample"]})
    rx = enc.copy()
    rx[:, mask == 1] = 0
    np.testing.assert_array_equal(codec.decode(rx, set(np.nonzero(mask)[0].tolist())), msgs)


def test_decode_r8_cfg1_golden(lch, bt8):
    cp = lch.CodeParams(8, 128)
    for row, (m, cw, mask, jd) in enumerate(zip(G8["cfg1_msg"], G8["cfg1_cw"], G8["cfg1_mask"],
                                                G8["cfg1_junk_dec"])):
        pat = lch.ErasurePattern.of(256, np.nonzero(mask)[0].tolist())
        rx = np.where(mask == 1, 0, cw).astype(np.uint16).tolist()
        assert lch.decode(cp, bt8, bt8.ft, rx, pat) == m.tolist()
        junk = O.gen_symbols(1404345801 ^ 0x5A5A, 8, row, 1, 256)[0].tolist()
        assert lch.decode(cp, bt8, bt8.ft, junk, pat) == jd.tolist()


@pytest.mark.parametrize("k", [1, 2, 8, 32, 128])
def test_decode_r8_batch_vs_oracle(lch, bt8, orc8, k):
    codec = lch.BatchCodec(lch.CodeParams(8, k), bt8)
    B = 1300
    junk = O.gen_symbols(5 + k, 8, 0, B, 256)
    for count in sorted({1, (256 - k) // 2 + 1, 256 - k}):
        mask = O.gen_erasures(99 + count, 256, count, 0, 1)[0]
        out = codec.decode(junk, set(np.nonzero(mask)[0].tolist()))
        want = orc8.decode_batch(k, junk, mask, 8)
        np.testing.assert_array_equal(out, want)


def test_locator_vs_golden(lch):
    ft8, ft16 = lch.tables_for(8), lch.tables_for(16)
    for mask, want in zip(G8["loc_mask"], G8["loc_val"]):
        lv = lch.locator_values(ft8, np.nonzero(mask)[0].tolist())
        got = np.zeros(256, np.uint16)
        for j, v in {**lv.pi_bar, **lv.pi_prime}.items():
            got[j] = v
        np.testing.assert_array_equal(got, want)
    c = G16["locator100"]
    lv = lch.locator_values(ft16, c["erased"])
    got = np.zeros(1 << 16, np.uint16)
    for j, v in {**lv.pi_bar, **lv.pi_prime}.items():
        got[j] = v
    check_digest(got, c)


def test_fwht_vs_oracle(lch):
    rng = np.random.default_rng(3)
    for n, mod in ((2, 255), (256, 255), (1 << 12, 65535), (1 << 16, 65535), (64, 1000003)):
        v = rng.integers(0, mod, n).tolist()
        np.testing.assert_array_equal(lch.fwht(list(v), mod), O.fwht(v, mod))
    assert lch.fwht([7, 3], 255) == [10, 4]
    assert lch.fwht([3, 7], 255) == [10, 251]


def test_decode_per_codeword_r8_cfg1_golden(lch, bt8):
    # config 1: 64 codewords, 128 erasures drawn per codeword (rs.decode row by row)
    codec = lch.BatchCodec(lch.CodeParams(8, 128), bt8)
    masks = G8["cfg1_mask"].astype(bool)
    rx = np.where(masks, 0, G8["cfg1_cw"]).astype(np.uint16)
    np.testing.assert_array_equal(codec.decode_patterns(rx, masks), G8["cfg1_msg"])
    junk = np.stack([O.gen_symbols(1404345801 ^ 0x5A5A, 8, row, 1, 256)[0] for row in range(64)])
    np.testing.assert_array_equal(codec.decode_patterns(junk, masks), G8["cfg1_junk_dec"])


@pytest.mark.parametrize("k", [1, 4, 64])
def test_decode_per_codeword_r8_mixed_counts(lch, bt8, orc8, k):
    codec = lch.BatchCodec(lch.CodeParams(8, k), bt8)
    B = 1100
    junk = O.gen_symbols(31 + k, 8, 0, B, 256)
    counts = [(7 * i) % (256 - k + 1) for i in range(B)]  # includes empty patterns
    masks = np.stack([O.gen_erasures(500 + i, 256, counts[i], i, 1)[0] for i in range(B)])
    out = codec.decode_patterns(junk, masks)
    for r in list(range(0, B, 97)) + [B - 1]:
        if counts[r] == 0:
            np.testing.assert_array_equal(out[r], junk[r, :k])
        else:
            np.testing.assert_array_equal(out[r], orc8.decode(k, junk[r], masks[r]), err_msg=f"row {r}")
    with pytest.raises(lch.TooManyErasuresError):
        bad = masks.copy()
        bad[3] = 0
        bad[3, : 256 - k + 1] = 1
        codec.decode_patterns(junk, bad)


def test_decode_per_codeword_r16_vs_oracle(lch, bt16, orc16):
    import torch
    from paper_1404_3458_b200 import gen as G
    from paper_1404_3458_b200.rs import decode_device, encode_device
    n, k, B = 1 << 16, 1 << 15, 1030
    cp = lch.CodeParams(16, k)
    msg = gen(bt16, 1404345803, 0, B, k)
    cw = torch.empty((B, n), dtype=torch.int16, device="cuda")
    cw[:, :k].copy_(msg)
    encode_device(cp, bt16, msg, cw[:, k:])
    emask = G.erasure_masks(bt16.ctx, 1404345804, n, n - k, 0, B)  # per-codeword patterns
    bits = G.mask_to_bits(emask).contiguous()
    rx = cw.masked_fill(emask, 0)
    out = torch.empty((B, k), dtype=torch.int16, device="cuda")
    decode_device(cp, bt16, rx, bits, out, [n - k] * B)
    np.testing.assert_array_equal(host(out), host(msg))
    # pattern generator matches the oracle's (rows 0 and 7)
    for r in (0, 7):
        np.testing.assert_array_equal(emask[r].cpu().numpy().astype(np.uint8),
                                      O.gen_erasures(1404345804, n, n - k, r, 1)[0])
    junk = gen(bt16, 99, 0, 3, n)
    jout = torch.empty((3, k), dtype=torch.int16, device="cuda")
    decode_device(cp, bt16, junk, bits[:3].contiguous(), jout, [n - k] * 3)
    jh, mh = host(junk), emask[:3].cpu().numpy().astype(np.uint8)
    for r in range(3):
        np.testing.assert_array_equal(host(jout)[r], orc16.decode(k, jh[r], mh[r]), err_msg=f"row {r}")


@pytest.mark.parametrize("r,h", [(8, 1), (8, 16), (8, 128), (16, 1024), (16, 1 << 15)])
def test_poly_mul_vs_oracle(lch, bt8, bt16, orc8, orc16, r, h):
    """transform.poly_mul (transform.py:189-206): forward of both zero-extended
    operands, pointwise product, inverse -- all on the GPU."""
    bt, orc = (bt8, orc8) if r == 8 else (bt16, orc16)
    a = O.gen_symbols(31, r, 0, 1, h)[0]
    b = O.gen_symbols(32, r, 0, 1, h)[0]
    got = lch.poly_mul(bt, lch.CoeffVec([int(x) for x in a]), lch.CoeffVec([int(x) for x in b])).data
    ea = orc.forward(np.concatenate([a, np.zeros(h, np.uint16)]), 0)
    eb = orc.forward(np.concatenate([b, np.zeros(h, np.uint16)]), 0)
    prod = np.array([orc.mul(int(x), int(y)) for x, y in zip(ea, eb)], np.uint16)
    np.testing.assert_array_equal(np.asarray(got, np.uint16), orc.inverse(prod, 0))
    if h == 1:
        assert lch.poly_mul(bt, lch.CoeffVec([1]), lch.CoeffVec([1])).data == [1, 0]  # test_transform.py:137-141


@pytest.mark.parametrize("r", [8, 16])
def test_pointwise_mul_vs_tables(lch, bt8, bt16, orc8, orc16, r):
    """lch_pointwise_mul against the log/exp product of the oracle's tables
    (field.py:100-129): r = 16 runs the table-free carry-less multiply
    (gf16_mul, also used by the per-codeword decode), r = 8 the table path.
    Random pairs plus every product of the edge symbols 0, 1, 2, top bit, all ones."""
    import torch

    from paper_1404_3458_b200 import _lib
    bt, orc = (bt8, orc8) if r == 8 else (bt16, orc16)
    t = orc.tables()
    m = (1 << r) - 1
    rng = np.random.default_rng(1404 + r)
    a = rng.integers(0, 1 << r, 1 << 20).astype(np.uint16)
    b = rng.integers(0, 1 << r, 1 << 20).astype(np.uint16)
    edge = np.array([0, 1, 2, 1 << (r - 1), m, m - 1, 0x5A & m], np.uint16)
    a = np.concatenate([a, np.repeat(edge, len(edge))])
    b = np.concatenate([b, np.tile(edge, len(edge))])
    lg, ex = t["log"].astype(np.int64), t["exp"].astype(np.int64)
    want = np.where((a == 0) | (b == 0), 0, ex[(lg[a] + lg[b]) % m]).astype(np.uint16)
    da, db = dev(a), dev(b)
    out = torch.empty_like(da)
    _lib.check(_lib.lib.lch_pointwise_mul(bt.ctx.handle, da.data_ptr(), db.data_ptr(), out.data_ptr(),
                                          len(a), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host(out), want)
