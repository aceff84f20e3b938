"""GPU parity at the exact BASELINE.json shapes (SURVEY §8c sample counts).

* config 5: 4 KiB packets (P = 2048: two bit-sliced groups per stripe group),
  two stripe groups with different erasure patterns, all three rates; >= 64
  sampled lanes per check against the oracle, plus lane 0 against the
  reference-generated digests of tests/golden/golden_r16_anyk.json (lane 0 is
  codeword 0 of seed 1404345805, its group's pattern is pattern 0 of the
  golden erasure seed), and a full-batch round trip;
* configs 3 / 4a / 4b: B = 4096 codewords, >= 64 / >= 64 / >= 8 sampled rows
  against the oracle, and full-batch round trips.
"""

import json
import os

import numpy as np
import pytest

from golden_util import check_digest, load_r16
from oracle import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
N = 1 << 16
P = 2048
SEED5, ERA5, JUNK5 = 1404345805, 1404345795, 1404356503
NTH = min(32, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def lch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_3458_b200 as m
    return m


@pytest.fixture(scope="module")
def bt16(lch):
    return lch.build_basis_tables(lch.tables_for(16), N)


@pytest.fixture(scope="module")
def orc():
    return O.Oracle(16)


def host(t):
    from paper_1404_3458_b200 import _lib
    return _lib.to_host_u16(t)


def lane_rows(p, idx):
    """rows idx (lane b = g * P + s) of a packet tensor [G, npos, P] (host)."""
    return np.stack([p[b // P, :, b % P] for b in idx])


def sample_lanes(G, count, seed):
    """Lanes at the edges of both bit-sliced groups of every stripe group, plus random ones."""
    fixed = []
    for g in range(G):
        fixed += [g * P + s for s in (0, 1, 31, 32, 1023, 1024, 1025, 2046, 2047)]
    rng = np.random.default_rng(seed)
    rest = rng.choice(np.setdiff1d(np.arange(G * P), fixed), count - len(fixed), replace=False)
    return sorted(set(fixed) | set(int(x) for x in rest))


@pytest.mark.parametrize("k", [1 << 15, 49152, 61440])
def test_cfg5_packets_4k(lch, bt16, orc, k):
    import torch
    from paper_1404_3458_b200 import gen
    G = 2
    gold = {int(c["k"]): c for c in json.load(open(os.path.join(HERE, "golden", "golden_r16_anyk.json")))}
    sc = lch.StripeCodec(bt16, k, P)
    msg = gen.packets(bt16.ctx, SEED5, 0, G, k, P)
    par = sc.encode(msg)
    mh, ph = host(msg), host(par)
    idx = sample_lanes(G, 64, k)
    ml = lane_rows(mh, idx)
    want = orc.encode_any_batch(k, ml, nthreads=NTH)
    np.testing.assert_array_equal(lane_rows(ph, idx), want)
    if k in gold:  # lane 0 against the reference's own composition (digest)
        check_digest(ph[0, :, 0], gold[k]["parity"])
    # per-group patterns (pattern g of the golden erasure seed for group g)
    masks = O.gen_erasures(ERA5, N, N - k, 0, G).astype(bool)
    if k in gold:
        check_digest(np.nonzero(masks[0])[0].astype(np.uint32), {"sha256": gold[k]["pattern_sha256"]})
    from paper_1404_3458_b200.gen import mask_to_bits
    bits = mask_to_bits(torch.from_numpy(masks).cuda()).contiguous()
    cw = torch.cat([msg, par], dim=1)
    junk = gen.packets(bt16.ctx, JUNK5, 0, G, N, P)
    me = torch.from_numpy(masks).cuda()[:, :, None]
    rx = torch.where(me, junk, cw)  # erased packets hold junk
    out = sc.decode(rx, bits)
    torch.testing.assert_close(out, msg, rtol=0, atol=0)  # whole batch: decode(encode(m)) == m
    # a non-codeword: decode of junk, sampled lanes against the oracle
    jout = host(sc.decode(junk, bits))
    jh = host(junk)
    jl = lane_rows(jh, idx)
    em = np.stack([masks[b // P] for b in idx]).astype(np.uint8)
    np.testing.assert_array_equal(lane_rows(jout, idx), orc.decode_any_batch(k, jl, em, nthreads=NTH))
    if k in gold:
        check_digest(jout[0, :, 0], gold[k]["junk_out"])


@pytest.fixture(scope="module")
def cfg34(lch, bt16):
    """4096 codewords of config 3 (seed 1404345803) encoded on the GPU."""
    import torch
    from paper_1404_3458_b200.rs import encode_device
    from paper_1404_3458_b200 import gen
    K, B = 1 << 15, 4096
    cp = lch.CodeParams(16, K)
    msg = gen.symbols(bt16.ctx, 1404345803, 0, B, K)
    cw = torch.empty((B, N), dtype=torch.int16, device="cuda")
    cw[:, :K].copy_(msg)
    encode_device(cp, bt16, msg, cw[:, K:])
    torch.cuda.synchronize()
    return cp, msg, cw


def test_cfg3_encode_4096(lch, bt16, orc, cfg34):
    cp, msg, cw = cfg34
    K = cp.k
    rows = sample_rows(4096, 64, 3)
    mh = host(msg[rows])
    np.testing.assert_array_equal(host(cw[rows, K:]), orc.encode_batch(K, mh, nthreads=NTH))
    hits = 0
    for e in load_r16()["encode"]:  # codewords against the reference's own digests
        if int(e["seed"]) == 1404345803 and int(e["cw"]) < 4096:
            check_digest(host(cw[int(e["cw"]):int(e["cw"]) + 1, K:])[0], e["parity"])
            hits += 1
    assert hits


def sample_rows(B, count, seed):
    rng = np.random.default_rng(seed)
    fixed = [r for r in (0, 1, 31, 32, 1023, 1024, 2047, 2048, 4094, 4095) if r < B]
    rest = rng.choice(np.setdiff1d(np.arange(B), fixed), count - len(fixed), replace=False)
    return sorted(set(fixed) | set(int(x) for x in rest))


def test_cfg4a_shared_decode_4096(lch, bt16, orc, cfg34):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device
    cp, msg, cw = cfg34
    K = cp.k
    emask = gen.erasure_masks(bt16.ctx, 1404345804, N, N - K, 0, 1)
    bits = gen.mask_to_bits(emask)[0].contiguous()
    junk = gen.symbols(bt16.ctx, 1404345806, 0, 4096, N)
    rx = torch.where(emask[0][None, :], junk, cw)
    out = torch.empty((4096, K), dtype=torch.int16, device="cuda")
    decode_device(cp, bt16, rx, bits, out, N - K)
    torch.testing.assert_close(out, msg, rtol=0, atol=0)
    decode_device(cp, bt16, junk, bits, out, N - K)  # non-codewords
    rows = sample_rows(4096, 64, 4)
    m = emask[0].cpu().numpy().astype(np.uint8)
    np.testing.assert_array_equal(host(out[rows]),
                                  orc.decode_batch(K, host(junk[rows]), m, nthreads=NTH))


def test_cfg4b_per_codeword_decode_4096(lch, bt16, orc, cfg34):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device
    cp, msg, cw = cfg34
    K = cp.k
    masks = gen.erasure_masks(bt16.ctx, 1404345804, N, N - K, 0, 4096)
    bits = gen.mask_to_bits(masks).contiguous()
    junk = gen.symbols(bt16.ctx, 1404345807, 0, 4096, N)
    rx = torch.where(masks, junk, cw)
    out = torch.empty((4096, K), dtype=torch.int16, device="cuda")
    decode_device(cp, bt16, rx, bits, out, [N - K] * 4096)
    torch.testing.assert_close(out, msg, rtol=0, atol=0)
    decode_device(cp, bt16, junk, bits, out, [N - K] * 4096)
    rows = sample_rows(4096, 12, 5)
    mh = masks[rows].cpu().numpy().astype(np.uint8)
    np.testing.assert_array_equal(host(out[rows]), orc.decode_batch(K, host(junk[rows]), mh, nthreads=NTH))


def test_cfg2_transforms_1024_x_2_16(lch, bt16, orc):
    """Config 2 exactly: 1024 polynomials, h = 2^16 (seed 1404345802):
    forward (shift 0 and a nonzero shift), inverse, derivative; 16 sampled
    polynomials against the oracle, full-batch round trips."""
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.derivative import run_derivative
    from paper_1404_3458_b200.transform import run_transform
    B = 1024
    x = gen.symbols(bt16.ctx, 1404345802, 0, B, N)
    xin = host(x)
    rows = sample_rows(B, 16, 6)
    for shift in (0, 40503):
        y = x.clone()
        run_transform(bt16, y, shift, False)
        got = host(y[rows])
        for i, r in enumerate(rows):
            np.testing.assert_array_equal(got[i], orc.forward(xin[r], shift), err_msg=f"row {r}")
        run_transform(bt16, y, shift, True)
        torch.testing.assert_close(y, x, rtol=0, atol=0)
    z = x.clone()
    run_transform(bt16, z, 0, True)
    got = host(z[rows])
    for i, r in enumerate(rows):
        np.testing.assert_array_equal(got[i], orc.inverse(xin[r], 0))
    d = torch.empty_like(x)
    run_derivative(bt16, x, d)
    got = host(d[rows[:8]])
    for i, r in enumerate(rows[:8]):
        np.testing.assert_array_equal(got[i], orc.derivative(xin[r]))
