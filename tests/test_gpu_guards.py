"""Memory-safety and determinism checks of the device path.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing
a reset), so the memcheck / racecheck evidence SURVEY §5 asks for is replaced
by checks of our own:

* guard bands: every output lives inside a larger tensor whose surrounding
  rows, and the columns between the logical width and the row stride, hold a
  sentinel; after encode / decode / transforms / derivative at ragged batch
  sizes (partial 1024-lane groups, single rows) the sentinels must be intact
  and the inputs unmodified (out-of-bounds or stray writes);
* determinism: the same call repeated, interleaved with unrelated work on
  another stream, gives bit-identical results (a shared-memory race between
  the warps of a tile, the TMA / generic proxies, or the named-barrier warp
  pairs would show up as run-to-run differences on these sizes).
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SENT = 0x5AA5
N, K = 1 << 16, 1 << 15


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


def guarded(rows, cols, stride, pad_rows=3):
    """(whole, view): view = rows x cols inside a sentinel-filled buffer."""
    import torch
    whole = torch.full((rows + 2 * pad_rows, stride), SENT, dtype=torch.int16, device="cuda")
    return whole, whole[pad_rows:pad_rows + rows, :cols]


def intact(whole, rows, cols, pad_rows=3):
    import torch
    m = torch.ones_like(whole, dtype=torch.bool)
    m[pad_rows:pad_rows + rows, :cols] = False
    return bool((whole[m] == SENT).all())


@pytest.mark.parametrize("B", [1, 37, 1025, 2047])
def test_codec_writes_stay_in_bounds(lch, bt16, B):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, encode_device
    cp = lch.CodeParams(16, K)
    msg = gen.symbols(bt16.ctx, 11, 0, B, K)
    msg0 = msg.clone()
    odd = B == 37  # odd row strides: the unaligned (non-vector, non-TMA) paths
    pw, par = guarded(B, N - K, N - K + (3 if odd else 24))
    encode_device(cp, bt16, msg, par)
    torch.cuda.synchronize()
    assert intact(pw, B, N - K) and torch.equal(msg, msg0)
    cw = torch.cat([msg, par], dim=1)
    mask = gen.erasure_masks(bt16.ctx, 12, N, N - K, 0, 1)
    bits = gen.mask_to_bits(mask)[0].contiguous()
    rx = torch.where(mask[0][None, :], torch.full_like(cw, 0x1234), cw)
    rx0 = rx.clone()
    ow, out = guarded(B, K, K + (5 if odd else 40))
    decode_device(cp, bt16, rx, bits, out, N - K)
    torch.cuda.synchronize()
    assert intact(ow, B, K) and torch.equal(rx, rx0)
    assert torch.equal(out, msg)
    # per-codeword patterns
    pm = gen.erasure_masks(bt16.ctx, 13, N, N - K, 0, B)
    pbits = gen.mask_to_bits(pm).contiguous()
    rx2 = torch.where(pm, torch.full_like(cw, 0x777), cw)
    ow2, out2 = guarded(B, K, K + 8)
    decode_device(cp, bt16, rx2, pbits, out2, [N - K] * B)
    torch.cuda.synchronize()
    assert intact(ow2, B, K) and torch.equal(out2, msg)


@pytest.mark.parametrize("B,lg", [(3, 16), (1030, 12), (1024, 1)])
def test_transform_and_derivative_in_bounds(lch, bt16, B, lg):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.derivative import run_derivative
    from paper_1404_3458_b200.transform import run_transform
    h = 1 << lg
    stride = h + 16
    dw, d = guarded(B, h, stride)
    d.copy_(gen.symbols(bt16.ctx, 14, 0, B, h))
    a0 = d.clone()
    run_transform(bt16, d, 5, False)
    run_transform(bt16, d, 5, True)
    torch.cuda.synchronize()
    assert intact(dw, B, h) and torch.equal(d, a0)
    ow, o = guarded(B, h, stride)
    run_derivative(bt16, d, o)
    torch.cuda.synchronize()
    assert intact(ow, B, h) and torch.equal(d, a0)
    orc = O.Oracle(16)
    from paper_1404_3458_b200 import _lib
    np.testing.assert_array_equal(_lib.to_host_u16(o[B - 1:B])[0], orc.derivative(_lib.to_host_u16(a0[B - 1:B])[0]))


def test_repeated_calls_bit_identical_under_concurrent_work(lch, bt16):
    import torch
    from paper_1404_3458_b200 import gen
    from paper_1404_3458_b200.rs import decode_device, encode_device
    B = 2048
    cp = lch.CodeParams(16, K)
    msg = gen.symbols(bt16.ctx, 15, 0, B, K)
    junk = gen.symbols(bt16.ctx, 16, 0, B, N)
    mask = gen.erasure_masks(bt16.ctx, 17, N, N - K, 0, 1)
    bits = gen.mask_to_bits(mask)[0].contiguous()
    side = torch.cuda.Stream()
    big = torch.empty(64 << 20, dtype=torch.int16, device="cuda")
    ref_p = ref_o = None
    for it in range(5):
        with torch.cuda.stream(side):  # unrelated traffic competing for the SMs / HBM
            big.add_(1)
        par = torch.empty((B, N - K), dtype=torch.int16, device="cuda")
        out = torch.empty((B, K), dtype=torch.int16, device="cuda")
        encode_device(cp, bt16, msg, par)
        decode_device(cp, bt16, junk, bits, out, N - K)  # non-codewords: every stage matters
        torch.cuda.synchronize()
        if it == 0:
            ref_p, ref_o = par.clone(), out.clone()
        else:
            assert torch.equal(par, ref_p) and torch.equal(out, ref_o), f"run {it} differs"
