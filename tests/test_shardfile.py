"""Shard files: format and consensus reader on the CPU;
GPU encode/decode of whole files byte-identical to the reference CLI
(golden digests from tests/golden/make_golden.py `make_shards`)."""

import hashlib
import json
import os

import numpy as np
import pytest

from golden_util import key

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden_shards.json")))


def file_bytes(seed, size):
    return bytes(key(seed, 0, j) & 0xFF for j in range(size))


def test_header_roundtrip_matches_reference_bytes():
    from paper_1404_3458_b200.shardfile import ShardHeader
    for c in GOLD["r16"]:
        h = ShardHeader(16, c["k"].bit_length() - 1, 7, c["size"], 0x1100B)
        assert h.pack().hex() == c["header7_hex"]
        assert ShardHeader.unpack(h.pack()) == h
        assert h.stripe_count == c["stripes"]


def test_read_shards_consensus(tmp_path):
    from paper_1404_3458_b200.shardfile import (ShardHeader, read_shards, shard_filename,
                                               write_shards, ShardFormatError)
    hdr = ShardHeader(8, 7, 0, 300, 0x11D)
    cw = np.arange(3 * 256, dtype=np.uint16).reshape(3, 256) & 0xFF
    paths = write_shards(str(tmp_path), hdr, cw)
    assert len(paths) == 256
    # corrupt magic, truncate, foreign header, duplicate index
    with open(paths[3], "r+b") as fh:
        fh.write(b"XXXX")
    with open(paths[4], "r+b") as fh:
        fh.truncate(25)
    with open(paths[5], "wb") as fh:
        fh.write(ShardHeader(8, 6, 5, 300, 0x11D).pack() + bytes(3))
    dup = os.path.join(str(tmp_path), "zz-dup.lchs")
    with open(paths[6], "rb") as src, open(dup, "wb") as dst:
        dst.write(src.read())
    header, cols, skipped = read_shards(paths + [dup])
    assert header == hdr
    assert set(cols) == set(range(256)) - {3, 4, 5}
    assert len(skipped) == 4
    np.testing.assert_array_equal(cols[7], cw[:, 7])
    with pytest.raises(ShardFormatError):
        ShardHeader.unpack(b"LCHS")
    assert shard_filename(12) == "shard-00012.lchs"


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(6))
def test_encode_file_matches_reference_cli(tmp_path, case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1404_3458_b200 import cli
    from paper_1404_3458_b200.shardfile import shard_filename
    c = GOLD["r8"][case]
    src = tmp_path / "in.bin"
    data = file_bytes(c["seed"], c["size"])
    src.write_bytes(data)
    out = tmp_path / "shards"
    assert cli.main(["encode", "--in", str(src), "--out", str(out), "--r", "8", "--k", str(c["k"])]) == 0
    got = [hashlib.sha256((out / shard_filename(j)).read_bytes()).hexdigest()[:32] for j in range(256)]
    assert got == c["shard_sha256_32"]
    # rebuild from exactly k shards chosen at random, plus a corrupt one
    rng = np.random.default_rng(case)
    keep = set(rng.choice(256, size=c["k"], replace=False).tolist())
    for j in range(256):
        if j not in keep:
            (out / shard_filename(j)).unlink()
    victim = sorted(keep)[0]
    (out / "extra-corrupt.lchs").write_bytes(b"LCHX" + bytes(30))
    dst = tmp_path / "out.bin"
    assert cli.main(["decode", "--shards", str(out), "--out", str(dst)]) == 0
    assert dst.read_bytes() == data
    assert victim in keep


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(2))
def test_r16_shard_payloads_match_reference(case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1404_3458_b200.shardfile import decode_columns, encode_bytes
    c = GOLD["r16"][case]
    data = file_bytes(c["seed"], c["size"])
    header, pay = encode_bytes(data, 16, c["k"])
    assert header.stripe_count == c["stripes"]
    assert hashlib.sha256(pay.tobytes()).hexdigest() == c["payloads_sha256"]
    # decode from the parity shards plus a few data shards
    n, k = 1 << 16, c["k"]
    rng = np.random.default_rng(case)
    keep = rng.choice(n, size=k, replace=False)
    cols = {int(j): pay[j].view("<u2").astype(np.uint16) for j in keep}
    assert decode_columns(header, cols) == data
