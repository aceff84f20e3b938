"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

It imports `binfec` from /root/reference/pkg/src and writes
tests/golden/golden_r8.npz (full arrays, small) and tests/golden/golden_r16.json
(sha256 digests + sampled entries of the large r=16 arrays).  The committed
outputs pin the oracle (tests/test_oracle_golden.py) and, through it, the GPU
path.  Nothing on the GPU box reads /root/reference.

Inputs are drawn from a pure-Python restatement of the counter-based generator
(identical to oracle/lch_oracle.c `orc_key` and csrc/lch_gen.cu),
so tests can regenerate them without storing the r=16 payloads.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from binfec import batch as ref_batch  # noqa: E402
from binfec import rs as ref_rs  # noqa: E402
from binfec import walsh as ref_walsh  # noqa: E402
from binfec.basis import build_basis_tables  # noqa: E402
from binfec.derivative import derivative_fast  # noqa: E402
from binfec.field import tables_for  # noqa: E402
from binfec.transform import CoeffVec, EvalVec, forward, inverse  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key(seed: int, cw: int, pos: int) -> int:
    s = mix64(seed + GAMMA)
    return mix64(s + (((cw << 32) | pos) * GAMMA))


def gen_symbols(seed: int, r: int, cw: int, length: int) -> list[int]:
    mask = (1 << r) - 1
    return [key(seed, cw, j) & mask for j in range(length)]


def gen_erasures(seed: int, n: int, count: int, cw: int) -> list[int]:
    order = sorted(range(n), key=lambda j: (key(seed, cw, j) >> 1, j))
    return sorted(order[:count])


def digest(a) -> str:
    return hashlib.sha256(np.asarray(a, dtype="<u4" if np.asarray(a).dtype == np.uint32 else "<u2").tobytes()).hexdigest()


def sample(a, n=64, seed=7) -> dict:
    a = np.asarray(a)
    rng = random.Random(seed)
    idx = sorted(rng.sample(range(a.size), min(n, a.size)))
    return {"idx": idx, "val": [int(a.flat[i]) for i in idx]}


def tables_of(ft, bt) -> dict:
    return dict(
        log=np.asarray(ft.log, np.uint16), exp=np.asarray(ft.exp, np.uint16),
        w_hat=np.asarray([x for lvl in bt.w_hat for x in lvl], np.uint16),
        w_prime=np.asarray(bt.w_prime, np.uint16),
        b_prod=np.asarray(bt.b_prod, np.uint16),
        b_prod_inv=np.asarray(bt.b_prod_inv, np.uint16),
        fwht_log=np.asarray(ref_walsh._fwht_of_log(ft), np.uint32),
        w_on_basis=np.asarray(bt.w_on_basis, np.uint16),
        w_norm=np.asarray(bt.w_norm, np.uint16))


def make_r8() -> None:
    ft = tables_for(8)
    bt = build_basis_tables(ft, 256)
    out = {f"tab_{k}": v for k, v in tables_of(ft, bt).items()}

    # transforms: every size, shifts {0, h, random}, forward + inverse + derivative
    rng = random.Random(1404)
    cases = []
    for lg in range(0, 9):
        h = 1 << lg
        for shift in sorted({0, h % 256, rng.randrange(256), 255}):
            d = [rng.randrange(256) for _ in range(h)]
            cases.append((h, shift, d))
    fw, inv, der, meta = [], [], [], []
    for h, shift, d in cases:
        fw.append(forward(bt, CoeffVec(d), shift).data)
        inv.append(inverse(bt, EvalVec(d, shift)).data)
        der.append(derivative_fast(bt, CoeffVec(d)).data)
        meta.append((h, shift))
    flat = lambda xs: np.asarray([x for v in xs for x in v], np.uint16)  # noqa: E731
    out["tr_meta"] = np.asarray(meta, np.int64)
    out["tr_in"] = flat([d for _, _, d in cases])
    out["tr_fwd"] = flat(fw)
    out["tr_inv"] = flat(inv)
    out["tr_der"] = flat(der)

    # fwht + locator logs for several patterns (walsh.py)
    pats = []
    for size in (1, 2, 40, 128, 200, 255):
        pats.append(sorted(random.Random(size).sample(range(256), size)))
    out["loc_mask"] = np.zeros((len(pats), 256), np.uint8)
    out["loc_val"] = np.zeros((len(pats), 256), np.uint16)
    for t, p in enumerate(pats):
        out["loc_mask"][t, p] = 1
        lv = ref_walsh.locator_values(ft, p)
        for j, v in lv.pi_bar.items():
            out["loc_val"][t, j] = v
        for j, v in lv.pi_prime.items():
            out["loc_val"][t, j] = v

    # config 1: (256, 128), 64 codewords, 128 per-codeword erasures (seed ...801)
    seed_m, seed_e = 1404345801, 1404345801 ^ 0xE
    cp = ref_rs.CodeParams(8, 128)
    msgs, cws, masks, decs, junk_out = [], [], [], [], []
    for cw in range(64):
        m = gen_symbols(seed_m, 8, cw, 128)
        c = ref_rs.encode(cp, bt, m).symbols
        e = gen_erasures(seed_e, 256, 128, cw)
        rx = [0 if j in set(e) else s for j, s in enumerate(c)]
        dec = ref_rs.decode(cp, bt, ft, rx, ref_rs.ErasurePattern.of(256, e))
        assert dec == m
        # non-codeword input: the decoder's output is then a deterministic
        # function of every intermediate step (locator, phi, transforms, derivative)
        junk = gen_symbols(seed_m ^ 0x5A5A, 8, cw, 256)
        jd = ref_rs.decode(cp, bt, ft, junk, ref_rs.ErasurePattern.of(256, e))
        msgs.append(m); cws.append(c); decs.append(dec); junk_out.append(jd)
        mk = np.zeros(256, np.uint8); mk[e] = 1; masks.append(mk)
    out["cfg1_msg"] = np.asarray(msgs, np.uint16)
    out["cfg1_cw"] = np.asarray(cws, np.uint16)
    out["cfg1_mask"] = np.asarray(masks, np.uint8)
    out["cfg1_junk_dec"] = np.asarray(junk_out, np.uint16)

    # every power-of-two k (rs.py), one codeword each, through BatchCodec too
    for k in (1, 2, 4, 16, 64, 256):
        cpk = ref_rs.CodeParams(8, k)
        m = np.asarray([gen_symbols(77, 8, cw, k) for cw in range(5)], np.uint16)
        enc = ref_batch.BatchCodec(cpk, bt).encode(m)
        for row in range(5):
            assert list(enc[row]) == ref_rs.encode(cpk, bt, [int(x) for x in m[row]]).symbols
        out[f"k{k}_msg"] = m
        out[f"k{k}_cw"] = enc
    # general k (no reference codec): codewords and decodes
    # composed from the reference's own primitives (locator_values, inverse,
    # derivative_fast, forward), i.e. rs.decode's algorithm evaluated at every
    # erased position, with encode = erasure-decode of E = [k, n)
    for k in (3, 100, 192, 240, 255):
        msgs, cws, masks, decs = [], [], [], []
        for cw in range(3):
            m = gen_symbols(1404345805, 8, cw, k)
            c = recover_all_ref(ft, bt, 256, m + [0] * (256 - k), list(range(k, 256)))
            assert c[:k] == m
            e = gen_erasures(1404345805 ^ 0xE, 256, 256 - k, cw)
            junk = gen_symbols(1404345805 ^ 0x5A5A, 8, cw, 256)
            rx = [junk[j] if j in set(e) else c[j] for j in range(256)]
            dec = recover_all_ref(ft, bt, 256, rx, e)
            assert dec == c
            mk = np.zeros(256, np.uint8); mk[e] = 1
            msgs.append(m); cws.append(c); masks.append(mk); decs.append(rx)
        out[f"anyk{k}_msg"] = np.asarray(msgs, np.uint16)
        out[f"anyk{k}_cw"] = np.asarray(cws, np.uint16)
        out[f"anyk{k}_mask"] = np.asarray(masks, np.uint8)
        out[f"anyk{k}_rx"] = np.asarray(decs, np.uint16)
    # power-of-two k: the composition equals rs.encode (fact iii)
    for k in (2, 32, 128):
        m = gen_symbols(1404345805, 8, 9, k)
        assert recover_all_ref(ft, bt, 256, m + [0] * (256 - k), list(range(k, 256))) == \
            ref_rs.encode(ref_rs.CodeParams(8, k), bt, m).symbols
    np.savez_compressed(os.path.join(HERE, "golden_r8.npz"), **out)


def recover_all_ref(ft, bt, n, received, erased):
    """rs.py:125-148 (locator, phi, n-point inverse, derivative, forward,
    division by Pi') with the recovered value written at EVERY erased position."""
    es = set(erased)
    lv = ref_walsh.locator_values(ft, erased)
    phi = [0 if j in es else ft.mul(received[j], lv.pi_bar[j]) for j in range(n)]
    coef = inverse(bt, EvalVec(phi, 0)).data
    d = derivative_fast(bt, CoeffVec(coef)).data
    ev = forward(bt, CoeffVec(d), 0).data
    full = list(received)
    for j in es:
        full[j] = ft.div(ev[j], lv.pi_prime[j])
    return full


def make_r16() -> None:
    ft = tables_for(16)
    bt = build_basis_tables(ft, 1 << 16)
    res: dict = {"tables": {}}
    for k, v in tables_of(ft, bt).items():
        res["tables"][k] = {"sha256": digest(v), "sample": sample(v), "size": int(v.size)}

    # config 2: transforms at h = 2^16, two seeded polynomials, shift 0 and 12345
    res["transform"] = []
    for t, shift in enumerate((0, 12345)):
        d = gen_symbols(1404345802, 16, t, 1 << 16)
        fwd = forward(bt, CoeffVec(d), shift).data
        inv = inverse(bt, EvalVec(d, shift)).data
        der = derivative_fast(bt, CoeffVec(d)).data
        res["transform"].append({
            "seed": 1404345802, "cw": t, "h": 1 << 16, "shift": shift,
            "fwd": {"sha256": digest(fwd), "sample": sample(fwd)},
            "inv": {"sha256": digest(inv), "sample": sample(inv)},
            "der": {"sha256": digest(der), "sample": sample(der)}})
    # smaller sizes, full arrays (cheap): h = 2^10 at several shifts
    res["transform_small"] = []
    for shift in (0, 1024, 4096 * 3, 65535):
        d = gen_symbols(99, 16, shift, 1024)
        res["transform_small"].append({
            "seed": 99, "cw": shift, "h": 1024, "shift": shift,
            "fwd": forward(bt, CoeffVec(d), shift).data,
            "inv": inverse(bt, EvalVec(d, shift)).data,
            "der": derivative_fast(bt, CoeffVec(d)).data})

    # config 3: encode, two codewords of RS(2^16, 2^15)
    cp = ref_rs.CodeParams(16, 1 << 15)
    res["encode"] = []
    for cw in range(2):
        m = gen_symbols(1404345803, 16, cw, 1 << 15)
        c = ref_rs.encode(cp, bt, m).symbols
        res["encode"].append({"seed": 1404345803, "cw": cw,
                              "parity": {"sha256": digest(c[1 << 15:]), "sample": sample(c[1 << 15:])}})
    # config 4: decode with 2^15 erasures; a true codeword and a non-codeword
    seed_e = 1404345804
    e = gen_erasures(seed_e, 1 << 16, 1 << 15, 0)
    pat = ref_rs.ErasurePattern.of(1 << 16, e)
    m = gen_symbols(1404345803, 16, 0, 1 << 15)
    c = ref_rs.encode(cp, bt, m).symbols
    es = set(e)
    rx = [0 if j in es else s for j, s in enumerate(c)]
    assert ref_rs.decode(cp, bt, ft, rx, pat) == m
    junk = gen_symbols(1404345804 ^ 0x5A5A, 16, 0, 1 << 16)
    jd = ref_rs.decode(cp, bt, ft, junk, pat)
    lv = ref_walsh.locator_values(ft, e)
    loc = np.zeros(1 << 16, np.uint16)
    for j, v in lv.pi_bar.items():
        loc[j] = v
    for j, v in lv.pi_prime.items():
        loc[j] = v
    res["decode"] = {"erasure_seed": seed_e, "erasure_cw": 0, "count": 1 << 15,
                     "pattern_sha256": digest(np.asarray(e, np.uint32)),
                     "locator": {"sha256": digest(loc), "sample": sample(loc)},
                     "junk_seed": 1404345804 ^ 0x5A5A,
                     "junk_out": {"sha256": digest(jd), "sample": sample(jd)}}
    # small locator pattern (walsh test_r16 style)
    e100 = sorted(random.Random(54).sample(range(1 << 16), 100))
    lv = ref_walsh.locator_values(ft, e100)
    loc = np.zeros(1 << 16, np.uint16)
    for j, v in lv.pi_bar.items():
        loc[j] = v
    for j, v in lv.pi_prime.items():
        loc[j] = v
    res["locator100"] = {"erased": e100, "sha256": digest(loc), "sample": sample(loc)}

    # test_batch.py:57-67 analogue: (2^16, 256), 60,000 shared erasures, BatchCodec
    cpb = ref_rs.CodeParams(16, 256)
    codec = ref_batch.BatchCodec(cpb, bt)
    msgs = np.asarray([gen_symbols(84, 16, cw, 256) for cw in range(3)], np.uint16)
    enc = codec.encode(msgs)
    e6 = gen_erasures(85, 1 << 16, 60000, 0)
    junk = np.asarray([gen_symbols(86, 16, cw, 1 << 16) for cw in range(3)], np.uint16)
    jd = codec.decode(junk, set(e6))
    res["batch_k256"] = {"msg_seed": 84, "erasure_seed": 85, "count": 60000, "junk_seed": 86,
                         "enc_sha256": digest(enc), "junk_dec_sha256": digest(jd),
                         "junk_dec_sample": sample(jd)}
    with open(os.path.join(HERE, "golden_r16.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def make_r16_anyk() -> None:
    """Storage-stripe rates k/n = 3/4, 15/16 (config 5) at r=16, composed from
    the reference primitives like make_r8's anyk vectors."""
    ft = tables_for(16)
    bt = build_basis_tables(ft, 1 << 16)
    n = 1 << 16
    res = []
    for k in (49152, 61440):
        m = gen_symbols(1404345805, 16, 0, k)
        c = recover_all_ref(ft, bt, n, m + [0] * (n - k), list(range(k, n)))
        assert c[:k] == m
        e = gen_erasures(1404345805 ^ 0xE, n, n - k, 0)
        junk = gen_symbols(1404345805 ^ 0x5A5A, 16, 0, n)
        es = set(e)
        rx = [junk[j] if j in es else c[j] for j in range(n)]
        assert recover_all_ref(ft, bt, n, rx, e)[:k] == m
        jd = recover_all_ref(ft, bt, n, junk, e)[:k]
        res.append(dict(k=k, seed=1404345805, cw=0, parity=dict(sha256=digest(c[k:]), sample=sample(c[k:])),
                        erasure_seed=1404345805 ^ 0xE, junk_seed=1404345805 ^ 0x5A5A,
                        pattern_sha256=digest(np.asarray(e, np.uint32)),
                        junk_out=dict(sha256=digest(jd), sample=sample(jd))))
    with open(os.path.join(HERE, "golden_r16_anyk.json"), "w") as f:
        json.dump(res, f, indent=1)


def file_bytes(seed: int, size: int) -> bytes:
    """Seeded file contents (the counter-based generator, one byte per key)."""
    return bytes(key(seed, 0, j) & 0xFF for j in range(size))


def make_shards() -> None:
    """Shard files written by the reference CLI (cli.py:40-60, shardfile.py),
    as sha256 per shard file, for r = 8; r = 16 through the same API without
    files (2^16 shard files per case): stripe packing + BatchCodec.encode +
    one concatenated digest of all shard payloads in index order."""
    import tempfile
    from binfec import cli as ref_cli
    from binfec import shardfile as ref_sf
    res = {"r8": [], "r16": []}
    for size, k in ((0, 128), (1, 128), (1000, 128), (100000, 128), (5000, 16), (3000, 1)):
        seed = 1404345800 + size + k
        with tempfile.TemporaryDirectory() as td:
            src = os.path.join(td, "in.bin")
            with open(src, "wb") as fh:
                fh.write(file_bytes(seed, size))
            outd = os.path.join(td, "shards")
            assert ref_cli.main(["encode", "--in", src, "--out", outd, "--r", "8", "--k", str(k)]) == 0
            shards = []
            for j in range(256):
                with open(os.path.join(outd, ref_sf.shard_filename(j)), "rb") as fh:
                    shards.append(hashlib.sha256(fh.read()).hexdigest()[:32])
        res["r8"].append({"seed": seed, "size": size, "k": k, "shard_sha256_32": shards})
    ft = tables_for(16)
    bt = build_basis_tables(ft, 1 << 16)
    for size, k in ((100000, 1024), (70000, 32768)):
        seed = 1404345800 + size + k
        data = file_bytes(seed, size)
        stripes = ref_sf.bytes_to_stripes(data, k, 16)
        cw = ref_batch.BatchCodec(ref_rs.CodeParams(16, k), bt).encode(stripes)
        h = hashlib.sha256()
        for j in range(1 << 16):
            h.update(cw[:, j].astype("<u2").tobytes())
        hdr = ref_sf.ShardHeader(16, k.bit_length() - 1, 7, size, 0x1100B).pack()
        res["r16"].append({"seed": seed, "size": size, "k": k, "stripes": int(stripes.shape[0]),
                           "payloads_sha256": h.hexdigest(), "header7_hex": hdr.hex()})
    with open(os.path.join(HERE, "golden_shards.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def make_fields() -> None:
    """Non-default fields (SURVEY §8a field row; field.py:28-53): other
    primitive reduction polynomials and other generators alpha.  Writes
    golden_fields.json: table digests, transforms, encode / decode outputs."""
    from binfec.field import FieldParams, build_tables
    from binfec.rs import CodeParams, ErasurePattern
    cases = []
    for r, poly, alpha, k in ((8, 0x12B, 2, 128), (8, 0x11D, 19, 128), (8, 0x163, 2, 32),
                              (16, 0x1002D, 2, 1 << 15), (16, 0x1100B, 3, 1 << 15)):
        ft = build_tables(FieldParams(r, poly, alpha))
        n = 1 << r
        bt = build_basis_tables(ft, n)
        seed = 1404345900 + r + alpha
        c = {"r": r, "poly": poly, "alpha": alpha, "k": k, "seed": seed,
             "log": digest(np.asarray(ft.log, np.uint16)), "exp": digest(np.asarray(ft.exp, np.uint16)),
             "w_hat": digest(np.asarray([x for lvl in bt.w_hat for x in lvl], np.uint16)),
             "b_prod": digest(np.asarray(bt.b_prod, np.uint16))}
        a = gen_symbols(seed, r, 0, n)
        c["forward_shift0"] = {"sha256": digest(forward(bt, CoeffVec(a), 0).data)}
        c["inverse_shift0"] = {"sha256": digest(inverse(bt, EvalVec(a, 0)).data)}
        h = n // 4
        c["forward_h4_shift"] = {"h": h, "shift": 3 * h,
                                 "sha256": digest(forward(bt, CoeffVec(a[:h]), 3 * h).data)}
        cp = CodeParams(r, k)
        ncw = 4 if r == 8 else 1
        enc, dec, junk_dec = [], [], []
        for cw in range(ncw):
            m = gen_symbols(seed + 1, r, cw, k)
            sym = ref_rs.encode(cp, bt, m).symbols
            enc.append(digest(sym[k:]))
            er = gen_erasures(seed + 2, n, n - k, cw)
            pat = ErasurePattern.of(n, er)
            junk = gen_symbols(seed + 3, r, cw, n)
            rx = [junk[j] if j in set(er) else sym[j] for j in range(n)]
            out = ref_rs.decode(cp, bt, ft, rx, pat)
            assert out == m
            dec.append(digest(out))
            junk_dec.append(digest(ref_rs.decode(cp, bt, ft, junk, pat)))
        c["encode_parity"] = enc
        c["decode_junk"] = junk_dec
        cases.append(c)
        print("fields", r, hex(poly), alpha, flush=True)
    with open(os.path.join(HERE, "golden_fields.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["r8", "r16"]
    if "r8" in which:
        make_r8()
        print("r8 done", flush=True)
    if "r16" in which:
        make_r16()
        print("r16 done", flush=True)
    if "r16" in which or "r16_anyk" in which:
        make_r16_anyk()
        print("r16_anyk done", flush=True)
    if "fields" in which:
        make_fields()
        print("fields done", flush=True)
    if "shards" in which or which == ["r8", "r16"]:
        make_shards()
        print("shards done", flush=True)
