"""Pin the CPU oracle to the reference (golden vectors + known answers).

The golden fixtures were produced by running the reference `binfec` package
(tests/golden/make_golden.py).  The known-answer values below are the ones the
reference's own tests assert (cited per test).
"""

import numpy as np
import pytest

from golden_util import check_digest, load_r8, load_r16, tr_cases
from oracle import oracle as O

G8 = load_r8()
G16 = load_r16()


def test_tables_r8_match_reference(orc8):
    t = orc8.tables()
    for k in ("log", "exp", "w_hat", "w_prime", "b_prod", "b_prod_inv", "fwht_log",
              "w_on_basis", "w_norm"):
        np.testing.assert_array_equal(t[k].ravel(), G8[f"tab_{k}"].ravel(), err_msg=k)


def test_tables_r16_match_reference(orc16):
    t = orc16.tables()
    for k, entry in G16["tables"].items():
        check_digest(t[k].ravel(), entry)


def test_known_answers(orc8):
    # test_field.py:26-29,46-50,76-78; test_basis.py:32-35; test_derivative.py:96-104
    assert orc8.mul(2, 128) == 29
    assert orc8.mul(2, 142) == 1            # inv(2) = 142
    t = orc8.tables()
    assert t["exp"][0] == 1 and t["exp"][1] == 2
    assert t["w_prime"][0] == 1 and t["w_prime"][3] == 41
    # W_2(5) = 117 (unnormalised): W^_2(5) * W_2(v_2)
    assert orc8.mul(orc8.eval_w_hat(2, 5), int(t["w_norm"][2])) == 117
    # test_walsh.py:14-16
    np.testing.assert_array_equal(O.fwht([7, 3], 255), [10, 4])
    np.testing.assert_array_equal(O.fwht([3, 7], 255), [10, 251])


def test_nonprimitive_poly_rejected():
    # test_field.py:81-85: x has order 51 modulo 0x11B
    with pytest.raises(ValueError):
        O.Oracle(8, 0x11B)
    with pytest.raises(ValueError):
        O.Oracle(8, 0x3)


def test_transforms_r8_match_reference(orc8):
    for h, shift, d, fwd, inv, der in tr_cases(G8):
        np.testing.assert_array_equal(orc8.forward(d, shift), fwd)
        np.testing.assert_array_equal(orc8.inverse(d, shift), inv)
        np.testing.assert_array_equal(orc8.derivative(d), der)


def test_op_count_spot_values_via_closed_form():
    # transform.py:16-21; test_transform.py:111-118 -> (24,12) and (17,5) for h=8
    from paper_1404_3458_b200.transform import transform_op_counts
    assert transform_op_counts(8, 8, 256) == (24, 12)
    assert transform_op_counts(8, 0, 256) == (17, 5)
    assert transform_op_counts(1, 3, 256) == (0, 0)


def test_locator_r8_match_reference(orc8):
    exp = orc8.tables()["exp"]
    for mask, want in zip(G8["loc_mask"], G8["loc_val"]):
        logs = orc8.locator_logs(mask)
        np.testing.assert_array_equal(exp[logs], want)


def test_cfg1_codec_r8_match_reference(orc8):
    for m, cw, mask, junk_dec, row in zip(G8["cfg1_msg"], G8["cfg1_cw"], G8["cfg1_mask"],
                                          G8["cfg1_junk_dec"], range(64)):
        np.testing.assert_array_equal(orc8.encode(128, m), cw)
        rx = np.where(mask == 1, 0, cw).astype(np.uint16)
        np.testing.assert_array_equal(orc8.decode(128, rx, mask), m)
        junk = O.gen_symbols(1404345801 ^ 0x5A5A, 8, row, 1, 256)[0]
        np.testing.assert_array_equal(orc8.decode(128, junk, mask), junk_dec)


def test_all_k_r8_match_reference(orc8):
    for k in (1, 2, 4, 16, 64, 256):
        for m, cw in zip(G8[f"k{k}_msg"], G8[f"k{k}_cw"]):
            np.testing.assert_array_equal(orc8.encode(k, m), cw)


def test_generator_matches_python_restatement():
    from golden_util import gen_erasures_py, gen_symbols_py
    np.testing.assert_array_equal(O.gen_symbols(5, 16, 3, 1, 300)[0], gen_symbols_py(5, 16, 3, 300))
    e = O.gen_erasures(9, 256, 77, 4, 1)[0]
    assert sorted(np.nonzero(e)[0].tolist()) == gen_erasures_py(9, 256, 77, 4)


def test_transforms_r16_small_match_reference(orc16):
    for c in G16["transform_small"]:
        d = O.gen_symbols(c["seed"], 16, c["cw"], 1, c["h"])[0]
        np.testing.assert_array_equal(orc16.forward(d, c["shift"]), c["fwd"])
        np.testing.assert_array_equal(orc16.inverse(d, c["shift"]), c["inv"])
        np.testing.assert_array_equal(orc16.derivative(d), c["der"])


def test_transforms_r16_full_match_reference(orc16):
    for c in G16["transform"]:
        d = O.gen_symbols(c["seed"], 16, c["cw"], 1, c["h"])[0]
        check_digest(orc16.forward(d, c["shift"]), c["fwd"])
        check_digest(orc16.inverse(d, c["shift"]), c["inv"])
        check_digest(orc16.derivative(d), c["der"])


def test_encode_r16_match_reference(orc16):
    for c in G16["encode"]:
        m = O.gen_symbols(c["seed"], 16, c["cw"], 1, 1 << 15)[0]
        check_digest(orc16.encode(1 << 15, m)[1 << 15:], c["parity"])


def test_decode_r16_match_reference(orc16):
    d = G16["decode"]
    mask = O.gen_erasures(d["erasure_seed"], 1 << 16, d["count"], d["erasure_cw"], 1)[0]
    check_digest(np.nonzero(mask)[0].astype(np.uint32), {"sha256": d["pattern_sha256"]})
    logs = orc16.locator_logs(mask)
    check_digest(orc16.tables()["exp"][logs], d["locator"])
    m = O.gen_symbols(1404345803, 16, 0, 1, 1 << 15)[0]
    cw = orc16.encode(1 << 15, m)
    rx = np.where(mask == 1, 0, cw).astype(np.uint16)
    np.testing.assert_array_equal(orc16.decode(1 << 15, rx, mask), m)
    junk = O.gen_symbols(d["junk_seed"], 16, 0, 1, 1 << 16)[0]
    check_digest(orc16.decode(1 << 15, junk, mask), d["junk_out"])


def test_locator100_r16(orc16):
    c = G16["locator100"]
    mask = np.zeros(1 << 16, np.uint8)
    mask[c["erased"]] = 1
    check_digest(orc16.tables()["exp"][orc16.locator_logs(mask)], c)


def test_batch_k256_r16(orc16):
    c = G16["batch_k256"]
    msgs = O.gen_symbols(c["msg_seed"], 16, 0, 3, 256)
    par = orc16.encode_batch(256, msgs, nthreads=3)
    check_digest(np.concatenate([msgs, par], axis=1), {"sha256": c["enc_sha256"]})
    mask = O.gen_erasures(c["erasure_seed"], 1 << 16, c["count"], 0, 1)[0]
    junk = O.gen_symbols(c["junk_seed"], 16, 0, 3, 1 << 16)
    out = orc16.decode_batch(256, junk, mask, nthreads=3)
    check_digest(out, {"sha256": c["junk_dec_sha256"], "sample": c["junk_dec_sample"]})
