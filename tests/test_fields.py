"""Non-default fields (field.py:28-53): any primitive reduction polynomial and
any generator alpha.  Golden vectors from the reference itself
(tests/golden/make_golden.py `make_fields`): r = 8 with 0x12B, 0x163 and
alpha = 19 under 0x11D; r = 16 with 0x1002D and alpha = 3 under 0x1100B.

CPU: the oracle (pinned restatement) and the product's native table builder
against the reference's tables.  GPU: transforms, encode and decode through
the shim (runtime-taps kernel instances for the non-default polynomials)
against the reference's outputs.
"""

import json
import os

import numpy as np
import pytest

from golden_util import digest, gen_erasures_py, gen_symbols_py
from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "golden_fields.json")))
IDS = [f"r{c['r']}-{c['poly']:#x}-a{c['alpha']}" for c in CASES]


def _inputs(c):
    r, n, k = c["r"], 1 << c["r"], c["k"]
    return r, n, k, gen_symbols_py(c["seed"], r, 0, n)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_oracle_matches_reference_fields(c):
    r, n, k, a = _inputs(c)
    if r == 16 and c["alpha"] != 2:
        pytest.skip("outputs do not depend on alpha (checked at r = 8); tables below")
    orc = O.Oracle(r, c["poly"])
    t = orc.tables()
    assert digest(t["w_hat"]) == c["w_hat"] and digest(t["b_prod"]) == c["b_prod"]
    if c["alpha"] == 2:
        assert digest(t["log"]) == c["log"] and digest(t["exp"]) == c["exp"]
    assert digest(orc.forward(a, 0)) == c["forward_shift0"]["sha256"]
    assert digest(orc.inverse(a, 0)) == c["inverse_shift0"]["sha256"]
    fh = c["forward_h4_shift"]
    assert digest(orc.forward(a[:fh["h"]], fh["shift"])) == fh["sha256"]
    if r == 8:  # the codec too (r = 16 codecs are checked on the GPU)
        for cw, want in enumerate(c["encode_parity"]):
            m = gen_symbols_py(c["seed"] + 1, r, cw, k)
            assert digest(orc.encode(k, m)[k:]) == want


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_product_tables_match_reference(c):
    """The native builder (lch_init_alpha + lch_get_tables), no device needed."""
    from paper_1404_3458_b200 import _lib
    ctx = _lib.Context(c["r"], c["poly"], c["r"], c["alpha"])
    t = ctx.tables()
    for name in ("log", "exp", "w_hat", "b_prod"):
        assert digest(t[name]) == c[name], name


def test_non_generator_alpha_rejected():
    import paper_1404_3458_b200 as lch
    with pytest.raises(ValueError):
        lch.build_tables(lch.FieldParams(8, 0x11D, 3))  # x + 1 does not generate GF(256)*


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_gpu_fields_match_reference(c):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_3458_b200 as lch
    r, n, k, a = _inputs(c)
    ft = lch.build_tables(lch.FieldParams(r, c["poly"], c["alpha"]))
    bt = lch.build_basis_tables(ft, n)
    assert digest(lch.forward(bt, lch.CoeffVec(a), 0).data) == c["forward_shift0"]["sha256"]
    assert digest(lch.inverse(bt, lch.EvalVec(a, 0)).data) == c["inverse_shift0"]["sha256"]
    fh = c["forward_h4_shift"]
    assert digest(lch.forward(bt, lch.CoeffVec(a[:fh["h"]]), fh["shift"]).data) == fh["sha256"]
    cp = lch.CodeParams(r, k)
    for cw, (want_p, want_j) in enumerate(zip(c["encode_parity"], c["decode_junk"])):
        m = gen_symbols_py(c["seed"] + 1, r, cw, k)
        sym = lch.encode(cp, bt, m).symbols
        assert digest(sym[k:]) == want_p
        er = gen_erasures_py(c["seed"] + 2, n, n - k, cw)
        junk = gen_symbols_py(c["seed"] + 3, r, cw, n)
        ers = set(er)
        rx = [junk[j] if j in ers else sym[j] for j in range(n)]
        pat = lch.ErasurePattern.of(n, er)
        assert lch.decode(cp, bt, ft, rx, pat) == m
        assert digest(lch.decode(cp, bt, ft, junk, pat)) == want_j


@pytest.mark.gpu
@pytest.mark.parametrize("poly", [0x12B, 0x163])
def test_gpu_batch_non_default_poly_r8(poly):
    """Bit-sliced batch path (>= 1024 codewords) with a runtime polynomial:
    BatchCodec encode / shared-pattern decode against the oracle built with
    the same polynomial."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_3458_b200 as lch
    ft = lch.tables_for(8, poly)
    bt = lch.build_basis_tables(ft, 256)
    codec = lch.BatchCodec(lch.CodeParams(8, 64), bt)
    msgs = O.gen_symbols(77, 8, 0, 2100, 64)
    cw = codec.encode(msgs)
    orc = O.Oracle(8, poly)
    np.testing.assert_array_equal(cw[:, 64:], orc.encode_batch(64, msgs, nthreads=8))
    er = set(gen_erasures_py(78, 256, 192, 0))
    rx = cw.copy()
    rx[:, sorted(er)] = 0x5A
    np.testing.assert_array_equal(codec.decode(rx, er), msgs)
