"""A/B timing of RS(2^16,2^15) encode + shared-pattern decode of 4096
codewords with CUDA events (experiments; LCH_SO_PATH selects a library build).
Checks decode(encode(m)) == m first.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch  # noqa: E402
from paper_1404_3458_b200 import gen  # noqa: E402
from paper_1404_3458_b200.rs import decode_device, encode_device  # noqa: E402

B = int(os.environ.get("B", "4096"))
N, K = 1 << 16, 1 << 15
REPS = int(os.environ.get("REPS", "10"))
bt = lch.build_basis_tables(lch.tables_for(16), N)
cp = lch.CodeParams(16, K)
msg = gen.symbols(bt.ctx, 1404345803, 0, B, K)
cw = torch.empty((B, N), dtype=torch.int16, device="cuda")
cw[:, :K].copy_(msg)
emask = gen.erasure_masks(bt.ctx, 1404345804, N, N - K, 0, 1)
bits = gen.mask_to_bits(emask)[0].contiguous()
out = torch.empty((B, K), dtype=torch.int16, device="cuda")
encode_device(cp, bt, msg, cw[:, K:])
rx = cw.clone()
rx[:, emask[0]] = 0
decode_device(cp, bt, rx, bits, out, N - K)
torch.cuda.synchronize()
ok = bool(torch.equal(out, msg))


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(REPS):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS


enc = timeit(lambda: encode_device(cp, bt, msg, cw[:, K:]))
dec = timeit(lambda: decode_device(cp, bt, cw, bits, out, N - K))
print(json.dumps({"lib": os.environ.get("LCH_SO_PATH", "default"), "roundtrip_ok": ok,
                  "encode_ms": round(enc, 4), "decode_ms": round(dec, 4),
                  "headline_gbs": round(2 * B * K * 2 / ((enc + dec) * 1e-3) / 1e9, 2)}))
