"""One stripe encode + decode (config 5 shapes) for launch-list profiling.

usage: python tools/prof_stripe.py K GROUPS [reps]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch  # noqa: E402
from paper_1404_3458_b200 import _lib, gen  # noqa: E402

N, P = 1 << 16, 2048
k, G = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
bt = lch.build_basis_tables(lch.tables_for(16), N)
ctx = bt.ctx.handle
s = torch.cuda.current_stream().cuda_stream
lanes = G * P
cw = torch.empty((G, N, P), dtype=torch.int16, device="cuda")
_lib.check(_lib.lib.lch_gen_packets(ctx, 5, 0, lanes, k, cw.data_ptr(), N, P, s))
out = torch.empty((G, k, P), dtype=torch.int16, device="cuda")
masks = gen.erasure_masks(bt.ctx, 7, N, N - k, 0, G)
bits = gen.mask_to_bits(masks).contiguous()
cnt = (ctypes.c_int64 * G)(*([N - k] * G))
par = cw.data_ptr() + k * P * 2
for i in range(reps):
    torch.cuda.nvtx.range_push("encode")
    _lib.check(_lib.lib.lch_encode_k(ctx, cw.data_ptr(), N, par, N, lanes, k, P, s))
    torch.cuda.nvtx.range_pop()
    _lib.check(_lib.lib.lch_decode_k(ctx, cw.data_ptr(), N, bits.data_ptr(), 0, out.data_ptr(), k,
                                     lanes, k, P, cnt, s))
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
_lib.check(_lib.lib.lch_encode_k(ctx, cw.data_ptr(), N, par, N, lanes, k, P, s))
ev[1].record()
_lib.check(_lib.lib.lch_decode_k(ctx, cw.data_ptr(), N, bits.data_ptr(), 0, out.data_ptr(), k,
                                 lanes, k, P, cnt, s))
ev[2].record()
torch.cuda.synchronize()
print(f"k={k} G={G}: encode {ev[0].elapsed_time(ev[1]):.3f} ms decode {ev[1].elapsed_time(ev[2]):.3f} ms",
      "ok" if torch.equal(out, cw[:, :k]) else "MISMATCH")
