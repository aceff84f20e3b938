"""Steady-state trace of the host-buffer pipeline: STEPS x (encode_host +
decode_host) queued without host syncs under LCH_PIPE_TRACE=1; the per-chunk
stage timestamps (ms since the first call) are printed by
lch_release_host_buffers.  Experiments only."""
import os
import sys
import time

import numpy as np
import torch

os.environ["LCH_PIPE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch  # noqa: E402
from paper_1404_3458_b200 import _lib, gen  # noqa: E402
from paper_1404_3458_b200.rs import decode_host, encode_device, encode_host  # noqa: E402

N, K, B = 1 << 16, 1 << 15, 4096
STEPS = int(os.environ.get("STEPS", "6"))
bt = lch.build_basis_tables(lch.tables_for(16), N)
cp = lch.CodeParams(16, K)
msg = gen.symbols(bt.ctx, 1, 0, B, K)
par = torch.empty((B, K), dtype=torch.int16, device="cuda")
encode_device(cp, bt, msg, par)
mask = gen.erasure_masks(bt.ctx, 2, N, N - K, 0, 1)
bits = gen.mask_to_bits(mask)[0].cpu().numpy().view(np.uint32).copy()
rx = torch.cat([msg, par], 1)
rx[:, mask[0]] = 0
h_msg, h_rx = msg.cpu().pin_memory(), rx.cpu().pin_memory()
h_par = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
h_out = torch.empty((B, K), dtype=torch.int16, pin_memory=True)
chunk = int(os.environ.get("CHUNK", "0"))
for rep in range(1):  # the first steps warm up (allocations): read the last ones
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stamps = []
    for _ in range(STEPS):
        encode_host(cp, bt, h_msg, h_par, chunk)
        stamps.append(time.perf_counter() - t0)
        decode_host(cp, bt, h_rx, bits, h_out, chunk)
        stamps.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"rep {rep}: {STEPS} steps in {1e3 * (t1 - t0):.2f} ms; host returned from the calls at (ms)",
          " ".join(f"{1e3 * s:.2f}" for s in stamps), flush=True)
    _lib.check(_lib.lib.lch_release_host_buffers(bt.ctx.handle))
assert torch.equal(h_out, msg.cpu())
