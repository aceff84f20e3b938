"""One encode_host + one decode_host with LCH_PIPE_TRACE=1 (per-chunk stage
timestamps on stderr) and per-call wall times.  Experiments only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch  # noqa: E402
from paper_1404_3458_b200 import gen  # noqa: E402
from paper_1404_3458_b200.rs import decode_host, encode_device, encode_host  # noqa: E402

N, K, B = 1 << 16, 1 << 15, 4096
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
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    encode_host(cp, bt, h_msg, h_par, chunk)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    decode_host(cp, bt, h_rx, bits, h_out, chunk)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: encode_host {1e3 * (t1 - t0):.2f} ms, decode_host {1e3 * (t2 - t1):.2f} ms", flush=True)
assert torch.equal(h_out, msg.cpu())
