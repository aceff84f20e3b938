"""e2e (host-buffer API) step time vs chunk size (rows per chunk)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch
from paper_1404_3458_b200 import gen
from paper_1404_3458_b200.rs import encode_device, encode_host, decode_host

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
for ce, cd in [(0, 0), (1024, 1024), (512, 1024), (2048, 1024), (1024, 2048), (0, 1024), (512, 512)]:
    def step():
        encode_host(cp, bt, h_msg, h_par, ce)
        decode_host(cp, bt, h_rx, bits, h_out, cd)
    step(); step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 4
    assert torch.equal(h_out, h_msg)
    print(f"chunks enc={ce} dec={cd}: {ms:.2f} ms/step, e2e {2 * B * K * 2 / ms / 1e6:.1f} GB/s")
