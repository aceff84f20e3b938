"""e2e host-buffer step: encode then decode on one thread vs the two independent
jobs issued from two host threads on two contexts/streams (experiment)."""
import os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch
from paper_1404_3458_b200 import gen
from paper_1404_3458_b200.rs import encode_device, encode_host, decode_host

N, K, B = 1 << 16, 1 << 15, 4096
bt = lch.build_basis_tables(lch.tables_for(16), N)
bt2 = lch.build_basis_tables(lch.tables_for(16), N)
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
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
reps = 6


def seq():
    with torch.cuda.stream(sa):
        for _ in range(reps):
            encode_host(cp, bt, h_msg, h_par)
            decode_host(cp, bt, h_rx, bits, h_out)
    torch.cuda.synchronize()


def conc():
    def ja():
        with torch.cuda.stream(sa):
            for _ in range(reps):
                encode_host(cp, bt, h_msg, h_par)
    def jb():
        with torch.cuda.stream(sb):
            for _ in range(reps):
                decode_host(cp, bt2, h_rx, bits, h_out)
    ta, tb = threading.Thread(target=ja), threading.Thread(target=jb)
    ta.start(); tb.start(); ta.join(); tb.join()
    torch.cuda.synchronize()


for name, fn in [("sequential", seq), ("concurrent", conc), ("sequential", seq), ("concurrent", conc)]:
    fn()
    t = time.perf_counter()
    fn()
    ms = (time.perf_counter() - t) * 1e3 / reps
    assert torch.equal(h_out, h_msg) and torch.equal(h_par, par.cpu())
    print(f"{name}: {ms:.2f} ms/step, e2e {2 * B * K * 2 / ms / 1e6:.1f} GB/s")
