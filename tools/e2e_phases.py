"""Host-buffer encode and decode timed separately (CUDA events around each call)."""
import sys, os, time
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
def timeit(fn, reps=4):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, (time.perf_counter() - t0) * 1e3 / reps
for name, fn in [("encode_host", lambda: encode_host(cp, bt, h_msg, h_par)),
                 ("decode_host", lambda: decode_host(cp, bt, h_rx, bits, h_out)),
                 ("both", lambda: (encode_host(cp, bt, h_msg, h_par), decode_host(cp, bt, h_rx, bits, h_out)))]:
    ev, wall = timeit(fn)
    print(f"{name}: {ev:.2f} ms (events), {wall:.2f} ms wall")
for mode in ("all", "auto", "all", "auto"):
    os.environ["LCH_COMPACT"] = mode
    ev, _ = timeit(lambda: decode_host(cp, bt, h_rx, bits, h_out), 6)
    ev2, _ = timeit(lambda: (encode_host(cp, bt, h_msg, h_par), decode_host(cp, bt, h_rx, bits, h_out)), 6)
    print(f"LCH_COMPACT={mode}: decode_host {ev:.2f} ms, both {ev2:.2f} ms")
