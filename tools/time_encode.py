"""Time RS(2^16,2^15) encode of 4096 codewords with CUDA events (experiments).

LCH_DBG_PASS=1 skips global I/O in the pass kernel, =2 skips butterflies
(results are then wrong; this only separates memory from compute time).
The flags need a library built with `make EXTRA=-DLCH_PASS_DBG`.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch  # noqa: E402
from paper_1404_3458_b200 import gen  # noqa: E402
from paper_1404_3458_b200.rs import encode_device  # noqa: E402

B = int(os.environ.get("B", "4096"))
K = 1 << 15
bt = lch.build_basis_tables(lch.tables_for(16), 1 << 16)
cp = lch.CodeParams(16, K)
msg = gen.symbols(bt.ctx, 1, 0, B, K)
par = torch.empty((B, K), dtype=torch.int16, device="cuda")
for _ in range(3):
    encode_device(cp, bt, msg, par)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    encode_device(cp, bt, msg, par)
e1.record()
torch.cuda.synchronize()
print(f"dbg={os.environ.get('LCH_DBG_PASS', '0')} B={B} encode_ms={e0.elapsed_time(e1) / n:.4f}")
