"""Host survivor-compaction throughput (lch_compact_rows) on this machine."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3458_b200 as lch
from paper_1404_3458_b200 import _lib
bt = lch.build_basis_tables(lch.tables_for(16), 1 << 16)
n, rows = 1 << 16, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rx = np.random.default_rng(0).integers(0, 65536, (rows, n)).astype(np.uint16)
mask = np.zeros(n, bool); mask[np.random.default_rng(1).choice(n, n // 2, replace=False)] = True
bits = _lib.bitmask_from_positions(n, np.nonzero(mask)[0])
out = np.empty((rows, n // 2), np.uint16)
for _ in range(2):
    _lib.check(_lib.lib.lch_compact_rows(bt.ctx.handle, rx.ctypes.data, n, bits.ctypes.data, n, rows, out.ctypes.data, n // 2))
t = time.perf_counter()
for _ in range(3):
    _lib.check(_lib.lib.lch_compact_rows(bt.ctx.handle, rx.ctypes.data, n, bits.ctypes.data, n, rows, out.ctypes.data, n // 2))
dt = (time.perf_counter() - t) / 3
assert np.array_equal(out[:3], rx[:3][:, ~mask])
print(f"compact {rows} rows: {dt*1e3:.2f} ms, read {rows*n*2/dt/1e9:.1f} GB/s")
