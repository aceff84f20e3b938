"""Per-opcode / per-region breakdown of an ncu source page (SASS) export.

  ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
  python tools/sass_profile.py src.csv [launch_index]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur is not None and len(r) > 5:
        cur.append(r)
H = {h: i for i, h in enumerate(hdr)}
b = blocks[which]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
execd = sum(int(r[H["Instructions Executed"]]) for r in b)
tot = sum(int(r[H["# Samples"]]) for r in b)
c, s = Counter(), Counter()
st = {}
for r in b:
    t = r[H["Source"]].strip().split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += int(r[H["Instructions Executed"]])
    s[op] += int(r[H["# Samples"]])
    d = st.setdefault(op, Counter())
    for k in stall_cols:
        d[k] += int(r[H[k]] or 0)
print(f"instructions executed (warp) {execd}, samples {tot}")
print("op           exec%   samples%  top stalls")
for op, n in c.most_common(16):
    top = ", ".join(f"{k[6:]}={v}" for k, v in st[op].most_common(3) if v)
    print(f"{op:10s} {100 * n / execd:6.1f}%  {100 * s[op] / tot:6.1f}%   {top}")
allst = Counter()
for d in st.values():
    allst.update(d)
print("stalls:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in allst.most_common(10)))
