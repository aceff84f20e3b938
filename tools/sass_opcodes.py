"""Static SASS opcode summary of every pass_kernel instance (and the other
kernels) in the built library: instruction count and the opcodes that prove
the B200 paths (UBLKCP = 1-D bulk copy, UTMALDG / UTMASTG = tensor-map TMA,
SYNCS = mbarrier, LOP3 = the bit-sliced arithmetic).  No GPU needed.

  python tools/sass_opcodes.py paper_1404_3458_b200/_build > profiles/r02_sass_opcodes.md
"""
import glob
import os
import re
import subprocess
import sys
from collections import Counter

build = sys.argv[1] if len(sys.argv) > 1 else "paper_1404_3458_b200/_build"
KEYS = ["LOP3", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "BAR", "LDS", "STS", "LDG", "STG", "BRA", "SHFL",
        "IMAD", "PRMT", "SHF", "BRX"]
print("# SASS opcode summary per kernel (static counts, `cuobjdump -sass`)\n")
print("| object | kernel | instructions | " + " | ".join(KEYS) + " |")
print("|---|---|---|" + "---|" * len(KEYS))
for obj in sorted(glob.glob(os.path.join(build, "*.o"))):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, cnt = None, Counter()
    rows = []

    def flush():
        if fn and sum(cnt.values()):
            rows.append((fn, cnt.copy()))

    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            flush()
            fn, cnt = m.group(1), Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            cnt[m.group(2)] += 1
            cnt["_total"] += 1
    flush()
    for f, c in rows:
        short = f.replace("_ZN3lch", "lch::")[:60]
        print(f"| {os.path.basename(obj)} | `{short}` | {c['_total']} | " +
              " | ".join(str(c[k]) for k in KEYS) + " |")
