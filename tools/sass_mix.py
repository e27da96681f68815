"""Opcode mix of one kernel from `ncu -i rep --page source --csv --print-source sass`.
usage: python tools/sass_mix.py sass.csv [entries]   (entries: divide counts per unit)"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, ie, iss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cnt, stall = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    src = r[ia].strip()
    m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    op = m.group(2)
    cnt[op] += float(r[ie] or 0)
    stall[op] += float(r[iss] or 0)
tot = sum(cnt.values())
print(f"total warp-instructions {tot:.4g}; per unit x32 threads: {32 * tot / units:.1f}")
for op, n in cnt.most_common(40):
    print(f"{op:12s} {n:14.0f} {100 * n / tot:6.2f}%  per-unit(thread) {32 * n / units:7.2f}  stall-samples {stall[op]:.0f}")
