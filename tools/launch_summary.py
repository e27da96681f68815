"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_summary.py launches.csv [header-line ...]
Per kernel (template arguments stripped): launch count, total ns, share.
ncu's per-launch times are cold-cache and serialised: compare SHARES with
the bench's live per-kernel event timing, not absolute times.
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        name = re.sub(r"^void ", "", name).replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = re.sub(r"\(.*$", "", name)
        base = re.sub(r"<.*$", "", name).split("::")[-1]
        tmpl = re.search(r"<(.*)>", name)
        key = base + ("<" + tmpl.group(1) + ">" if tmpl and "matvec" in base else "")
        agg[key][0] += 1
        agg[key][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    for line in sys.argv[2:]:
        print(line)
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:60s} launches {n:6d}  total_ns {ns:16.0f}  share {100 * ns / tot:6.2f}%")


if __name__ == "__main__":
    main()
