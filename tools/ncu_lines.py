"""Executed warp instructions per CUDA source line of an ncu report captured
with --import-source on (library built with -lineinfo).

usage: python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    start = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[start]
    li, ie, st = hdr.index("Line No"), hdr.index("Instructions Executed"), hdr.index("# Samples")
    agg, smp, text, cur = defaultdict(int), defaultdict(int), {}, None
    for r in rows[start + 1:]:
        if len(r) <= ie:
            continue
        if r[li].strip():
            cur = r[li]
            text[cur] = r[1]
            continue  # the line's own row repeats the sum of its SASS rows
        try:
            agg[cur] += int(r[ie])
            smp[cur] += int(r[st])
        except (ValueError, TypeError):
            pass
    tot, ts = sum(agg.values()) or 1, sum(smp.values()) or 1
    print(f"total warp instructions {tot}, stall samples {ts}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v / tot * 100:5.1f}% inst {smp[k] / ts * 100:5.1f}% samples  line {k}: {text[k].strip()[:100]}")


if __name__ == "__main__":
    main()
