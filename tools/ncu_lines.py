#!/usr/bin/env python
"""Aggregate an ncu source page (sass,cuda) by CUDA source line.

    python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top] [--stall]   (--stall: sort by stall samples)
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    by_stall = "--stall" in sys.argv
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                          "sass,cuda"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    iE = h.index("Instructions Executed")
    iS = h.index("Warp Stall Sampling (All Samples)")
    agg = collections.defaultdict(lambda: [0, 0, ""])
    seen = set()
    for r in rows[1:]:
        if len(r) != len(h) or not r[0].strip():
            continue
        key = (r[0], r[2])
        if key in seen:
            continue
        seen.add(key)
        try:
            e, s = int(r[iE] or 0), int(r[iS] or 0)
        except ValueError:
            continue
        a = agg[r[0]]
        a[0] += e
        a[1] += s
        a[2] = r[1][:90]
    te = sum(a[0] for a in agg.values()) or 1
    ts = sum(a[1] for a in agg.values()) or 1
    print(f"total warp instructions {te}, stall samples {ts}")
    for ln, (e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1 if by_stall else 0])[:top]:
        print(f"{ln:>5} inst {e / te:6.1%} stall {s / ts:6.1%}  {src}")


if __name__ == "__main__":
    main()
