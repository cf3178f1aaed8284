#!/usr/bin/env python
"""Summarise an ncu report and a launch list into profiles/<round>_summary.md.

    python profiles/ncu_summary.py <report.ncu-rep> <launches.csv> <out prefix>

Writes <prefix>_ncu_raw.csv (selected metrics per captured launch),
<prefix>_launches.csv (copy of the launch list) and <prefix>_summary.md.
"""
import collections
import csv
import io
import shutil
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stalls / issue"),
]


def main(rep, launches, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    cols = ["Kernel Name"] + [m for m, _ in METRICS if m in hdr]
    idx = [hdr.index(c) for c in cols]
    with open(prefix + "_ncu_raw.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(cols)
        w.writerow([units[i] for i in idx])
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
    shutil.copy(launches, prefix + "_launches.csv")
    text = open(launches).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    lrows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    agg = collections.defaultdict(list)
    for r in lrows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        if name.startswith("sphbuf::"):
            name = name[len("sphbuf::"):]
        if not name.startswith("k_"):
            continue          # input generation etc. (torch), not the library
        agg[name].append(float(r["Metric Value"]))
    tot = sum(sum(v) for k, v in agg.items() if "register" not in k)
    out = [f"# ncu summary ({prefix.split('/')[-1]})", "",
           "## Launch list (gpu__time_duration.sum, cold-cache and serialised: compare shares)", "",
           "| kernel | launches | mean us | share of step kernels |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = sum(v) / tot if "register" not in k else 0.0
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {share:.3f} |")
    out += ["", "## Captured launches (ncu --set full)", "",
            "| kernel | " + " | ".join(lbl for m, lbl in METRICS if m in hdr) + " |",
            "|---|" + "---|" * len(cols[1:])]
    for r in rows[2:]:
        vals = [r[i] for i in idx]
        name = vals[0].split("(")[0].replace("void ", "")[:40]
        out.append(f"| {name} | " + " | ".join(vals[1:]) + " |")
    out += ["", "units: " + ", ".join(f"{lbl}={units[hdr.index(m)]}" for m, lbl in METRICS if m in hdr)]
    open(prefix + "_summary.md", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:4])
