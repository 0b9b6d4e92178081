#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list CSV (--metrics gpu__time_duration.sum) and
optionally a `--set full` report, into markdown.

usage: python scripts/ncu_summary.py launches.csv [prof.ncu-rep] > profiles/<name>.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    for d in data:
        by.setdefault(d["Kernel Name"].split("(")[0].split("<")[0], []).append(float(d["Metric Value"]))
    unit = data[0]["Metric Unit"] if data else "ns"
    print(f"## Launch list ({path.split('/')[-1]}: cold-cache, serialised; compare shares)\n")
    print("| kernel | launches | mean | median | share of listed time |")
    print("|---|---|---|---|---|")
    total = sum(sum(v) for v in by.values()) or 1
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        sv = sorted(v)
        print(f"| {k} | {len(v)} | {sum(v)/len(v)/1e3:.2f} us | {sv[len(sv)//2]/1e3:.2f} us | "
              f"{100*sum(v)/total:.1f}% |" if unit == "ns" else f"| {k} | {len(v)} | {sum(v)/len(v)} {unit} | | |")
    print()


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return
    hdr, units = r[0], r[1]
    print(f"## ncu --set full ({path.split('/')[-1]})\n")
    cols = [k for k in KEYS if k in hdr]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")].split("(")[0]
        vals = [f"{row[hdr.index(k)]} {units[hdr.index(k)]}".strip() for k in cols]
        print(f"| {name} | " + " | ".join(vals) + " |")
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    print("\nTop stall reasons (PC sampling share):\n")
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")].split("(")[0]
        items = []
        for h in stall:
            try:
                items.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(row[hdr.index(h)].replace(",", ""))))
            except ValueError:
                pass
        tot = sum(v for _, v in items) or 1
        items.sort(key=lambda x: -x[1])
        print(f"- {name}: " + ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in items[:5] if v))
    print()


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
