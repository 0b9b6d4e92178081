#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list CSV (--metrics gpu__time_duration.sum) and
optionally a `--set full` report, into markdown.

usage: python scripts/ncu_summary.py launches.csv [prof.ncu-rep] [--traffic=profiles/step_traffic.json]
       > profiles/<name>.md
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


def launches(path, traffic_out=None):
    """Launch list with gpu__time_duration.sum (and optionally dram__bytes_read/write.sum) per
    launch; traffic_out: write the per-step DRAM bytes of the chain (sum over its kernels, mean
    over the listed steps) as JSON for bench.py's roofline.traffic."""
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = collections.OrderedDict()  # (launch id, kernel) -> {metric: value}
    for d in data:
        k = (d["ID"], d["Kernel Name"].split("(")[0].split("<")[0])
        per.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    by = collections.OrderedDict()
    for (_, name), m in per.items():
        by.setdefault(name, []).append(m)
    print(f"## Launch list ({path.split('/')[-1]}: cold-cache, serialised; compare shares)\n")
    print("| kernel | launches | mean time | median time | share of listed time | DRAM read / launch | DRAM write / launch |")
    print("|---|---|---|---|---|---|---|")
    tkey = "gpu__time_duration.sum"
    total = sum(sum(x.get(tkey, 0) for x in v) for v in by.values()) or 1
    for k, v in sorted(by.items(), key=lambda kv: -sum(x.get(tkey, 0) for x in kv[1])):
        ts = sorted(x.get(tkey, 0) for x in v)
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in v) / len(v)
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in v) / len(v)
        print(f"| {k} | {len(v)} | {sum(ts)/len(ts)/1e3:.2f} us | {ts[len(ts)//2]/1e3:.2f} us | "
              f"{100*sum(ts)/total:.1f}% | {rd/1e6:.3f} MB | {wr/1e6:.3f} MB |")
    print()
    if traffic_out:
        import json
        steps = min(len(v) for v in by.values())
        b = sum(sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in v) / len(v)
                for v in by.values())
        json.dump({"dram_bytes_per_launch": int(b), "steps": steps,
                   "per_kernel_bytes": {k: int(sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
                                                   for x in v) / len(v)) for k, v in by.items()},
                   "source": f"ncu launch list {path.split('/')[-1]}: dram__bytes_read.sum + dram__bytes_write.sum "
                             "of the five chain kernels of one step (mean over the listed steps; ncu replays each "
                             "kernel cold, so this is an upper bound of one step's DRAM traffic)"},
                  open(traffic_out, "w"), indent=1)


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
    traffic = None
    args = [a for a in sys.argv[1:] if not a.startswith("--traffic=")]
    for a in sys.argv[1:]:
        if a.startswith("--traffic="):
            traffic = a.split("=", 1)[1]
    launches(args[0], traffic)
    if len(args) > 1:
        full(args[1])
