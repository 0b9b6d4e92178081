#!/usr/bin/env python
"""Per-source-line warp-stall samples of one ncu report (ncu --page source --print-source
cuda,sass), optionally restricted to a line range: python scripts/ncu_lines.py REP [lo hi] [top]."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10 ** 9)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = cur_line = None
hdr = None
agg = collections.Counter()
stall = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0] and r[0].isdigit():
        cur_line = int(r[0])
        src[(cur_file, cur_line)] = r[1]
    try:
        n = int(r[4]) if r[4] not in ("", "-") else 0
    except ValueError:
        n = 0
    if n and lo <= (cur_line or 0) <= hi:
        agg[(cur_file, cur_line)] += n
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    v = int(r[i])
                except ValueError:
                    continue
                if v:
                    stall[(cur_file, cur_line)][h[6:]] += v
tot = sum(agg.values())
print("samples", tot)
for (f, l), n in agg.most_common(top):
    t = ", ".join(f"{k}:{v}" for k, v in stall[(f, l)].most_common(3))
    print(f"{n:7d} {100 * n / max(tot, 1):5.1f}% {f}:{l} {src.get((f, l), '').strip()[:60]} | {t}")
