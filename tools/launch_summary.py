"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): runs
of consecutive launches of the same kernel and grid, in launch order, with
count, total, per-launch time and share of the whole.
    python tools/launch_summary.py launches.csv [title]"""
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.DictReader(lines)
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
    name = re.sub(r"\(.*$", "", r["Kernel Name"]).replace("dfm::", "").replace("<unnamed>::", "")
    rows.append((name, r["Grid Size"], us))
total = sum(r[2] for r in rows)
runs = []
for name, grid, us in rows:
    if runs and runs[-1][0] == name and runs[-1][1] == grid:
        runs[-1][2] += 1
        runs[-1][3] += us
    else:
        runs.append([name, grid, 1, us])
title = sys.argv[2] if len(sys.argv) > 2 else ""
print(f"{title}total {total / 1e3:.2f} ms over {len(rows)} launches")
for name, grid, n, us in runs:
    print(f"{n:5d} {us:10.1f}us {us / n:9.2f}us/launch {100 * us / total:5.1f}%  grid{grid} {name[:90]}")
