"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): the
launches of each (kernel, grid) in order of first launch, with count, total,
per-launch time and share of the whole.
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
runs = {}  # (kernel, grid) in order of first launch
for name, grid, us in rows:
    r = runs.setdefault((name, grid), [name, grid, 0, 0.0])
    r[2] += 1
    r[3] += us
runs = list(runs.values())
title = sys.argv[2] if len(sys.argv) > 2 else ""
print(f"{title}total {total / 1e3:.2f} ms over {len(rows)} launches")
for name, grid, n, us in runs:
    print(f"{n:5d} {us:10.1f}us {us / n:9.2f}us/launch {100 * us / total:5.1f}%  grid{grid} {name[:90]}")
