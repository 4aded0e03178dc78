"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total us, share of the listed time.

usage: python scripts/launch_summary.py launches.csv [skip_first_n_launches]
"""
import csv
import re
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    if int(r["ID"]) < skip:
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("fmh::<unnamed>::", "")
    ns = float(r["Metric Value"].replace(",", ""))
    if r["Metric Unit"] == "us":
        ns *= 1e3
    elif r["Metric Unit"] == "ms":
        ns *= 1e6
    rows.append((name, ns))
agg = defaultdict(lambda: [0, 0.0])
for n, ns in rows:
    agg[n][0] += 1
    agg[n][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {tot / 1e3:.1f} us")
for n, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ns / tot * 100:6.2f}%  {c:6d}  {ns / 1e3:10.1f} us  {ns / c / 1e3:8.2f} us/launch  {n[:110]}")
