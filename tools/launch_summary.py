"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name, launches,
total and mean device time, share.  usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "nsecond")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    name = d["Kernel Name"].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += v * scale
tot = sum(v[1] for v in agg.values()) or 1.0
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {n:8d} {us:12.1f} {us / n:10.2f} {us / tot:7.1%}")
