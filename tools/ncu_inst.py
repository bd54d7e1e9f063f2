"""Executed warp instructions per source line (top N).  usage: python tools/ncu_inst.py X.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
hdr = None
fname = None
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    ki = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
    if ki is None or ki >= len(r):
        continue
    try:
        v = int(r[ki])
    except ValueError:
        continue
    rows.append((v, f"{fname}:{r[0]}", r[1].strip()[:70]))
T = sum(v for v, _, _ in rows) or 1
print("total", T)
for v, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{v / T:6.1%} {v:12d} {loc:22s} {src}")
