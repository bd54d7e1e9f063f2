"""Stall-reason totals and the top source lines by stall samples.  usage: python tools/ncu_stalls.py X.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
hdr = None
fname = None
agg = []
tot = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        samp = int(r[6])
    except (ValueError, IndexError):
        continue
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r) and r[i].isdigit() and int(r[i]) > 0:
            st[h[6:]] = int(r[i])
            tot[h[6:]] = tot.get(h[6:], 0) + int(r[i])
    agg.append((samp, f"{fname}:{r[0]}", r[1].strip()[:64], st))
T = sum(a[0] for a in agg) or 1
print("stall totals:", ", ".join(f"{k} {v / T:.0%}" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for samp, loc, src, st in sorted(agg, reverse=True)[:n]:
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{samp / T:6.1%} {loc:20s} {src:64s} {top}")
