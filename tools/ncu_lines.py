"""Per-CUDA-source-line instruction and stall-sample totals from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py X.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
fname = None
hdr = None
agg = []
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
    d = dict(zip(hdr[2:], r[2:]))  # skip the duplicated 'Source' column pair
    try:
        ex = int(r[7])
        samp = int(r[6])
    except (ValueError, IndexError):
        continue
    agg.append((ex, samp, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(a[0] for a in agg) or 1
tots = sum(a[1] for a in agg) or 1
print(f"total warp-instructions {tot:.3e}, samples {tots}")
for ex, samp, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{ex / tot:6.1%} {samp / tots:6.1%}  {loc:18s} {src}")
