"""Summarise an ncu --page source --print-source=sass CSV: hottest SASS instructions by executed
count and by stall samples.  usage: ncu -i X.ncu-rep --page source --csv --print-source=sass > s.csv;
python tools/ncu_sass.py s.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot_exec = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
tot_samp = sum(int(r[ix["# Samples"]] or 0) for r in data)
print(f"instructions: {len(data)}  executed(warp) {tot_exec:.3e}  samples {tot_samp}")
stall_cols = [h for h in hdr if h.startswith("stall_")]
print("stalls:", {h: sum(int(r[ix[h]] or 0) for r in data) for h in stall_cols if sum(int(r[ix[h]] or 0) for r in data)})
print(f"{'idx':>5} {'exec':>10} {'samp':>6}  sass")
for k, r in enumerate(data):
    ex = int(r[ix["Instructions Executed"]] or 0)
    sa = int(r[ix["# Samples"]] or 0)
    if ex > tot_exec / n / 4 or sa > tot_samp / n:
        st = {h[6:]: int(r[ix[h]]) for h in stall_cols if int(r[ix[h]] or 0) > sa / 4 and sa > 5}
        print(f"{k:5d} {ex:10d} {sa:6d}  {r[ix['Source']].strip()[:70]:70s} {st}")
