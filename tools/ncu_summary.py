"""Print the key roofline numbers of an ncu report (first kernel): duration, DRAM/L2/SM throughput,
occupancy, issue activity, dram bytes, instruction count.  usage: python tools/ncu_summary.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = {"Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Memory Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Instructions", "Grid Size", "Block Size", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Active Warps Per Scheduler"}
seen = set()
name = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if name is None:
        name = d.get("Kernel Name", "")[:110]
        print(name)
    m = d.get("Metric Name", "")
    if m in want and m not in seen:
        seen.add(m)
        print(f"  {m:38s} {d.get('Metric Value', '')} {d.get('Metric Unit', '')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units, v = rr[0], rr[1], rr[2]
for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
            "gpu__time_duration.sum"):
    if key in h:
        i = h.index(key)
        print(f"  {key:38s} {v[i]} {units[i]}")
