"""Write profiles/<round>/traffic.json (the `traffic` of bench.py's roofline) from ncu_<kind>_<cfg>.txt summaries:
dram__bytes_read.sum + dram__bytes_write.sum of one `ncu --set full` launch per kernel kind and workload.
usage: python tools/make_traffic.py DIR  (reads DIR/ncu_{fwd,bwd}_cfg{3,4,5}.txt, writes DIR/traffic.json)"""
import json
import os
import re
import sys

d = sys.argv[1]
names = {3: "cfg3-rgg20k-k6", 4: "cfg4-road200x200", 5: "cfg5-rgg5k-k8-many"}
out = {"note": "ncu --set full --clock-control none, one launch per kernel kind (tools/prof.py --config C --sweeps 1, "
               "launch 20 of the kind), dram__bytes_read.sum + dram__bytes_write.sum per launch; keyed by bench "
               "workload and kernel kind; summaries in ncu_*.txt"}
for cfg, wl in names.items():
    for kind, key in (("fwd", "fwd_fused"), ("bwd", "bwd_step")):
        path = os.path.join(d, f"ncu_{kind}_cfg{cfg}.txt")
        if not os.path.exists(path):
            continue
        txt = open(path).read()
        lines = txt.splitlines()
        if not lines:
            continue
        m = {k: re.search(rf"{k}\s+([0-9.]+)\s+(\w+)", txt) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                                                      "gpu__time_duration.sum")}
        if not all(m.values()):
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(m["dram__bytes_read.sum"].group(1)) * scale.get(m["dram__bytes_read.sum"].group(2), 1)
        wr = float(m["dram__bytes_write.sum"].group(1)) * scale.get(m["dram__bytes_write.sum"].group(2), 1)
        us = float(m["gpu__time_duration.sum"].group(1)) * (1e-3 if m["gpu__time_duration.sum"].group(2) == "nsecond" else 1)
        out.setdefault(wl, {})[key] = {"kernel": lines[0].split("(")[0].replace("void ", "").strip(), "dram_read": int(rd), "dram_write": int(wr),
                                       "duration_us": round(us, 2)}
json.dump(out, open(os.path.join(d, "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
