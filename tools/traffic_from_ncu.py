"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of a kernel from an
`ncu --set full` report and record it for bench.py's roofline `traffic` field.

    python tools/traffic_from_ncu.py gpurun_out/prof_scan_cta_rXX.ncu-rep scan profiles/traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, vals = r[0], r[1], r[2]
d = dict(zip(h, vals))
u = dict(zip(h, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(name):
    return float(d[name].replace(",", "")) * scale.get(u[name], 1)


rec = {"kernel": d.get("Kernel Name", ""), "report": os.path.basename(rep),
       "dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
       "duration_ns_under_ncu": float(d["gpu__time_duration.sum"].replace(",", "")) if "gpu__time_duration.sum" in d else None}
rec["traffic_bytes"] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
db = json.load(open(out)) if os.path.exists(out) else {}
db[key] = rec
json.dump(db, open(out, "w"), indent=1)
print(json.dumps(rec))
