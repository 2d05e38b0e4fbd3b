"""Per-opcode executed-instruction and stall-sample histogram of one kernel from an ncu report:
python tools/sass_hist.py rep.ncu-rep [units]   (units: divide counts, e.g. warp-blocks)"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[iss] or 0) for r in data) or 1
ops, smp = collections.Counter(), collections.Counter()
for r in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[ia].strip()).split()[0]
    ops[op] += int(r[iex] or 0)
    smp[op] += int(r[iss] or 0)
print(f"total executed {sum(ops.values()) / units:.1f} per unit; stall samples {tot}")
for op, c in ops.most_common(40):
    print(f"{op:28s} {c / units:9.1f}  samples {smp[op] / tot * 100:5.1f}%")
