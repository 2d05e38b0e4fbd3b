"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, mean, share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
            name = d["Kernel Name"].split("(")[0][-48:]
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':50s} {'n':>4s} {'mean_us':>10s} {'total_us':>10s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {n:4d} {t / n:10.1f} {t:10.1f} {t / tot:6.1%}")
