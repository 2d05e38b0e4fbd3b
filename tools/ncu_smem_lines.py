"""Per-SASS-instruction shared-memory wavefronts (and stall samples) from an ncu report's source
page: python tools/ncu_smem_lines.py rep.ncu-rep [units] [top]  (units: divide counts, e.g.
warp-rounds)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, iex, iwf, iid, ism = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                                      "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                                      "Warp Stall Sampling (All Samples)"))
tot, lst = 0.0, []
for r in rows[2:]:
    try:
        wf = float(r[iwf] or 0)
    except ValueError:
        continue
    tot += wf
    if wf > 0:
        lst.append((wf, r[ia][-5:], r[isrc].strip()[:64], float(r[iex] or 0), float(r[iid] or 0), r[ism]))
print(f"total shared wavefronts per unit: {tot / units:.1f}")
lst.sort(key=lambda x: -x[0])
for wf, ad, src, ex, idl, sm in lst[:top]:
    print(f"{ad} {wf / units:7.2f} (ideal {idl / units:6.2f}, exec {ex / units:5.2f}, stall samples {sm:>6})  {src}")
