#!/bin/bash
# BASELINE configs[0-2] on B200: C1 (M=8, 1 deg) and the paper-style scan-resolution sweep C3
# (M=16, D=3, N=1024, one frame, 0.1 -> 0.0001 deg, L up to 1.8M points), all four estimators per
# step, CUDA-graph replay, inputs resident; plus the oracle's time per frame for the same frame.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in c1 c2 c3_0.1 c3_0.001 c3_0.0001; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 10 --no-e2e --cpu-seconds 5 2>/dev/null | tail -1
done > gpurun_out/c3_sweep.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/c3_sweep.jsonl"):
    d = json.loads(l)
    c = d["config"]
    cpu = d.get("cpu_baseline") or {}
    print(f"{c['workload']:10s} L={c['L']:8d}  {d['ms_per_step']*1e3:8.1f} us/frame (4 algs)  "
          f"{d['points_per_s']:.3g} pts/s  oracle {1e6/cpu.get('value',float('nan')) if cpu else float('nan'):.0f} us/frame")
PY
