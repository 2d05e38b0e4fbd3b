#!/bin/bash
# The paper's own workload on B200 (NEXT-1): 8-element UCA, MUSIC+PHD+EV+MN, scan ranges
# 360 x {1, 30, 60, 90} (Tables 8/10), single frame (latency) and 4096-frame batches.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY' > gpurun_out/paper_sweep.jsonl
import json, subprocess, sys
from synth.array import ARRAY_CONFIGS
for nel in (1, 30, 60, 90):
    for frames in (1, 4096):
        name = "e1" if nel == 1 else "e1_360x90"
        cmd = [sys.executable, "bench.py", "--workload", name, "--frames", str(frames), "--steps", "20",
               "--warmup", "5", "--no-e2e", "--no-cpu-baseline"]
        env = {"DOA_BENCH_NEL": str(nel)}
        import os
        r = subprocess.run(cmd, capture_output=True, text=True, env={**os.environ, **env})
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-500:]})
        print(line, flush=True)
PY
cat gpurun_out/paper_sweep.jsonl | cut -c1-300
