#!/bin/bash
# Quick GPU check: gpu tests (optionally filtered) + a short bench; prints summaries.
K=${1:-}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log | tail; exit 1; }
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_quick.log 2>&1;
else timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; fi
tail -15 gpurun_out/pytest_quick.log | grep -vE "^\s*$|Warning|warnings|fork" | tail -12
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
python - <<'PY'
import json
try:
    d=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
    print("value", d['value'], "ms/step", d['ms_per_step'], "scan_ms", d['roofline']['kernel_ms'], "frac", d['roofline']['frac'], d['clocks'])
except Exception as e:
    print("bench failed", e); print(open('gpurun_out/bench_quick.log').read()[-2000:])
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_quick.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_quick.csv
