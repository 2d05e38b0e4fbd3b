#!/bin/bash
# Quick round-2 GPU iteration: build, GPU suite (optionally -k), single-frame sweep, c4 bench line,
# c4 launch list.   usage: tools/r02_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -20 $OUT/build_$TAG.log; exit 1; }
if [ -n "$2" ]; then timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$2" > $OUT/pytest_$TAG.log 2>&1;
else timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_$TAG.log 2>&1; fi
grep -E "passed|failed|error" $OUT/pytest_$TAG.log | tail -3; grep -E "^FAILED|Error" $OUT/pytest_$TAG.log | head -10
for w in c1 c2 c3_0.1 c3_0.001 c3_0.0001; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
done > $OUT/c3_sweep_$TAG.jsonl
python - "$OUT/c3_sweep_$TAG.jsonl" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        continue
    c = d["config"]
    print(f"{c['workload']:10s} L={c['L']:8d}  {d['ms_per_step']*1e3:8.1f} us/frame (4 algs)  {d['points_per_s']:.3g} pts/s launches/step {d['gpu_launches']/d['steps']:.0f}")
PY
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$TAG.jsonl 2> $OUT/bench_c4_$TAG.err
python - "$OUT/bench_c4_$TAG.jsonl" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]; n = d.get("north_star") or {}
    print("c4", round(d["value"]), "frames/s", round(d["ms_per_step"], 3), "ms/step; spectrum", round(r["kernel_ms"], 3),
          "ms frac", round(r["frac"], 3), "step_frac", round(r.get("step_frac", 0), 3), "| ns", round(n.get("value", 0)),
          "frames/s step_frac", round(n.get("step_frac", 0), 3), "| e2e", round((d.get("e2e") or {}).get("value", 0)), d["clocks"])
except Exception as e:
    print("bench failed", e); print(open(sys.argv[1].replace("jsonl", "err")).read()[-3000:])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_$TAG.csv > $OUT/launches_$TAG.txt; cat $OUT/launches_$TAG.txt
