#!/bin/bash
# Round measurement: smoke, full gpu tests, bench (c4 with e2e + cpu baseline, clocks), ns bench,
# reference arm, ncu launch list + full captures of every kernel of the step.
TAG=${1:-r01}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1; tail -1 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4_$TAG.jsonl 2> $OUT/bench_c4_$TAG.err; tail -c 1500 $OUT/bench_c4_$TAG.jsonl
timeout 900 python bench.py --workload ns --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_ns_$TAG.jsonl 2> $OUT/bench_ns_$TAG.err; tail -c 600 $OUT/bench_ns_$TAG.jsonl
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.jsonl 2> $OUT/bench_ref_$TAG.err; tail -c 400 $OUT/bench_ref_$TAG.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_$TAG.csv > $OUT/launches_$TAG.txt; cat $OUT/launches_$TAG.txt
bash tools/prof.sh $TAG scan_cta eig16h cov16 coef_mma select_kernel
