#!/bin/bash
# One GPU round: build, smoke, gpu tests, bench, ncu launch list, ncu full capture of the scan kernel.
# usage: tools/gpu_round.sh <tag> [skip-tests]
set -u
TAG=${1:-run}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1 || { echo SMOKE FAILED; tail -20 $OUT/smoke_$TAG.log; }
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1
  tail -3 $OUT/pytest_gpu_$TAG.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > $OUT/bench_$TAG.log 2>&1; tail -1 $OUT/bench_$TAG.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_stdout_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan -s 2 -c 1 -o $OUT/prof_scan_$TAG \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_stdout_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eig -s 1 -c 1 -o $OUT/prof_eig_$TAG \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_eig_stdout_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:covariance -s 1 -c 1 -o $OUT/prof_cov_$TAG \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_cov_stdout_$TAG.log 2>&1
ls -la $OUT
