#!/bin/bash
# Late round-2 GPU check: tools/r02_check.sh (smoke, GPU suite with tie counts, default c4 bench line,
# 2-rank strong-scaling run, c4 launch list) + C5, the single-frame sweep, the paper UCA sweep with
# its launch list, the c4 scan's ncu --set full capture and the small-batch (8-GPU share) c4 line.
TAG=${1:-r02z}
bash tools/r02_check.sh $TAG
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_$TAG.jsonl 2>/dev/null; tail -c 400 gpurun_out/bench_c5_$TAG.jsonl
bash tools/c3_sweep.sh; cp gpurun_out/c3_sweep.jsonl gpurun_out/c3_sweep_$TAG.jsonl
bash tools/paper_sweep.sh > /dev/null 2>&1; cp gpurun_out/paper_sweep.jsonl gpurun_out/paper_sweep_$TAG.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_e1_$TAG.csv \
   python bench.py --workload e1_360x90 --frames 4096 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_e1_$TAG.csv > gpurun_out/launches_e1_$TAG.txt
timeout 300 python bench.py --frames 8192 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-north-star > gpurun_out/bench_c4_8192_$TAG.jsonl 2>/dev/null
bash tools/prof.sh $TAG scan_cta
