#!/bin/bash
# Round-2 GPU check: build + smoke, the full GPU suite (tie counts -> gpurun_out/parity_ties.json),
# the default bench line (c4 + north_star + e2e + cpu baseline), a 2-rank strong-scaling bench on
# one GPU (gloo test hook), and the launch list of one c4 step.
TAG=${1:-r02a}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_gpu_$TAG.log 2>&1; tail -4 $OUT/pytest_gpu_$TAG.log
cp $OUT/parity_ties.json $OUT/parity_ties_$TAG.json 2>/dev/null
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4_$TAG.jsonl 2> $OUT/bench_c4_$TAG.err; tail -c 2500 $OUT/bench_c4_$TAG.jsonl; tail -3 $OUT/bench_c4_$TAG.err
DOA_BENCH_ONE_GPU=1 DOA_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-north-star \
  > $OUT/bench_2rank_$TAG.jsonl 2> $OUT/bench_2rank_$TAG.err; tail -c 1200 $OUT/bench_2rank_$TAG.jsonl; tail -3 $OUT/bench_2rank_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_$TAG.csv > $OUT/launches_$TAG.txt; cat $OUT/launches_$TAG.txt
