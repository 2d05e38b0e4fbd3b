#!/bin/bash
# NEXT-2 GPU check: build, the fp32-engine tests + full GPU suite, c4 bench with the fp32 engine,
# one ncu --set full capture of scan_f32_kernel.   usage: tools/r02_fp32.sh TAG
TAG=${1:-f32}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -20 $OUT/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_$TAG.log 2>&1
grep -E "passed|failed|error" $OUT/pytest_$TAG.log | tail -3; grep -E "^FAILED|Error" $OUT/pytest_$TAG.log | head -10
cat $OUT/fp32_engine.json | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v) for k,v in d.items()]"
timeout 900 python bench.py --engine direct_fp32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > $OUT/bench_c4_f32_$TAG.jsonl 2> $OUT/bench_c4_f32_$TAG.err
tail -1 $OUT/bench_c4_f32_$TAG.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fp32 engine c4', round(d['value']), 'frames/s', round(d['ms_per_step'],2), 'ms/step; scan', round(r['kernel_ms'],3), 'ms/launch', round(r['achieved'],2), 'TFLOP/s frac', round(r['frac'],3))" || tail -5 $OUT/bench_c4_f32_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_f32 -s 4 -c 1 -o $OUT/prof_scan_f32_$TAG \
  python bench.py --engine direct_fp32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star --graph off > $OUT/prof_scan_f32_$TAG.log 2>&1
python tools/ncu_summary.py $OUT/prof_scan_f32_$TAG.ncu-rep > $OUT/ncu_scan_f32_$TAG.summary.txt 2>&1
ncu -i $OUT/prof_scan_f32_$TAG.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/ncu_scan_f32_$TAG.raw.csv.gz
cat $OUT/ncu_scan_f32_$TAG.summary.txt
