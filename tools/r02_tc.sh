#!/bin/bash
# tcgen05 NEXT-2 engine: engine tests, c4 bench with each engine, ncu of scan_tc_kernel.  tools/r02_tc.sh TAG
TAG=${1:-tc}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fp32_engine.py -q -p no:cacheprovider 2>&1 | tail -3
python -c "import json; d=json.load(open('$OUT/fp32_engine.json')); [print(k, v) for k, v in d.items() if 'tf32' in k]"
for eng in direct_tf32x3; do
  timeout 900 python bench.py --engine $eng --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > $OUT/bench_c4_${eng}_$TAG.jsonl 2>$OUT/bench_c4_${eng}_$TAG.err
  tail -1 $OUT/bench_c4_${eng}_$TAG.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$eng c4', round(d['value']), 'frames/s', round(d['ms_per_step'],2), 'ms/step; scan', round(r['kernel_ms'],3), 'ms/launch', round(r['achieved'],1), 'TFLOP/s frac', round(r['frac'],3))" || tail -5 $OUT/bench_c4_${eng}_$TAG.err
done
timeout 900 ncu --set full --clock-control none -k regex:scan_tc -s 1 -c 1 -o $OUT/prof_scan_tc_$TAG \
  python bench.py --engine direct_tf32x3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star --graph off > $OUT/prof_scan_tc_$TAG.log 2>&1
python tools/ncu_summary.py $OUT/prof_scan_tc_$TAG.ncu-rep > $OUT/ncu_scan_tc_$TAG.summary.txt 2>&1
ncu -i $OUT/prof_scan_tc_$TAG.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/ncu_scan_tc_$TAG.raw.csv.gz
cat $OUT/ncu_scan_tc_$TAG.summary.txt
zcat $OUT/ncu_scan_tc_$TAG.raw.csv.gz | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in h:
    if 'tensor' in k and 'pct' in k and 'sustained_active' in k: print(k, v[h.index(k)])
" | head -12
