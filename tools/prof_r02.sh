#!/bin/bash
# Round-2 ncu captures (one launch each, --set full): the c4 scan (-> profiles/traffic.json), the
# frame kernel (eig16h<16, FUSE>), the covariance; plus the c4 launch list.  usage: tools/prof_r02.sh TAG
TAG=${1:-r02}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rx in scan_cta eig16h cov16_kernel; do
  rep=$OUT/prof_${rx}_$TAG
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o $rep \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star --graph off > $rep.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep > $OUT/ncu_${rx}_$TAG.summary.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/ncu_${rx}_$TAG.raw.csv.gz
done
python tools/traffic_from_ncu.py $OUT/prof_scan_cta_$TAG.ncu-rep scan $OUT/traffic_$TAG.json
cat $OUT/traffic_$TAG.json
for rx in scan_cta eig16h cov16_kernel; do echo "== $rx"; head -16 $OUT/ncu_${rx}_$TAG.summary.txt; tail -6 $OUT/ncu_${rx}_$TAG.summary.txt; done
rm -f $OUT/prof_eig16h_$TAG.ncu-rep $OUT/prof_cov16_kernel_$TAG.ncu-rep
