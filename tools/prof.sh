#!/bin/bash
# ncu --set full capture of one launch of each kernel regex; keeps a text summary (+ the .ncu-rep
# only when KEEP_REP=1, since gpurun_out is capped at 64 MiB).  tools/prof.sh TAG regex1 [regex2 ...]
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rx in "$@"; do
  rep=gpurun_out/prof_${rx}_$TAG
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o $rep \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $rep.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
  ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  if [ "$rx" = "scan_cta" ] || [ "$rx" = "scan_ws" ]; then python tools/traffic_from_ncu.py $rep.ncu-rep scan gpurun_out/traffic_$TAG.json; fi
  if [ "${KEEP_REP:-0}" != "1" ]; then rm -f $rep.ncu-rep; fi
done
du -sh gpurun_out
