#!/bin/bash
# ncu --set full of each C5 (M = 64) kernel on a 1024-frame batch: tools/prof_c5.sh TAG regex...
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rx in "$@"; do
  rep=gpurun_out/prof_c5_${rx}_$TAG
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o $rep \
     python bench.py --workload c5 --frames 1024 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $rep.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
  echo "== $rx"; grep -E "Duration|bank|wavefronts_mem|fp64|dmma|stalls|Issue Slots|DRAM Throughput" $rep.summary.txt
done
