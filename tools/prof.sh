#!/bin/bash
# ncu --set full capture of one launch of each kernel regex given: tools/prof.sh TAG regex1 [regex2 ...]
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rx in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o gpurun_out/prof_${rx}_$TAG \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_${rx}_$TAG.log 2>&1
done
