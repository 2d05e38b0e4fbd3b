#!/bin/bash
# A/B of libdoa builds on the c4 bench: tools/lib_ab.sh [WORKLOAD] lib1.so lib2.so ...  ("-" = in-tree libdoa.so)
WL=c4
if [[ "$1" != *.so && "$1" != "-" ]]; then WL=$1; shift; fi
for lib in "$@"; do
  if [ "$lib" = "-" ]; then unset DOA_LIB; else export DOA_LIB=$PWD/$lib; fi
  for rep in 1 2; do
  echo -n "$lib [$WL] "
  timeout 300 python bench.py --workload $WL --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']),'ms/step',round(d['ms_per_step'],3),'spec_ms',round(d['roofline']['kernel_ms'],4),'frac',round(d['roofline']['frac'],3))"
  done
done
