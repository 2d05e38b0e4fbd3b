#!/bin/bash
# A/B of libdoa builds over batch sizes (c4 frames) and the ns workload: tools/batch_ab.sh lib1.so lib2.so ...
for lib in "$@"; do
  export DOA_LIB=$PWD/$lib
  for f in 8192 16384 65536; do
    echo -n "$lib frames=$f "
    timeout 300 python bench.py --frames $f --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-north-star 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']),'ms/step',round(d['ms_per_step'],3),'spec_ms',round(d['roofline']['kernel_ms'],4),'frac',round(d['roofline']['frac'],3))"
  done
  echo -n "$lib ns "
  timeout 300 python bench.py --workload ns --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']),'ms/step',round(d['ms_per_step'],3),'spec_ms',round(d['roofline']['kernel_ms'],4),'frac',round(d['roofline']['frac'],3))"
done
