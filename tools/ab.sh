#!/bin/bash
# A/B env-var variants of the bench: tools/ab.sh "NAME=VAL" ["NAME2=VAL2" ...]; "-" = default
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "$@"; do
  if [ "$v" = "-" ]; then envs=""; else envs="$v"; fi
  echo "== $v"
  env $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']),'ms/step',round(d['ms_per_step'],3),'spec_ms',round(d['roofline']['kernel_ms'],3),'frac',round(d['roofline']['frac'],3))"
done
