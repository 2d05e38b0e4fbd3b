#!/bin/bash
# A/B the scan kernel: bench c4 with the default libdoa.so and every build_variants/*.so (built
# with -D overrides of the DOA_* knobs in csrc/); extra args = env settings for all.  Full logs
# go to gpurun_out/variant_<name>.log.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/variants_build.log 2>&1
for v in default build_variants/*.so; do
  if [ "$v" = default ]; then unset DOA_LIB; else export DOA_LIB=$PWD/$v; fi
  log=gpurun_out/variant_$(basename $v .so).log
  printf "%-36s " "$v"
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $log 2>&1
  tail -1 $log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value']),'ms/step',round(d['ms_per_step'],3),'spec_ms',round(d['roofline']['kernel_ms'],3),'frac',round(d['roofline']['frac'],3))" 2>/dev/null || { echo "FAILED:"; tail -5 $log; }
done
