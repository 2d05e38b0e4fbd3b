#!/bin/bash
# A/B the scan kernel builds: default (2 CTAs/SM) vs DOA_SCAN_MINB=3.
./tools/fp64_peaks > gpurun_out/fp64_peaks_mix.txt 2>&1
for v in default build_variants/libdoa_minb3.so; do
  if [ "$v" = default ]; then unset DOA_LIB; else export DOA_LIB=$PWD/$v; fi
  echo "== $v" >> gpurun_out/scan_variants.txt
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> gpurun_out/scan_variants.txt 2>&1
done
unset DOA_LIB
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_v2.log 2>&1; tail -2 gpurun_out/pytest_gpu_v2.log
cat gpurun_out/scan_variants.txt gpurun_out/fp64_peaks_mix.txt
