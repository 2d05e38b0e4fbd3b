bash tools/r02_check.sh r02x
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_r02x.jsonl 2>gpurun_out/bench_c5_r02x.err; tail -c 600 gpurun_out/bench_c5_r02x.jsonl
bash tools/c3_sweep.sh; cp gpurun_out/c3_sweep.jsonl gpurun_out/c3_sweep_r02x.jsonl
bash tools/prof.sh r02x scan_cta
