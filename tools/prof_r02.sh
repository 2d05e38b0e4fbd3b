set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eig16h -s 1 -c 1 -o $OUT/prof_eig16h_r02b python tools/eig_once.py > $OUT/prof_eig16h_r02b.log 2>&1
python tools/ncu_summary.py $OUT/prof_eig16h_r02b.ncu-rep > $OUT/prof_eig16h_r02b.summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_cta -s 1 -c 1 -o $OUT/prof_scan_r02b python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > $OUT/prof_scan_r02b.log 2>&1
python tools/ncu_summary.py $OUT/prof_scan_r02b.ncu-rep > $OUT/prof_scan_r02b.summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_c3_001_r02b.csv python bench.py --workload c3_0.001 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph off > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c3_001_r02b.csv > $OUT/launches_c3_001_r02b.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_c1_r02b.csv python bench.py --workload c1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph off > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c1_r02b.csv > $OUT/launches_c1_r02b.txt
ls -la $OUT
