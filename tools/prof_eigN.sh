python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rep=gpurun_out/prof_eigN_c5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eigN -s 1 -c 1 -o $rep python bench.py --workload c5 --frames 1024 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $rep.log 2>&1
python tools/ncu_summary.py $rep.ncu-rep > $rep.summary.txt 2>&1
cat $rep.summary.txt
python tools/sass_hist.py $rep.ncu-rep 1024 2>/dev/null | head -30
