OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eig16h -s 1 -c 1 -o $OUT/prof_eig16h_r02h python tools/eig_once.py > $OUT/prof_eig16h_r02h.log 2>&1
python tools/ncu_summary.py $OUT/prof_eig16h_r02h.ncu-rep > $OUT/prof_eig16h_r02h.summary.txt 2>&1
cat $OUT/prof_eig16h_r02h.summary.txt
