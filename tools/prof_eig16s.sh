OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eig16s -s 1 -c 1 -o $OUT/prof_eig16s_r02i python tools/eig_once.py 1 > $OUT/prof_eig16s_r02i.log 2>&1
python tools/ncu_summary.py $OUT/prof_eig16s_r02i.ncu-rep > $OUT/prof_eig16s_r02i.summary.txt 2>&1
cat $OUT/prof_eig16s_r02i.summary.txt
