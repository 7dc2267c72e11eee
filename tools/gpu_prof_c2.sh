OUT=gpurun_out/${1:-c2gray}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2w_count|k2w_emit" -s 0 -c 2 -o $OUT/rep python tools/run_config2_once.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full $OUT/rep.ncu-rep > $OUT/full.txt 2>&1
python tools/ncu_source.py $OUT/rep.ncu-rep 30 > $OUT/source.txt 2>&1
rm -f $OUT/rep.ncu-rep
