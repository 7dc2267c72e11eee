python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/host_trace_calls.py
OUT=gpurun_out/p3; mkdir -p $OUT
for K in k2w_count k2w_emit; do
ITERS=2 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 2 -c 1 -o $OUT/$K python tools/run_config2_once.py > $OUT/ncu_$K.log 2>&1
python tools/ncu_summary.py full $OUT/$K.ncu-rep > $OUT/$K.full.txt 2>&1
python tools/ncu_source.py $OUT/$K.ncu-rep 40 > $OUT/$K.source.txt 2>&1
rm -f $OUT/$K.ncu-rep
done
