# ncu --set full captures of the current top kernels; summaries written as text on the box,
# reports > 12 MB dropped (gpurun brings back <= 64 MiB)
OUT=gpurun_out/${1:-prof2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
summ() { python tools/ncu_summary.py full $1.ncu-rep > $1.full.txt 2>&1; python tools/ncu_source.py $1.ncu-rep 30 > $1.source.txt 2>&1;
         [ $(stat -c %s $1.ncu-rep) -gt 12000000 ] && rm -f $1.ncu-rep; }
ITERS=2 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2w_count|k2w_emit|k3t|k1_kernel" -s 4 -c 5 -o $OUT/c2 python tools/run_config2_once.py > $OUT/ncu_c2.log 2>&1; echo "c2 rc=$?"; summ $OUT/c2
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2_block" -s 1 -c 1 -o $OUT/c3 python tools/bench_configs.py --configs 3 --steps 1 --warmup 1 > $OUT/ncu_c3.log 2>&1; echo "c3 rc=$?"; summ $OUT/c3
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2_block|k1_kernel" -s 2 -c 2 -o $OUT/c4 python tools/bench_configs.py --configs 4 --steps 1 --warmup 1 > $OUT/ncu_c4.log 2>&1; echo "c4 rc=$?"; summ $OUT/c4
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k3t" -s 1 -c 2 -o $OUT/c5 python tools/bench_configs.py --configs 5 --steps 1 --warmup 0 > $OUT/ncu_c5.log 2>&1; echo "c5 rc=$?"; summ $OUT/c5
du -sh $OUT
