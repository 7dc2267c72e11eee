# ncu --set full of K1 on config 4 (3-D) and config 5, summaries + source hot lines. usage: bash tools/gpu_k1_ncu.sh TAG
TAG=${1:-k1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for c in 4 5; do
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k1_kernel" -s 1 -c 1 -o $OUT/k1_c$c python tools/bench_configs.py --configs $c --steps 1 --warmup 1 > $OUT/ncu_k1_c$c.log 2>&1; echo "ncu k1 c$c rc=$?"
python tools/ncu_summary.py full $OUT/k1_c$c.ncu-rep > $OUT/k1_c$c.full.txt 2>&1
python tools/ncu_source.py $OUT/k1_c$c.ncu-rep 30 > $OUT/k1_c$c.source.txt 2>&1
rm -f $OUT/k1_c$c.ncu-rep
done
