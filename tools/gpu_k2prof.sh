# ncu --set full (+ source) of one k2_block launch of the config-4 bench step (run under gpurun).
#   bash tools/gpu_k2prof.sh TAG [config4|config3]
TAG=${1:-k2p}; C=${2:-config4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python tools/run_config.py $C 2 > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_block -s 1 -c 1 -o $OUT/k2block_$C python tools/run_config.py $C 2 > $OUT/ncu_full.log 2>&1
echo "full k2_block rc=$?"
python tools/ncu_summary.py full $OUT/k2block_$C.ncu-rep > $OUT/k2block_$C.full.txt 2>&1
python tools/ncu_source.py $OUT/k2block_$C.ncu-rep 40 > $OUT/k2block_$C.source.txt 2>&1
rm -f $OUT/*.ncu-rep
head -40 $OUT/k2block_$C.full.txt
