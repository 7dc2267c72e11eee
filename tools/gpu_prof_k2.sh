# ncu --set full of K2's block kernel on configs 4 and 3 (run under gpurun; each
# command runs once without ncu first).   bash tools/gpu_prof_k2.sh TAG
TAG=${1:-pk2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in config4 config3; do
  python tools/run_config.py $c 2 > $OUT/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_block -s 1 -c 1 -o $OUT/k2block_$c python tools/run_config.py $c 2 > $OUT/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
  python tools/ncu_summary.py full $OUT/k2block_$c.ncu-rep > $OUT/k2block_$c.full.txt 2>&1
  python tools/ncu_source.py $OUT/k2block_$c.ncu-rep 30 > $OUT/k2block_$c.source.txt 2>&1
done
rm -f $OUT/*.ncu-rep
