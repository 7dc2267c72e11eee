# Per-kernel launch lists of the bench configs' steps + host/device timeline (run under gpurun).
#   bash tools/gpu_launches.sh TAG "config4 config2 config3"
TAG=${1:-ll}; CFGS=${2:-config4 config2 config3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for c in $CFGS; do
  EUCALC_HOST_TRACE=1 timeout 300 python tools/host_trace.py $c 5 > $OUT/host_$c.txt 2>&1; echo "host $c rc=$?"; cat $OUT/host_$c.txt | tail -3
done
for c in $CFGS; do
  python tools/run_config.py $c 2 > $OUT/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/run_config.py $c 2 > $OUT/ncu_$c.log 2>&1
  echo "launches $c rc=$?"
  python tools/ncu_summary.py launches $OUT/launches_$c.csv > $OUT/launches_$c.txt 2>&1; head -14 $OUT/launches_$c.txt
done
