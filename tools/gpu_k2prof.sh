# ncu --set full (+ source) of one launch of a kernel of a config's bench step, plus
# the step's launch list (run under gpurun).  bash tools/gpu_k2prof.sh TAG [config4] [regex:k2_unit]
TAG=${1:-k2p}; C=${2:-config4}; K=${3:-regex:k2_unit}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python tools/run_config.py $C 2 > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$C.csv python tools/run_config.py $C 2 > $OUT/ncu_l.log 2>&1
python tools/ncu_summary.py launches $OUT/launches_$C.csv > $OUT/launches_$C.txt 2>&1; head -12 $OUT/launches_$C.txt
timeout 900 ncu --set full --clock-control none --import-source on -k $K -s ${SKIP:-1} -c 1 -o $OUT/full_$C python tools/run_config.py $C 2 > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py full $OUT/full_$C.ncu-rep > $OUT/full_$C.txt 2>&1
python tools/ncu_source.py $OUT/full_$C.ncu-rep 40 > $OUT/source_$C.txt 2>&1
rm -f $OUT/*.ncu-rep
head -40 $OUT/full_$C.txt
