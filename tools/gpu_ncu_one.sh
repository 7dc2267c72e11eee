# ncu --set full of one kernel (regex $2) in command $3.. ; summaries under gpurun_out/$1
TAG=$1; K=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${SKIP:-1} -c 1 -o $OUT/$K "$@" > $OUT/ncu_$K.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full $OUT/$K.ncu-rep > $OUT/$K.full.txt 2>&1
python tools/ncu_source.py $OUT/$K.ncu-rep 40 > $OUT/$K.source.txt 2>&1
rm -f $OUT/$K.ncu-rep
grep -E "Grid|time_duration|inst_executed.sum|issue_active|warps_active|registers_per" $OUT/$K.full.txt
head -30 $OUT/$K.source.txt
