# one ncu --set full capture: bash tools/gpu_prof_one.sh TAG REGEX SKIP CMD...
TAG=$1; RX=$2; SK=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SK -c 1 -o $OUT/rep "$@" > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full $OUT/rep.ncu-rep > $OUT/full.txt 2>&1
python tools/ncu_source.py $OUT/rep.ncu-rep ${NLINES:-25} > $OUT/source.txt 2>&1
[ $(stat -c %s $OUT/rep.ncu-rep) -gt 30000000 ] && rm -f $OUT/rep.ncu-rep
head -3 $OUT/source.txt
