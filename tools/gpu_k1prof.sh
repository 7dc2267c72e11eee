# K1 check + profile on config 4 (GPU): K1 parity tests, launch list with
# instruction counts, --set full of the count pass. bash tools/gpu_k1prof.sh TAG
TAG=${1:-k1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "k1 or critical or config1 or degenerate or random_parity or counts" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
python tools/run_config.py config4 2 > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/run_config.py config4 2 > $OUT/ncu1.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_pencil -s 1 -c 1 -o $OUT/k1 python tools/run_config.py config4 2 > $OUT/ncu2.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py full $OUT/k1.ncu-rep > $OUT/k1.full.txt 2>&1
python tools/ncu_source.py $OUT/k1.ncu-rep 30 > $OUT/k1.source.txt 2>&1
rm -f $OUT/*.ncu-rep
