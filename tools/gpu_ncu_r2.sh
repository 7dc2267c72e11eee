# ncu evidence for the round-2 bench records (run under gpurun, one GPU):
#   launch list of the headline bench command, DRAM traffic of each record's K2,
#   k3t shared-memory wavefronts / pipe counters (config 5), --set full of the
#   headline's top kernel. Every command runs once without ncu first.
#   bash tools/gpu_ncu_r2.sh TAG
TAG=${1:-ncu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
B="python bench.py --steps 2 --warmup 3 --headline-only --no-cpu-baseline"
$B > $OUT/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?"
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.txt 2>&1; head -20 $OUT/launches.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in config4 config2 config2_fused_ht config3; do
  python tools/run_config.py $c 2 > $OUT/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/traffic_$c.csv python tools/run_config.py $c 2 > $OUT/ncu_traffic_$c.log 2>&1
  echo "traffic $c rc=$?"
done
M5=l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,sm__inst_executed_pipe_lsu.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for kp in "gauss f32" "gauss f64" "cos f32" "cos f64"; do
  set -- $kp
  python tools/run_config.py config5 1 $1 $2 > $OUT/plain_c5_$1_$2.log 2>&1 && \
  timeout 900 ncu --metrics $M5 --clock-control none -k regex:k3t --csv --log-file $OUT/k3t_$1_$2.csv python tools/run_config.py config5 1 $1 $2 > $OUT/ncu_k3t_$1_$2.log 2>&1
  echo "k3t $1 $2 rc=$?"
done
python tools/run_config.py config4 2 > $OUT/plain_c4b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_unit -s 2 -c 1 -o $OUT/k2unit_c4 python tools/run_config.py config4 2 > $OUT/ncu_full_c4.log 2>&1
echo "full k2_unit rc=$?"
python tools/ncu_summary.py full $OUT/k2unit_c4.ncu-rep > $OUT/k2unit_c4.full.txt 2>&1
python tools/ncu_source.py $OUT/k2unit_c4.ncu-rep 30 > $OUT/k2unit_c4.source.txt 2>&1
python tools/run_config.py config5 1 cos f32 > $OUT/plain_c5full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3t -c 1 -o $OUT/k3t_c5 python tools/run_config.py config5 1 cos f32 > $OUT/ncu_full_c5.log 2>&1
echo "full k3t rc=$?"
python tools/ncu_summary.py full $OUT/k3t_c5.ncu-rep > $OUT/k3t_c5.full.txt 2>&1
python tools/ncu_source.py $OUT/k3t_c5.ncu-rep 30 > $OUT/k3t_c5.source.txt 2>&1
rm -f $OUT/*.ncu-rep
du -sh $OUT
python tools/ncu_records.py $OUT $OUT/records > $OUT/records.log 2>&1; cat $OUT/records.log | head -30
