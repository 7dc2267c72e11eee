# Evidence run: GPU tests, smoke, bench (+ reference arm), ncu launch list of the
# bench command, K2 traffic, ncu --set full of the top kernel, all-config stage
# times and the f4 experiments. Usage: bash tools/gpu_final.sh TAG
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cat $OUT/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.txt 2>&1
timeout 900 python tools/traffic.py $OUT > $OUT/traffic.log 2>&1; echo "traffic rc=$?"; cat $OUT/traffic.log
ITERS=2 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k2w_emit" -s 1 -c 1 -o $OUT/top python tools/run_config2_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py full $OUT/top.ncu-rep > $OUT/top.full.txt 2>&1
python tools/ncu_source.py $OUT/top.ncu-rep 30 > $OUT/top.source.txt 2>&1
rm -f $OUT/top.ncu-rep
timeout 1200 python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?"
timeout 900 python tools/experiments.py > $OUT/experiments.jsonl 2> $OUT/experiments.err; echo "experiments rc=$?"
du -sh $OUT
