#!/bin/bash
# One gpurun session: GPU tests, bench (no profiler), ncu launch list, one full
# ncu capture of the top kernel. Diagnostics, not product code.
#   gpurun --timeout 1500 -- 'bash tools/gpu_session.sh TAG [KREGEX]'
set -u
TAG=${1:-run}
KREGEX=${2:-k2w_emit}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo BUILD FAILED; tail -30 "$OUT/build.log"; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  tail -5 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
  tail -2 "$OUT/smoke.log"
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"
cat "$OUT/bench.json"
tail -3 "$OUT/bench.err"
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s 2 -c 1 \
    -o "$OUT/top" python tools/run_config2_once.py > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?"
fi
