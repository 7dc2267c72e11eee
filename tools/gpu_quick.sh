# Quick GPU iteration (run under gpurun): build check, selected GPU tests, stage timings.
#   bash tools/gpu_quick.sh TAG "pytest -k expr" "bench_configs args"
TAG=${1:-q}; K=${2:-}; BC=${3:---configs 4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
fi
timeout 900 python tools/bench_configs.py $BC > $OUT/stages.jsonl 2> $OUT/stages.err; echo "stages rc=$?"
python - $OUT/stages.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(d.get("config"), d.get("variant"), d.get("stage"), round(d.get("ms",0),4), round(d.get("hbm_frac",0) or 0,3))
PY
