# ubench + selected GPU tests + full bench (run under gpurun).  bash tools/gpu_s7b.sh TAG "pytest -k"
TAG=${1:-s7b}; K=${2:-block_regime or config4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
./tools/ubench/atoms > $OUT/atoms.jsonl 2>&1; cat $OUT/atoms.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench rc=$?
python - $OUT/bench.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); c=d.pop("configs",{})
print("headline", d["value"], d["ms_per_step"], d["stages_ms_per_step"], d["roofline"]["frac"], d["roofline"].get("smem_atomics"), d["e2e"]["value"], d["clocks"])
for k,v in c.items(): print(k, v.get("value"), v.get("ms_per_step"), v.get("stages_ms_per_step"))
PY
