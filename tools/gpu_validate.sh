# Validation run (under gpurun): ubenches, whole GPU suite, smoke, full bench. bash tools/gpu_validate.sh TAG
TAG=${1:-s8}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
./tools/ubench/dsmem_atoms > $OUT/dsmem_atoms.jsonl 2>&1; cat $OUT/dsmem_atoms.jsonl
./tools/ubench/atoms > $OUT/atoms.jsonl 2>&1; cat $OUT/atoms.jsonl
( time timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1 ) 2> $OUT/pytest_time.txt; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log; cat $OUT/pytest_time.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
( time timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err ) 2> $OUT/bench_time.txt; echo bench rc=$?; cat $OUT/bench_time.txt
python - $OUT/bench.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); c=d.pop("configs",{})
print("headline", d["value"], d["ms_per_step"], d["stages_ms_per_step"], d["roofline"]["frac"], d["roofline"].get("smem_atomics"), d["e2e"]["value"], d["clocks"])
for k,v in c.items(): print(k, v.get("value"), v.get("ms_per_step"), v.get("stages_ms_per_step"))
PY
