# tests + bench + per-config stage timings (no profiler). usage: bash tools/gpu_check.sh TAG [CONFIGS]
TAG=${1:-check}; CFG=${2:-1,2,3,4,5}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err
timeout 900 python tools/bench_configs.py --configs $CFG > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?"
python - <<'PY' "$OUT/configs.jsonl"
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d["config"], d["variant"], d["stage"], round(d["ms"],3), "ms", {k:round(v,3) if isinstance(v,float) else v for k,v in d.items() if k in ("gbs","hbm_frac","image_directions_per_s","terms_per_s")})
PY
tail -3 $OUT/configs.err
