# A/B: GPU parity tests (default path), then config-2 stage times and bench.py
# with an environment switch off/on. Usage: bash tools/gpu_ab.sh TAG VAR [tests-filter]
TAG=${1:-ab}; VAR=${2:-EUCALC_K2_FUSED}; FILT=${3:-"tests/test_gpu_parity.py"}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest $FILT -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
for v in 0 1; do
  env $VAR=$v timeout 600 python tools/bench_configs.py --configs ${CONFIGS:-2} --steps 10 > $OUT/configs_$v.jsonl 2> $OUT/configs_$v.err; echo "configs $VAR=$v rc=$?"
  grep k2_transforms $OUT/configs_$v.jsonl | python -c "import sys,json; [print(json.loads(l)['config'], json.loads(l)['variant'], round(json.loads(l)['ms'],4)) for l in sys.stdin]"
  env $VAR=$v timeout 600 python bench.py --steps 30 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err; echo "bench $VAR=$v rc=$?"
  python -c "import json; d=json.load(open('$OUT/bench_$v.json')); print('bench', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['launch_ms'])"
done
