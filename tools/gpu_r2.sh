# Round-2 GPU evidence pass (run under gpurun): GPU tests, smoke, bench.
#   bash tools/gpu_r2.sh TAG [pytest -k expr]
TAG=${1:-r2}; K=${2:-}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x -k "$K" --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -30 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
