# Session-7 baseline (run under gpurun): GPU tests + smoke + bench on HEAD, then
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py.
#   bash tools/gpu_s7.sh TAG
TAG=${1:-s7}
bash tools/gpu_r2.sh $TAG
OUT=gpurun_out/$TAG
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench rc=$?
tail -c 400 $OUT/bench.json
python tools/sanitize_run.py > $OUT/sanitize_plain.log 2>&1; echo "sanitize plain rc=$?"
bash tools/gpu_sanitize.sh $TAG/san
