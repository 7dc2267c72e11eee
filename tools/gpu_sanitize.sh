# compute-sanitizer over tools/sanitize_run.py (run under gpurun).  bash tools/gpu_sanitize.sh TAG [tools]
TAG=${1:-san}; TOOLS=${2:-memcheck racecheck synccheck}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for t in $TOOLS; do
  extra=""; [ $t = memcheck ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $t $extra --print-limit 50 --target-processes all python tools/sanitize_run.py > $OUT/$t.log 2>&1
  echo "$t rc=$?"; tail -3 $OUT/$t.log
done
