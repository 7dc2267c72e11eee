# Development timing with libeucalc_dev.so (built here; no build on the box): bash tools/gpu_dev.sh TAG "configs"
TAG=${1:-dev}; C=${2:-3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
EUCALC_LIB=dev python tools/bench_configs.py --configs $C > $OUT/stages.jsonl 2> $OUT/stages.err; tail -3 $OUT/stages.err
python - $OUT/stages.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(d.get("config"), d.get("variant"), d.get("stage"), round(d.get("ms",0),4), round(d.get("hbm_frac",0) or 0,3))
PY
