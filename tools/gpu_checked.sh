# Device bounds checks (T8 stand-in: compute-sanitizer is refused on the GPU pool):
# the whole GPU test suite against libeucalc_checked.so (EU_DCHECK compiled in),
# plus a self-test that an injected out-of-range output capacity traps.
#   bash tools/gpu_checked.sh TAG
TAG=${1:-chk}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "from paper_2405_02256_b200 import _build; _build.build(); _build.build(checked=True)" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
EUCALC_LIB=checked timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_checked.log 2>&1; echo "checked pytest rc=$?"; tail -3 $OUT/pytest_gpu_checked.log
EUCALC_LIB=checked timeout 300 python - > $OUT/selftest.log 2>&1 <<'PY'
import os, sys
sys.path.insert(0, ".")
import numpy as np, synth, paper_2405_02256_b200 as eu
print("library:", eu.LIB_PATH)
imgs = synth.blob_images(4, 28, 1)
dirs = synth.random_directions(8, 2, 16, 2)
cr = eu.critical_points(eu.build_complex(imgs, "vertex"))
eu.transforms(cr, dirs)  # clean run
import torch; torch.cuda.synchronize()
print("clean run ok")
os.environ["EUCALC_DCHECK_INJECT"] = "1"
try:
    eu.transforms(cr, dirs); torch.cuda.synchronize()
    print("SELFTEST FAILED: no trap")
except Exception as e:
    print("injected out-of-range position trapped as expected:", type(e).__name__, str(e)[:200])
PY
echo "selftest rc=$?"; cat $OUT/selftest.log | grep -v "^$" | tail -6
