bash tools/gpu_r2.sh base
timeout 900 python bench.py > gpurun_out/base/bench.json 2> gpurun_out/base/bench.err; echo bench rc=$?
tail -c 600 gpurun_out/base/bench.json
