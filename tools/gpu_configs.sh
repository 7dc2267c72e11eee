mkdir -p gpurun_out/r1b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1b/build.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/r1b/configs.jsonl 2> gpurun_out/r1b/configs.err; echo "configs rc=$?"
cat gpurun_out/r1b/configs.jsonl; tail -5 gpurun_out/r1b/configs.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k3_f32" -c 1 -o gpurun_out/r1b/k3f32 python tools/bench_configs.py --configs 5 --steps 1 --warmup 0 > gpurun_out/r1b/ncu_k3.log 2>&1; echo "ncu k3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k3_f64" -c 1 -o gpurun_out/r1b/k3f64 python tools/bench_configs.py --configs 5 --steps 1 --warmup 0 > gpurun_out/r1b/ncu_k3d.log 2>&1; echo "ncu k3d rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k2_block" -c 1 -o gpurun_out/r1b/k2block python tools/bench_configs.py --configs 3 --steps 1 --warmup 0 > gpurun_out/r1b/ncu_k2b.log 2>&1; echo "ncu k2b rc=$?"
