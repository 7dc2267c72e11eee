# ncu captures of K1 on configs 2 (2-D batch), 3 (2-D large), 4 (3-D) + host timing of the bench step
mkdir -p gpurun_out/r1c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1c/build.log 2>&1
timeout 300 python tools/host_profile.py > gpurun_out/r1c/host_profile.txt 2>&1; echo "host rc=$?"
cat gpurun_out/r1c/host_profile.txt
for c in 2 3 4; do
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k1_kernel" -s 1 -c 1 -o gpurun_out/r1c/k1_c$c python tools/bench_configs.py --configs $c --steps 1 --warmup 1 > gpurun_out/r1c/ncu_k1_c$c.log 2>&1; echo "ncu k1 c$c rc=$?"
done
