OUT=gpurun_out/k1a; mkdir -p $OUT
./tools/ubench/atoms > $OUT/atoms.jsonl 2>&1; cat $OUT/atoms.jsonl
bash tools/gpu_quick.sh k1a "k1 or config4 or config5_sampled or degenerate or config2_small" "--configs 4,5 --steps 5"
