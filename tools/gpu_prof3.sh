OUT=gpurun_out/prof3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
one() { tag=$1; rx=$2; sk=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c 1 -o $OUT/$tag "$@" > $OUT/ncu_$tag.log 2>&1; echo "$tag rc=$?"
  python tools/ncu_summary.py full $OUT/$tag.ncu-rep > $OUT/$tag.full.txt 2>&1
  python tools/ncu_source.py $OUT/$tag.ncu-rep 25 > $OUT/$tag.source.txt 2>&1
  rm -f $OUT/$tag.ncu-rep; }
#one k3t_f32 k3t 4 python tools/bench_configs.py --configs 5 --steps 1 --warmup 0
one k1_c4 k1_kernel 1 python tools/bench_configs.py --configs 4 --steps 1 --warmup 1
