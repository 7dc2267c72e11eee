# bench.py repeatability (diagnostics): RUNS runs per setting of $VAR (default BENCH_NO_GC)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
VAR=${VAR:-BENCH_NO_GC}
for i in $(seq ${RUNS:-3}); do for v in 0 1; do
  env $VAR=$v python bench.py --steps ${STEPS:-100} --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['ms_per_step'],4), {k: round(x, 3) for k, x in d['step_ms_spread'].items()}, round(d['roofline']['launch_ms'],4), round(d['e2e']['value']/1e6,1))"
done; done
