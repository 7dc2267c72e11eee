# bench.py repeatability (diagnostics): N runs, per-run mean and step spread
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in $(seq ${RUNS:-6}); do
  python bench.py --steps ${STEPS:-100} --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['step_ms_spread'], round(d['roofline']['launch_ms'],4))"
done
