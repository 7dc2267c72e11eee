python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do python bench.py --steps ${STEPS:-100} --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,1), d['e2e']['step_ms_spread'])"; done
