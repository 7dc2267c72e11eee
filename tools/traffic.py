"""DRAM traffic of the bench's dominant stage (K2: k2w_count + k2_scan + k2w_emit,
fused HT) from an ncu capture of tools/run_config2_once.py: the launches of the
second iteration (one bench step) -> profiles/<round>/k2_traffic.json.
Run on the GPU box:  python tools/traffic.py profiles/r1"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r1")
cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--clock-control",
       "none", "-k", "regex:k2w_|k2_scan|k3_table", "--csv", sys.executable,
       os.path.join(ROOT, "tools", "run_config2_once.py")]
r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, ITERS="2"))
rows = [x for x in csv.reader(io.StringIO(r.stdout)) if len(x) > 10]
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
launch = {}
for x in rows[1:]:
    v = float(x[vi].replace(",", "")) * scale.get(x[ui], 1)
    launch.setdefault(int(x[ii]), {"kernel": x[ki].split("(")[0]})[x[mi]] = v
ids = sorted(launch)
half = ids[len(ids) // 2:]  # second iteration (warm)
tot = sum(launch[i]["dram__bytes_read.sum"] + launch[i]["dram__bytes_write.sum"] for i in half)
res = {"stage": "k2_transforms (k2w_count + k2_scan + k2w_emit + k3_table, fused HT)",
       "dram_bytes_per_step": tot, "launches_per_step": len(half),
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/traffic.py), "
                 "second iteration (one bench step) of tools/run_config2_once.py",
       "per_kernel": [{k: launch[i][k] for k in launch[i]} for i in half]}
os.makedirs(out_dir, exist_ok=True)
json.dump(res, open(os.path.join(out_dir, "k2_traffic.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "per_kernel"}))
