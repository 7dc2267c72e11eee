"""Summarise an ncu source page per CUDA source line: instructions executed,
stall samples and the dominant stall reasons.
usage: python tools/ncu_source.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, hdr, fn = [], None, ""
for r in rows:
    if r and r[0] == "Function Name":
        fn = r[1]
    elif r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        stall_cols = [(h, i) for h, i in hdr.items() if h.startswith("stall_") and "Not Issued" not in h]
    elif hdr and r and r[0] not in ("", "File Path") and len(r) > 8:
        try:
            stalls = {h[6:]: int(r[i] or 0) for h, i in stall_cols if i < len(r) and (r[i] or "0").isdigit()}
            res.append((fn, int(r[0]), r[1].strip()[:70], int(r[hdr["Instructions Executed"]] or 0),
                        int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0), stalls))
        except (ValueError, KeyError):
            pass
fns = sorted({x[0] for x in res})
for f in fns:
    sel = [x for x in res if x[0] == f]
    ti = sum(x[3] for x in sel)
    ts = sum(x[4] for x in sel)
    tot = {}
    for x in sel:
        for k, v in x[5].items():
            tot[k] = tot.get(k, 0) + v
    reasons = ", ".join(f"{k} {100 * v / max(ts, 1):.0f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:6])
    print(f"== {f[:110]}\n   total inst {ti}  samples {ts}  stalls: {reasons}")
    for x in sorted(sel, key=lambda x: -x[4])[:top]:
        st = ", ".join(f"{k} {v}" for k, v in sorted(x[5].items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"  L{x[1]:<5} inst {x[3]:>11} {100 * x[3] / max(ti, 1):5.1f}%  samp {x[4]:>7} "
              f"{100 * x[4] / max(ts, 1):5.1f}%  {x[2]}  [{st}]")
