"""Summarise an ncu source page per CUDA source line (instructions executed, stall samples).
usage: python tools/ncu_source.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
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
    elif hdr and r and r[0] not in ("", "File Path") and len(r) > 8:
        try:
            res.append((fn, int(r[0]), r[1].strip()[:80], int(r[hdr["Instructions Executed"]] or 0),
                        int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, KeyError):
            pass
fns = sorted({x[0] for x in res})
for f in fns:
    sel = [x for x in res if x[0] == f]
    ti = sum(x[3] for x in sel); ts = sum(x[4] for x in sel)
    print(f"== {f[:110]}\n   total inst {ti}  samples {ts}")
    for x in sorted(sel, key=lambda x: -x[4])[:top]:
        print(f"  L{x[1]:<5} inst {x[3]:>11} {100*x[3]/max(ti,1):5.1f}%  samp {x[4]:>7} {100*x[4]/max(ts,1):5.1f}%  {x[2]}")
if len(sys.argv) > 3:
    for f in fns:
        sel = [x for x in res if x[0] == f]
        ti = sum(x[3] for x in sel)
        print(f"== by instructions: {f[:80]}")
        for x in sorted(sel, key=lambda x: -x[3])[:top]:
            print(f"  L{x[1]:<5} inst {x[3]:>11} {100*x[3]/max(ti,1):5.1f}%  {x[2]}")
