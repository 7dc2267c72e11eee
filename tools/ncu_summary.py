"""Summaries of ncu outputs for profiles/ (diagnostics, not product code).

  python tools/ncu_summary.py launches LAUNCHES.csv      # per-kernel share of a --metrics gpu__time_duration run
  python tools/ncu_summary.py full REPORT.ncu-rep         # key --set full metrics of each captured launch
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = re.compile(
    r"^(Kernel Name|Grid Size|Block Size|gpu__time_duration.sum|dram__bytes_(read|write).sum|"
    r"dram__throughput.avg.pct_of_peak_sustained_elapsed|sm__throughput.avg.pct_of_peak_sustained_elapsed|"
    r"gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed|lts__t_sector_hit_rate.pct|"
    r"l1tex__data_pipe_lsu_wavefronts_mem_shared(_op_atom|_op_ld|_op_st)?.sum|"
    r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared(_op_atom)?.sum|"
    r"sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread|"
    r"launch__occupancy_limit_(registers|shared_mem|warps)|launch__waves_per_multiprocessor|"
    r"smsp__issue_active.avg.pct_of_peak_sustained_active|smsp__inst_executed.sum|"
    r"sm__inst_executed_pipe_(alu|fma|fmaheavy|fp64|xu|lsu|uniform)\.avg\.pct_of_peak_sustained_active|"
    r"sm__pipe_(alu|fma|fmaheavy|fmalite|fp64|shared|xu)_cycles_active.avg.pct_of_peak_sustained_active|"
    r"sm__cycles_elapsed.avg.per_second|smsp__sass_thread_inst_executed_op_(fadd|fmul|ffma|dadd|dmul|dfma)_pred_on.sum)$")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[re.sub(r"\(.*", "", r[ki])[:90]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':90s} {'launches':>8s} {'mean_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:90s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:6.3f}")
    print(f"total {tot / 1e3:.1f} us over {sum(len(v) for v in agg.values())} launches")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        print("-" * 100)
        for i, k in enumerate(h):
            if KEYS.match(k) and r[i] not in ("",):
                print(f"{k:80s} {r[i]} {u[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
