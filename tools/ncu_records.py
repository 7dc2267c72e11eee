"""Turns the ncu CSVs of tools/gpu_ncu_r2.sh into the JSON files bench.py reads:

  profiles/<round>/traffic.json      per record: DRAM bytes (read + write) of the
                                     step's K2 launches (second step of
                                     tools/run_config.py = one bench step)
  profiles/<round>/k3t_counters.json per (kernel, precision): shared-memory
                                     wavefronts and pipe counters of one k3t launch

  python tools/ncu_records.py gpurun_out/TAG profiles/r2
"""
import csv
import json
import os
import re
import sys


def rows(path):
    lines = [l for l in open(path) if l.startswith('"')]
    return list(csv.DictReader(lines))


def per_launch(path):
    """{launch id: {"kernel": name, metric: value}} in launch order."""
    out = {}
    for r in rows(path):
        d = out.setdefault(int(r["ID"]), {"kernel": re.sub(r"\(.*", "", r["Kernel Name"])})
        try:
            d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    return [out[k] for k in sorted(out)]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    traffic = {}
    for c in ("config4", "config2", "config3"):
        p = os.path.join(src, f"traffic_{c}.csv")
        if not os.path.exists(p):
            continue
        ls = per_launch(p)
        k2 = [l for l in ls if "k2" in l["kernel"]]
        half = len(k2) // 2  # two steps were run: keep the second
        step = k2[half:] if half else k2
        traffic[c] = {
            "dram_bytes_per_step": sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
                                       for l in step),
            "launches": [{"kernel": l["kernel"], "dram_read": l.get("dram__bytes_read.sum"),
                          "dram_write": l.get("dram__bytes_write.sum"), "ns": l.get("gpu__time_duration.sum")}
                         for l in step],
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/gpu_ncu_r2.sh, {src}): "
                      f"K2 launches of the second step of tools/run_config.py {c}",
        }
    json.dump(traffic, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
    k3 = {}
    for kern in ("gauss", "cos"):
        for prec in ("f32", "f64"):
            p = os.path.join(src, f"k3t_{kern}_{prec}.csv")
            if not os.path.exists(p):
                continue
            ls = per_launch(p)
            if not ls:
                continue
            l = ls[-1]
            k3[f"{kern}_{prec}"] = {
                "kernel": l["kernel"],
                "lsu_wavefronts_shared_per_launch": l.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                "lsu_wavefronts_shared_ld": l.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
                "inst_lsu": l.get("sm__inst_executed_pipe_lsu.sum"),
                "inst_xu": l.get("sm__inst_executed_pipe_xu.sum"),
                "inst_total": l.get("smsp__inst_executed.sum"),
                "fma_pipe_pct": l.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                "alu_pipe_pct": l.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": l.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "shared_pipe_pct": l.get("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
                "ncu_ns": l.get("gpu__time_duration.sum"),
                "source": f"ncu --metrics (tools/gpu_ncu_r2.sh, {src}): one k3t launch of config 5, "
                          f"tools/run_config.py config5 1 {kern} {prec}",
            }
    json.dump(k3, open(os.path.join(dst, "k3t_counters.json"), "w"), indent=1)
    print(json.dumps({"traffic": {k: v["dram_bytes_per_step"] for k, v in traffic.items()},
                      "k3t": {k: {kk: v[kk] for kk in ("lsu_wavefronts_shared_per_launch", "ncu_ns", "fma_pipe_pct",
                                                       "alu_pipe_pct", "fp64_pipe_pct")} for k, v in k3.items()}},
                     indent=1))


if __name__ == "__main__":
    main()
