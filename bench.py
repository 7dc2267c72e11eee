"""Benchmark of the hot path on BASELINE.json config 2.

One step = build (A0) + critical points (A1-A2) + exact ECT and Radon (A3-A5)
+ hybrid transform (A6, kappa = sin as in the paper's experiments P:140, fp64;
computed from K2's merged histogram, eucalc_transforms_ht = NEXT row f2)
for a batch of 1024 synthetic 28x28 u8 blob images AND its binarised variant
(BJ:8), vertex construction, 256 integer directions in [-16,16]^2.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0). Multi-GPU (torchrun): every rank processes its
own shard of the global batch (independent images, no data-path collective):
weak scaling; time = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "exact ECT/Radon directions/s per image and HT GFLOP/s; % of HBM/FP32 roofline"
UNIT = "image-directions/s"
IMAGES_PER_SHARD = 1024
NDIRS = 256
HT_KERNEL = "sin"


def shard_range(n_units: int, rank: int, world: int):
    """Contiguous [start, stop) of n_units for this rank."""
    per = (n_units + world - 1) // world
    a = min(n_units, rank * per)
    return a, min(n_units, a + per)


def workload(rank: int):
    import synth

    seed = synth.IMAGE_SEED[2] + 7919 * rank  # shard 0 == config 2 exactly
    gray = synth.blob_images(IMAGES_PER_SHARD, 28, seed)
    binary = synth.binarize(gray, 128)
    dirs = synth.random_directions(NDIRS, 2, 16, synth.DIR_SEED[2])
    return gray, binary, dirs


def step_batches(gray, binary):
    """The step's input batches: the 1024 gray images and their binary variant as
    ONE batch of 2048 images (one build, one K1 launch, one K2 call; the library
    is batched, and the two variants share shape and directions)."""
    return [np.concatenate([gray, binary])]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """Samples nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        return self.start()

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        if os.environ.get("BENCH_NO_CLOCKS") == "1":  # diagnostics: measure without the sampler
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "25"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def mark(self):
        """Only samples taken after this call count (the timed region starts)."""
        self.first = len(self.samples)

    def end(self):
        """The timed region ends (one more sample, in flight, still counts)."""
        self.last = len(self.samples) + 1

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        self.stop()

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        first = getattr(self, "first", 0)
        samples = self.samples[first:max(getattr(self, "last", len(self.samples)), first + 1)]
        self.samples = samples
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- GPU arm

_STREAMS = []


def run_step(eu, torch, imgs_dev, dirs, record=None):
    """One pass of the whole hot path over the step's batches (bench: one batch of
    gray + binary images, step_batches). Returns host-free results.

    Several batches go to CUDA streams forked from and joined back into the
    current stream, each batch's calls issued in full before the next's."""
    if len(imgs_dev) == 1:  # one batch: the current stream, no fork/join
        cx = eu.build_complex(imgs_dev[0], "vertex")
        cr = eu.critical_points(cx)
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(HT_KERNEL, 1.0, "f64"))
        return [(cx, cr, r, r["ht"])]
    cur = torch.cuda.current_stream()
    while len(_STREAMS) < len(imgs_dev):
        _STREAMS.append(torch.cuda.Stream())
    streams = _STREAMS[:len(imgs_dev)]
    for st in streams:
        st.wait_stream(cur)
    out = []
    for img, st in zip(imgs_dev, streams):
        with torch.cuda.stream(st):
            cx = eu.build_complex(img, "vertex", stream=st)
            cr = eu.critical_points(cx, stream=st)
            # ECT + Radon + HT in one pass over the merged histogram (eucalc_transforms_ht)
            r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(HT_KERNEL, 1.0, "f64"),
                              stream=st)
        out.append((cx, cr, r, r["ht"]))
    for st in streams:
        cur.wait_stream(st)
    return out


def run_step_e2e(eu, torch, imgs_host, dirs):
    """Same step through the C ABI with HOST buffers: pinned host images in,
    host (pinned) representations and HT out; returns (h2d, d2h) bytes."""
    h2d = d2h = 0
    cxs = [eu.build_complex(img, "vertex") for img in imgs_host]  # H2D inside the ABI
    crs = [eu.critical_points(cx) for cx in cxs]
    for img, cx, cr in zip(imgs_host, cxs, crs):
        h2d += img.numel() * img.element_size()
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, device="cpu",
                          ht=(HT_KERNEL, 1.0, "f64"))  # D2H inside the ABI
        ht = r.pop("ht")
        for k, st in r.items():
            n = int(st["offsets"][-1])
            eb = st["value"].element_size()
            d2h += st["offsets"].numel() * 8 + n * eb + (n * eb if (k != "classical") else 0)
        d2h += ht.numel() * 8
        h2d += dirs.nbytes
    return h2d, d2h


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2405_02256_b200 as eu

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    eu.lib()
    gray, binary, dirs = workload(rank)
    batches = step_batches(gray, binary)
    imgs_dev = [torch.from_numpy(x).cuda() for x in batches]
    imgs_host = [torch.from_numpy(x).pin_memory() for x in batches]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    s = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the clock sampler starts before the warm-up: nvidia-smi's start-up (NVML
    # initialisation) stalls the driver for milliseconds and must not fall in
    # the timed region
    clk = Clocks(local).start()
    time.sleep(0.5)
    for _ in range(args.warmup):
        run_step(eu, torch, imgs_dev, dirs)
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, L2 flushed between steps (untimed)
    times = []
    k2_ms = 0.0
    stage_ms = {}
    k2_span = 0.0  # wall span of the step's (concurrent) K2 launches
    launches = 0
    if True:
        # BENCH_NO_GC=1 (diagnostics): no Python garbage collection inside the timed steps
        gc_was = gc.isenabled()
        if os.environ.get("BENCH_NO_GC") == "1":
            gc.collect()
            gc.disable()
        barrier()
        clk.mark()
        for _ in range(args.steps):
            flush.fill_(1.0)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eu.profile_enable(True)
            eu.launch_count(reset=True)
            ev0.record(s)
            res = run_step(eu, torch, imgs_dev, dirs)
            ev1.record(s)
            launches += eu.launch_count()
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            for st in ("build", "k1_critical", "k2_transforms", "k3_hybrid"):
                stage_ms[st] = stage_ms.get(st, 0.0) + eu.profile_read(st)[0]
            k2_span += eu.profile_span("k2_transforms")
            eu.profile_enable(False)
        barrier()
        clk.end()
        if gc_was:
            gc.enable()
        clk.stop()
    dev_ms = float(np.sum(times))
    if world > 1:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    units = 2 * IMAGES_PER_SHARD * NDIRS * world * args.steps
    value = units / (dev_ms / 1e3)

    # ---- roofline of the dominant stage (K2, both variants' launches running
    # concurrently on their streams) from the last step's actual sizes: bytes of
    # both launches over the wall span from the first K2 start to the last K2 end
    k2_launch_ms = k2_span / args.steps
    k2_bytes = 0
    for cx, cr, r, ht in res:
        S = cx.batch * NDIRS
        ne = int(r["ect"]["offsets"][S])
        no = int(r["ordinary"]["offsets"][S])
        eb = r["ect"]["value"].element_size()
        lists = list_bytes(cr, dirs)
        # ECT (h,v) + ordinary (h,v) + classical (v; heights shared) + 3 offset arrays + HT (f64)
        k2_bytes += lists + ne * 2 * eb + no * 2 * eb + ne * eb + 3 * (S + 1) * 8 + S * 8
    peak, peak_src = peaks()
    achieved = k2_bytes / (k2_launch_ms / 1e3) / 1e9
    traffic = None  # measured DRAM bytes per K2 call, from the committed ncu capture (tools/traffic.py)
    tp = os.path.join(ROOT, "profiles", "r1", "k2_traffic.json")
    if os.path.exists(tp):  # both variants' K2 calls of one step, as the roofline's bytes
        tj = json.load(open(tp))
        traffic = tj.get("dram_bytes_per_step")

    # ---- e2e through the ABI with host buffers
    torch.cuda.synchronize()
    run_step_e2e(eu, torch, imgs_host, dirs)
    torch.cuda.synchronize()
    e2e_t = []
    h2d = d2h = 0
    barrier()
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        h2d, d2h = run_step_e2e(eu, torch, imgs_host, dirs)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    barrier()
    e2e_s = float(np.sum(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = 2 * IMAGES_PER_SHARD * NDIRS * world * len(e2e_t) / e2e_s

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int16 (ECT/Radon outputs), int32 (histogram), f64 (HT)",
            "data": "synthetic (seeded generators, synth/; config-2 recipe of SURVEY.md 8(d))",
            "config": arm_config(world),
            "stages_ms_per_step": {k: v / args.steps for k, v in stage_ms.items()},
            "step_ms_spread": {"min": float(np.min(times)), "median": float(np.median(times)),
                               "max": float(np.max(times))},
            "roofline": {"bound": "hbm", "kernel": "k2_transforms (k2w_count+k2_scan+k2w_emit, fused HT) over the "
                                                  "step's 2048-image batch (gray + binary)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": "profiles/r1/k2_traffic.json (ncu, the step's K2 call)",
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": k2_bytes,
                         "launch": "one step's K2 stage (2048 images)",
                         "launch_ms": k2_launch_ms},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "step_ms_spread": {"min": 1e3 * float(np.min(e2e_t)), "median": 1e3 * float(np.median(e2e_t)),
                                       "max": 1e3 * float(np.max(e2e_t))}},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def arm_config(world):
    return {
        "workload": "BASELINE.json configs[1]: 1024 x 28x28 u8 Gaussian-blob images + binary variant "
                    "(>=128), vertex construction, 256 integer directions in [-16,16]^2; "
                    "ECT + Radon (all three streams) + HT (kappa=sin, fp64) per image-direction "
                    "(HT fused into K2, eucalc_transforms_ht)",
        "images_per_gpu": 2 * IMAGES_PER_SHARD, "directions": NDIRS, "parallelism": f"dp{world}",
        "l2": "flushed between timed steps (256 MB write, untimed)",
        "output": "CSR, narrowest exact int width (int16 here), classical heights shared with ECT",
    }


def list_bytes(cr, dirs):
    """Algorithmic read bytes of K2: every record (8 B) of the direction's orthant
    pair list, once per (image, direction)."""
    lens = cr.list_lengths()  # [B, Q]
    n = dirs.shape[1]
    full = (1 << n) - 1
    e = ((dirs > 0).astype(np.int64) << np.arange(n)).sum(1)
    q = np.where((e >> (n - 1)) & 1, e ^ full, e)
    return int(lens[:, q].sum()) * 8


# ----------------------------------------------------------------------------- CPU oracle arm

def oracle_step(images_list, dirs, threads=None):
    import oracle

    n = 0
    for imgs in images_list:
        oracle.transforms_batch(imgs, dirs, "vertex", threads=threads)
        oracle.ht_batch(imgs, dirs, "vertex", HT_KERNEL, 1.0, threads=threads)
        n += imgs.shape[0] * len(dirs)
    return n


def cpu_baseline(n_images):
    gray, binary, dirs = workload(0)
    sample = [gray[:n_images], binary[:n_images]]
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    units = oracle_step(sample, dirs, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": units / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n_images} gray + {n_images} binary images of config 2 x all {len(dirs)} "
                      f"directions (ECT+Radon swept oracle + HT quadrature), {dt:.1f} s wall"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    gray, binary, dirs = workload(0)
    # each step a bounded sample of the workload: with the default 100 steps the
    # whole run stays within a couple of minutes on the host cores
    n = args.ref_sample
    sample = [gray[:n], binary[:n]]
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_step([s[:1] for s in sample], dirs, threads=cores)
    t0 = time.perf_counter()
    units = 0
    for _ in range(args.steps):
        units += oracle_step(sample, dirs, threads=cores)
    dt = time.perf_counter() - t0
    v = units / dt
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64 (ECT/Radon), f64 (HT)",
        "data": "synthetic (seeded generators, synth/)", "impl": "reference",
        "config": dict(arm_config(int(os.environ.get("WORLD_SIZE", "1"))),
                       sample=f"oracle on host cores; each step {n} gray + {n} binary images x {len(dirs)} directions"),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n} gray + {n} binary config-2 images x {len(dirs)} directions per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=96, help="images per variant in the cpu_baseline sample")
    ap.add_argument("--ref-sample", type=int, default=8, help="images per variant per --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    main()
