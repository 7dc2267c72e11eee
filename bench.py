"""Benchmark of the hot path on BASELINE.json's configs.

Headline (the contract line's `value`): BASELINE.json configs[3] (config 4), the
largest single-GPU ECT/Radon workload: a 256^3 u8 smoothed-noise volume AND its
binary variant (v > median, P:146 / E15) as one batch of two volumes, vertex
construction, 1024 integer-rounded Fibonacci directions (E12). One step =
build (A0) + critical points (A1-A2, K1) + exact ECT and Radon, all three streams
(A3-A5, K2), for both volumes: 2048 image-directions.

Sub-records in the same JSON line ("configs"), each timed the same way with its
own oracle cpu_baseline sample from the same run:
  config1   32x32 u8 TOP, 32 directions: ECT + Radon (latency, us per step)
  config2   1024 x 28x28 blob images + binary variant, 256 directions: ECT + Radon
  config2_fused_ht  the same + the histogram-fused HT (kappa = sin, fp64; NEXT f2)
            — round 1's headline workload
  config3   2048^2 int16 GRF, 4096 directions: ECT + Radon
  config5   16 x 128^3 volumes, 10^4 directions: HT with exp(-t^2/2) and
            cos(2 pi t/64) in fp64 and fp32 (BJ:11): terms/s, GFLOP/s, LSU and FP32
            roofline fractions

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--shard images|directions]

Prints ONE JSON line (rank 0). --gpus N > 1 re-launches itself under
torch.distributed.run (one process per GPU, NCCL). Default sharding: every rank
runs the headline step on its own pair of volumes (rank 0 = config 4 exactly;
independent problems, no data-path collective): weak scaling. --shard directions:
every rank runs K1 on the same volumes and K2 on its contiguous chunk of the
orthant-grouped directions: strong scaling. Times are CUDA events
on the launching stream, max over ranks.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
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
HEADLINE = "config4"
C2_IMAGES = 1024
HT_KERNEL_C2 = "sin"
C5_KERNELS = [("gauss", 1.0), ("cos", 64.0)]
# flops per HT term of the tabulated kbar kernel k3t (the default K3 path), from
# its SASS inner loop (tools/k3t_sass.py): fp32 = one FFMA (J*kbar - c) + three
# FADD (Kahan), fp64 = one DFMA; the DP4A height and the table gather are not flops
F_TERM = {"f32": 5, "f64": 2}
SMS = 148


# ----------------------------------------------------------------------------- plumbing

def shard_range(n_units: int, rank: int, world: int):
    """Contiguous [start, stop) of n_units for this rank."""
    per = (n_units + world - 1) // world
    a = min(n_units, rank * per)
    return a, min(n_units, a + per)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args, argv):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run
    with N processes (rank 0 prints the line). Returns the exit code, or None when
    this process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


class Dist:
    """Rank info and the two collectives the bench needs (barrier, max)."""

    def __init__(self, backend):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()
        if self.backend == "nccl":
            import torch

            torch.cuda.synchronize()

    def max(self, x: float) -> float:
        if not self.dist:
            return float(x)
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """Samples nvidia-smi clocks and throttle reasons; mark()/end() bracket a timed region."""

    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index
        self.regions = {}
        self._open = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "25"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def mark(self, name):
        self._open = (name, len(self.samples))

    def end(self):
        name, first = self._open
        self.regions[name] = (first, len(self.samples) + 1)  # one more sample, in flight, counts

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self, name):
        a, b = self.regions.get(name, (0, len(self.samples)))
        s = self.samples[a:max(b, a + 1)]
        if not s and self.samples:  # a region shorter than the 25 ms sampling period: nearest sample
            i = min(a, len(self.samples) - 1)
            s = self.samples[i:i + 1]
        if not s:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(x[0]) for x in s if x[0].replace(".", "").isdigit()]
        mx = [float(x[1]) for x in s if len(x) > 1 and x[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for x in s for i in range(4) if len(x) > 3 + i and x[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(s)}


# ----------------------------------------------------------------------------- workloads

def pair_index(dirs):
    n = dirs.shape[1]
    full = (1 << n) - 1
    e = ((dirs > 0).astype(np.int64) << np.arange(n)).sum(1)
    return np.where((e >> (n - 1)) & 1, e ^ full, e)


def list_bytes(cr, dirs):
    """Algorithmic read bytes of K2: every record of the direction's orthant pair
    list, once per (image, direction); 8 B (12 B for int32 weights)."""
    lens = cr.list_lengths()  # [B, Q]
    rb = 8  # every bench config has |weights| <= 255: 8-byte records (int16 Delta^- halves)
    return int(lens[:, pair_index(dirs)].sum()) * rb


def k2_bytes(cr, dirs, r, ht=False):
    """Algorithmic bytes of one K2 call: the lists, ECT (h,v) + ordinary (h,v) +
    classical (v; heights shared with the ECT) + 3 offset arrays (+ HT f64)."""
    S = cr.cx.batch * len(dirs)
    ne = int(r["ect"]["offsets"][S])
    no = int(r["ordinary"]["offsets"][S])
    eb = r["ect"]["value"].element_size()
    return list_bytes(cr, dirs) + ne * 2 * eb + no * 2 * eb + ne * eb + 3 * (S + 1) * 8 + (S * 8 if ht else 0)


def workload(name, rank=0):
    """Inputs of a config for a rank (rank 0 = the BASELINE.json config exactly;
    other ranks draw their own images with the same recipe: weak scaling)."""
    import synth

    sh = 7919 * rank
    if name == "config4":
        gray = synth.smooth_volume(256, synth.IMAGE_SEED[4] + sh)
        dirs, nfix = synth.fibonacci_directions(1024, 32.0)
        return dict(images=np.stack([gray, synth.median_binarize(gray)]), dirs=dirs, construction="vertex",
                    variants="gray + binary (v > median)", zero_fixed=nfix)
    if name in ("config2", "config2_fused_ht"):
        gray = synth.blob_images(C2_IMAGES, 28, synth.IMAGE_SEED[2] + sh)
        return dict(images=np.concatenate([gray, synth.binarize(gray, 128)]),
                    dirs=synth.random_directions(256, 2, 16, synth.DIR_SEED[2]), construction="vertex",
                    variants="1024 gray + 1024 binary (>= 128)")
    if name == "config3":
        return dict(images=synth.grf_image(2048, synth.IMAGE_SEED[3] + sh)[None],
                    dirs=synth.random_directions(4096, 2, 64, synth.DIR_SEED[3]), construction="vertex",
                    variants="gray (256 levels, int16)")
    if name == "config1":
        return dict(images=synth.uniform_image((32, 32), 256, synth.IMAGE_SEED[1] + sh)[None],
                    dirs=synth.random_directions(32, 2, 8, synth.DIR_SEED[1]), construction="top",
                    variants="uniform u8")
    if name == "config5":
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(8) as ex:
            vols = list(ex.map(lambda j: synth.smooth_volume(128, 1500 + j + sh), range(16)))
        dirs, nfix = synth.fibonacci_directions(10000, 64.0)
        return dict(images=np.stack(vols), dirs=dirs, construction="vertex", variants="16 gray volumes",
                    zero_fixed=nfix)
    raise ValueError(name)


DESCR = {
    "config4": "BASELINE.json configs[3]: 256^3 u8 smoothed-noise volume (sigma 3) + its binary variant (v > median) "
               "as one batch, vertex construction, 1024 integer-rounded Fibonacci directions (x32); exact ECT + Radon "
               "(all three streams) per image-direction",
    "config2": "BASELINE.json configs[1]: 1024 x 28x28 u8 Gaussian-blob images + binary variant (>=128), vertex "
               "construction, 256 integer directions in [-16,16]^2; ECT + Radon for every image",
    "config2_fused_ht": "BASELINE.json configs[1] as config2, plus the HT (kappa=sin, fp64) from K2's merged "
                        "histogram (NEXT f2, eucalc_transforms_ht)",
    "config3": "BASELINE.json configs[2]: 2048^2 int16 k^-3 Gaussian random field (256 levels), vertex construction, "
               "4096 integer directions in [-64,64]^2; exact ECT + Radon",
    "config1": "BASELINE.json configs[0]: 32x32 u8 uniform, top construction, 32 directions in [-8,8]^2; ECT + Radon",
    "config5": "BASELINE.json configs[4]: 16 x 128^3 u8 smoothed-noise volumes, vertex construction, 10^4 "
               "integer-rounded Fibonacci directions (x64); HT with exp(-t^2/2) and cos(2 pi t/64), fp64 and fp32",
}


# ----------------------------------------------------------------------------- GPU steps

def transforms_step(eu, imgs_dev, dirs, construction, ht=None):
    cx = eu.build_complex(imgs_dev, construction)
    cr = eu.critical_points(cx)
    r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=ht)
    return cx, cr, r


def timed_loop(torch, eu, fn, steps, warmup, flush, dist=None):
    """W untimed warm-up steps, then K steps timed with CUDA events on the current
    stream (L2 flushed before each, untimed). Returns (last result, per-step ms,
    summed stage ms, launches)."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times, stage, launches, spans = [], {}, 0, {}
    res = None
    for _ in range(steps):
        flush.fill_(1.0)
        res = None  # the previous step's outputs are released before the next step
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eu.profile_enable(True)
        eu.launch_count(reset=True)
        e0.record(s)
        res = fn()
        e1.record(s)
        launches += eu.launch_count()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        for st in ("build", "k1_critical", "k2_transforms", "k3_hybrid"):
            stage[st] = stage.get(st, 0.0) + eu.profile_read(st)[0]
            spans[st] = spans.get(st, 0.0) + eu.profile_span(st)
        eu.profile_enable(False)
    if dist:
        dist.barrier()
    return res, times, stage, launches, spans


def spread(times):
    return {"min": float(np.min(times)), "median": float(np.median(times)), "max": float(np.max(times))}


def e2e_transforms(eu, torch, imgs_host, dirs, construction, steps, ht=None):
    """The same step through the C ABI with HOST buffers: pinned host images in
    (H2D inside eucalc_build_complex), host representations out (D2H inside
    eucalc_transforms). Returns (seconds per step list, h2d bytes, d2h bytes)."""

    def one():
        cx = eu.build_complex(imgs_host, construction)
        cr = eu.critical_points(cx)
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, device="cpu", ht=ht)
        h2d = imgs_host.numel() * imgs_host.element_size() + dirs.nbytes
        d2h = 0
        for k, st in r.items():
            if k == "ht":
                d2h += st.numel() * st.element_size()
                continue
            n = int(st["offsets"][-1])
            eb = st["value"].element_size()
            d2h += st["offsets"].numel() * 8 + n * eb + (n * eb if k != "classical" else 0)
        return h2d, d2h

    one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        h2d, d2h = one()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return ts, h2d, d2h


# ----------------------------------------------------------------------------- CPU oracle samples

def cores():
    return os.cpu_count() or 1


def oracle_transforms_sample(images, dirs, construction, dsel, ht=None):
    """Oracle ECT/Radon (+ HT quadrature) of every image x the directions `dsel`.
    Grid materialisation (once per image) is timed separately and charged to
    the sample in proportion len(dsel)/len(dirs), as the full workload amortises
    it over all its directions. Returns (units, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    nc = cores()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(min(nc, len(images))) as ex:
        grids = list(ex.map(lambda im: oracle.Grid(im, construction), images))
    t_grid = time.perf_counter() - t0
    pairs = [(b, d) for b in range(len(images)) for d in dsel]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(nc) as ex:
        list(ex.map(lambda bd: grids[bd[0]].transforms(dirs[bd[1]]), pairs))
        if ht:
            list(ex.map(lambda bd: grids[bd[0]].ht_quad(dirs[bd[1]], *ht), pairs))
    t_dirs = time.perf_counter() - t0
    return len(pairs), t_dirs + t_grid * len(dsel) / len(dirs), t_grid, t_dirs


def cpu_baseline(name, w, n_dirs):
    """The oracle (oracle/, plain C, threads over (image, direction)) on a bounded
    sample of the config's workload on this host's cores."""
    rng = np.random.default_rng(1)
    dirs = w["dirs"]
    images = w["images"]
    if name in ("config2", "config2_fused_ht"):
        n_img = n_dirs  # images per variant
        imgs = np.concatenate([images[:n_img], images[C2_IMAGES:C2_IMAGES + n_img]])
        ht = (HT_KERNEL_C2, 1.0) if name == "config2_fused_ht" else None
        units, secs, tg, td = oracle_transforms_sample(imgs, dirs, "vertex", list(range(len(dirs))), ht=ht)
        sample = (f"first {n_img} gray + {n_img} binary images x all {len(dirs)} directions (ECT+Radon"
                  + (" + HT quadrature)" if ht else ")"))
    else:
        dsel = sorted(rng.choice(len(dirs), min(n_dirs, len(dirs)), replace=False).tolist())
        units, secs, tg, td = oracle_transforms_sample(images, dirs, w["construction"], dsel)
        sample = (f"all {len(images)} image(s) x {len(dsel)} seeded directions (ECT+Radon swept oracle); grid "
                  f"materialisation {tg:.1f} s charged pro rata ({len(dsel)}/{len(dirs)})")
    return {"value": units / secs, "unit": UNIT, "cores": cores(), "kind": "oracle",
            "sample": sample + f", {td:.1f} s of direction work"}


def cpu_baseline_ht(w, n_vol, n_dirs):
    """Oracle HT (Radon quadrature, long double) on n_vol volumes x n_dirs directions, both kernels."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    dirs = w["dirs"]
    rng = np.random.default_rng(2)
    dsel = sorted(rng.choice(len(dirs), n_dirs, replace=False).tolist())
    nc = cores()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(min(nc, n_vol)) as ex:
        grids = list(ex.map(lambda im: oracle.Grid(im, "vertex"), w["images"][:n_vol]))
    tg = time.perf_counter() - t0
    pairs = [(b, d) for b in range(n_vol) for d in dsel]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(nc) as ex:
        for kern, param in C5_KERNELS:
            list(ex.map(lambda bd: grids[bd[0]].ht_quad(dirs[bd[1]], kern, param), pairs))
    td = time.perf_counter() - t0
    secs = td + tg * n_dirs / len(dirs)
    units = len(pairs) * len(C5_KERNELS)
    return {"value": units / secs, "unit": "image-direction HTs/s (one kernel)", "cores": nc, "kind": "oracle",
            "sample": f"{n_vol} volumes x {n_dirs} seeded directions x {len(C5_KERNELS)} kernels (Radon quadrature, "
                      f"long double; precision-independent), {td:.1f} s"}


# ----------------------------------------------------------------------------- records

def record_transforms(name, eu, torch, args, dist, flush, clk, steps, warmup, ht=None, headline=False):
    w = workload(name, dist.rank)
    dirs = w["dirs"]
    world = dist.world
    if headline and args.shard == "directions":
        import paper_2405_02256_b200 as eup

        w = workload(name, 0)
        idx, dirs = eup.shard_directions(w["dirs"], dist.rank, world)
        dirs = np.ascontiguousarray(dirs)
    imgs_dev = torch.from_numpy(np.ascontiguousarray(w["images"])).cuda()
    cons = w["construction"]
    clk.mark(name)
    res, times, stage, launches, spans = timed_loop(
        torch, eu, lambda: transforms_step(eu, imgs_dev, dirs, cons, ht), steps, warmup, flush, dist)
    clk.end()
    cx, cr, r = res
    dev_ms = dist.max(float(np.sum(times)))
    B, D = cx.batch, len(dirs)
    units_rank = B * D
    if headline and args.shard == "directions":
        units = B * len(w["dirs"]) * steps
    else:
        units = units_rank * world * steps
    value = units / (dev_ms / 1e3)
    hbm, _, psrc = peaks()
    k2_ms = spans["k2_transforms"] / steps
    kb = k2_bytes(cr, dirs, r, ht=ht is not None)
    achieved = kb / (k2_ms / 1e3) / 1e9
    npair = int(cr.list_lengths()[:, pair_index(dirs)].sum())
    _, mhz, _ = peaks()
    clk_mhz = (clk.summary(name).get("sm_mhz") or mhz)
    # K2 adds every record of a segment's list into the segment's histogram with one
    # shared atomic (packed bins): npair / 32 warp atomics per step
    warp_atoms = npair / 32.0
    rate = warp_atoms / (k2_ms / 1e3) / SMS / (clk_mhz * 1e6)
    apeak, asrc = atomics_peak()
    rec = {
        "value": value, "unit": UNIT, "ms_per_step": dev_ms / steps, "steps": steps, "warmup": warmup,
        "workload": DESCR[name], "images": B, "directions": D,
        "stages_ms_per_step": {k: v / steps for k, v in stage.items() if v},
        "step_ms_spread": spread(times),
        "critical_points_per_s": npair / (k2_ms / 1e3),
        "roofline": {"bound": "hbm", "kernel": "K2 (k2_transforms launches of the step)", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                     "peak_source": psrc, "algorithmic_bytes_per_launch": kb, "launch_ms": k2_ms,
                     "smem_atomics": {"warp_atomics_per_launch": warp_atoms,
                                      "achieved_per_clk_per_sm": rate, "peak_per_clk_per_sm": apeak,
                                      "frac": (rate / apeak) if apeak else None, "clock_mhz": clk_mhz,
                                      "peak_source": asrc,
                                      "note": "list bytes re-read per direction mostly hit L2 (SURVEY 8(d)): "
                                              "the fill is bound by shared-memory atomics, not HBM"}},
        "gpu_launches": int(launches),
        "clocks": clk.summary(name),
        "elem_bytes": int(r["ect"]["value"].element_size()),
    }
    if "zero_fixed" in w:
        rec["zero_fixed_directions"] = w["zero_fixed"]
    return rec, w, (cx, cr, r, dirs)


def atomics_peak():
    """Shared-memory atomic throughput measured on a B200 by tools/ubench/atoms.cu
    (profiles/r2/s7/atoms_ubench.jsonl): warp ATOMS instructions per clock per SM for
    pseudo-random addresses with the result used and OR-ed (K2's checked packed add)."""
    p = os.path.join(ROOT, "profiles", "r2", "s7", "atoms_ubench.jsonl")
    if os.path.exists(p):
        for line in open(p):
            try:
                d = json.loads(line)
            except ValueError:
                continue
            if d.get("mode", "").startswith("random, checked"):
                return float(d["warp_atoms_per_clk_per_sm"]), "measured (tools/ubench/atoms.cu, " + p[len(ROOT) + 1:] + ")"
    return None, None


def traffic_for(name):
    """ncu DRAM bytes per K2 launch group of this record (profiles/r2/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "r2", "traffic.json")
    if os.path.exists(p):
        t = json.load(open(p)).get(name)
        if t:
            return t.get("dram_bytes_per_step"), t.get("source")
    return None, None


def record_ht(eu, torch, args, dist, flush, clk, steps, warmup):
    w = workload("config5", dist.rank)
    dirs = w["dirs"]
    imgs_dev = torch.from_numpy(np.ascontiguousarray(w["images"])).cuda()
    cx = eu.build_complex(imgs_dev, "vertex")
    cr = eu.critical_points(cx)
    cnt = cr.counts()  # [B, 8, 2]
    e = ((dirs > 0).astype(np.int64) << np.arange(3)).sum(1)
    terms = int(cnt[:, e, 1].sum())  # ordinary points summed over (volume, direction)
    records = int(cr.list_lengths()[:, pair_index(dirs)].sum())
    _, mhz, _ = peaks()
    out = {"workload": DESCR["config5"], "images": cx.batch, "directions": len(dirs), "terms_per_call": terms,
           "records_per_call": records, "per_kernel": {}}
    clk.mark("config5")
    tot_ms = 0.0
    counters = {}
    cp = os.path.join(ROOT, "profiles", "r2", "k3t_counters.json")
    if os.path.exists(cp):
        counters = json.load(open(cp))
    for kern, param in C5_KERNELS:
        for prec in ("f64", "f32"):
            res, times, stage, launches, spans = timed_loop(
                torch, eu, lambda: eu.hybrid(cr, dirs, kern, param, prec), steps, warmup, flush, dist)
            ms = float(np.median(times))
            k3_ms = spans["k3_hybrid"] / steps
            tot_ms += ms
            tps = terms / (ms / 1e3)
            gf = tps * F_TERM[prec] / 1e9
            fp_peak = SMS * 128 * 2 * mhz * 1e6 / 1e9 if prec == "f32" else SMS * 64 * 2 * mhz * 1e6 / 1e9
            rec = {"ms": ms, "k3_ms": k3_ms, "terms_per_s": tps, "image_directions_per_s": cx.batch * len(dirs) / (ms / 1e3),
                   "gflops": gf, "flops_per_term": F_TERM[prec],
                   "fp_peak_gflops": fp_peak, "fp_frac": gf / fp_peak, "algorithm": "table (k3t)",
                   "step_ms_spread": spread(times), "gpu_launches": int(launches / steps)}
            c = counters.get(f"{kern}_{prec}")
            if c:
                wf = c["lsu_wavefronts_shared_per_launch"]
                lsu_peak = SMS * mhz * 1e6  # 1 shared-memory wavefront per clock per SM
                rec["lsu"] = {"wavefronts_per_launch": wf, "achieved_per_s": wf / (k3_ms / 1e3),
                              "peak_per_s": lsu_peak, "frac": wf / (k3_ms / 1e3) / lsu_peak,
                              "source": c.get("source")}
            out["per_kernel"][f"{kern}_{prec}"] = rec
    clk.end()
    out["ms_per_step_all_four"] = tot_ms
    out["clocks"] = clk.summary("config5")
    return out, w


def gpu_arm(args):
    import torch

    import paper_2405_02256_b200 as eu

    dist = Dist("nccl")
    torch.cuda.set_device(dist.local)
    eu.lib()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    clk = Clocks(dist.local).start()
    time.sleep(0.5)  # nvidia-smi start-up stalls the driver: keep it out of the timed region
    gc_was = gc.isenabled()

    head, w, (cx, cr, r, dirs) = record_transforms(HEADLINE, eu, torch, args, dist, flush, clk, args.steps,
                                                   args.warmup, headline=True)
    traffic, tsrc = traffic_for(HEADLINE)
    head["roofline"]["traffic"] = traffic
    head["roofline"]["traffic_source"] = tsrc
    del cx, cr, r
    # ---- e2e through the ABI with host buffers (pinned images in, host CSR out)
    imgs_host = torch.from_numpy(np.ascontiguousarray(w["images"])).pin_memory()
    dist.barrier()
    ts, h2d, d2h = e2e_transforms(eu, torch, imgs_host, dirs, w["construction"], max(3, min(args.steps, 10)))
    e2e_s = dist.max(float(np.sum(ts)))
    # units per step over all ranks: every rank's images x its directions
    units_step = head["images"] * (len(w["dirs"]) if args.shard == "directions" else head["directions"] * dist.world)
    e2e_value = units_step * len(ts) / e2e_s
    del imgs_host

    subs = {}
    if dist.world == 1 and not args.headline_only:
        sub_steps = max(3, min(args.steps, 10))
        for name, ht in (("config2", None), ("config2_fused_ht", (HT_KERNEL_C2, 1.0, "f64")), ("config3", None),
                         ("config1", None)):
            if name not in args.sub:
                continue
            rec, wsub, _ = record_transforms(name, eu, torch, args, dist, flush, clk,
                                             sub_steps if name != "config1" else max(10, args.steps),
                                             args.warmup, ht=ht)
            if name == "config1":
                rec["us_per_step"] = rec["ms_per_step"] * 1e3
            t, s = traffic_for(name)
            rec["roofline"]["traffic"], rec["roofline"]["traffic_source"] = t, s
            if not args.no_cpu_baseline:
                rec["cpu_baseline"] = cpu_baseline(name, wsub, {"config2": 96, "config2_fused_ht": 64, "config3": 192,
                                                                "config1": 32}[name])
            subs[name] = rec
            torch.cuda.empty_cache()
        if "config5" in args.sub:
            rec, w5 = record_ht(eu, torch, args, dist, flush, clk, max(3, min(args.steps, 5)), args.warmup)
            if not args.no_cpu_baseline:
                rec["cpu_baseline"] = cpu_baseline_ht(w5, 2, 48)
            subs["config5"] = rec
    clk.stop()
    if gc_was:
        gc.enable()

    line = None
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": dist.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if args.shard == "directions" else "weak", "vs_baseline": None,
            "dtype": "int32 (ECT/Radon outputs and histogram), int16 (critical records)",
            "data": "synthetic (seeded generators, synth/; recipes of SURVEY.md 8(d))",
            "config": {"workload": DESCR[HEADLINE], "images_per_gpu": head["images"],
                       "directions": head["directions"],
                       "parallelism": (f"dp{dist.world} (directions sharded)" if args.shard == "directions"
                                       else f"dp{dist.world}"),
                       "l2": "flushed between timed steps (256 MB write, untimed); inputs 33.5 MB",
                       "output": "CSR, narrowest exact int width, classical heights shared with ECT"},
            "stages_ms_per_step": head["stages_ms_per_step"],
            "step_ms_spread": head["step_ms_spread"],
            "critical_points_per_s": head["critical_points_per_s"],
            "roofline": head["roofline"],
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "step_ms_spread": {k: 1e3 * v for k, v in spread(ts).items()}},
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "zero_fixed_directions": head.get("zero_fixed_directions"),
            "configs": subs,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(HEADLINE, workload(HEADLINE, 0), 48)
        print(json.dumps(line), flush=True)
    dist.close()
    return line


# ----------------------------------------------------------------------------- reference arm (oracle)

def reference_arm(args):
    """The oracle on the headline's config, metric and unit, on the host cores:
    each step the full config-4 batch (gray + binary) x a bounded seeded sample of
    directions; grid materialisation once per volume, charged pro rata."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    w = workload(HEADLINE, 0)
    dirs = w["dirs"]
    nc = cores()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(2) as ex:
        grids = list(ex.map(lambda im: oracle.Grid(im, "vertex"), w["images"]))
    t_grid = time.perf_counter() - t0
    rng = np.random.default_rng(3)
    per_step = args.ref_sample

    def step():
        ds = rng.choice(len(dirs), per_step, replace=False)
        pairs = [(b, int(d)) for b in range(len(grids)) for d in ds]
        with ThreadPoolExecutor(nc) as ex:
            list(ex.map(lambda bd: grids[bd[0]].transforms(dirs[bd[1]]), pairs))
        return len(pairs)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    units = sum(step() for _ in range(args.steps))
    dt = time.perf_counter() - t0 + t_grid * (args.steps * per_step) / len(dirs)
    v = units / dt
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64 (ECT/Radon)",
        "data": "synthetic (seeded generators, synth/)", "impl": "reference",
        "config": {"workload": DESCR[HEADLINE], "images_per_gpu": 2, "directions": len(dirs),
                   "sample": f"oracle on host cores; each step both volumes x {per_step} seeded directions; grid "
                             f"materialisation ({t_grid:.1f} s for both volumes) charged pro rata"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nc, "kind": "oracle",
                         "sample": f"both config-4 volumes x {per_step} directions per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


# ----------------------------------------------------------------------------- plumbing check (CPU, gloo)

def plumbing_check(args):
    """The multi-rank plumbing of this script (spawn, rendezvous, per-rank shards,
    barrier, max over ranks, rank-0 line) on CPU with gloo. No compute: the
    'step' is the per-rank shard bookkeeping; tests/test_abi.py drives it."""
    dist = Dist("gloo")
    w_seed = [7919 * dist.rank]
    a, b = shard_range(1024, dist.rank, dist.world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dist.barrier()
    dt = dist.max(time.perf_counter() - t0)
    shards = [None] * dist.world
    if dist.dist:
        dist.dist.all_gather_object(shards, (dist.rank, a, b, w_seed[0]))
    else:
        shards = [(0, a, b, 0)]
    line = None
    if dist.rank == 0:
        line = {"metric": METRIC, "value": (b - a) * dist.world * args.steps / max(dt, 1e-9), "unit": UNIT,
                "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup, "plumbing_check": True,
                "shards": shards}
        print(json.dumps(line), flush=True)
    dist.close()
    return line


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="images", choices=["images", "directions"])
    ap.add_argument("--sub", default="config1,config2,config2_fused_ht,config3,config5",
                    help="sub-records to add at N=1 (comma list)")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=4, help="directions per volume per --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plumbing-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    args.sub = [s for s in args.sub.split(",") if s]
    if args.warmup < 3:
        args.warmup = 3
    rc = maybe_spawn(args, argv)
    if rc is not None:
        sys.exit(rc)
    if args.plumbing_check:
        return plumbing_check(args)
    if args.impl == "reference":
        return reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    main()
