"""Host vs device timeline of one bench step (diagnostics): host perf_counter at
every call boundary of build -> critical_points -> transforms, and a CUDA event
recorded right after each call (device time at which the stream reached it).

  python tools/host_trace.py [config2|config4|config3] [reps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    import paper_2405_02256_b200 as eu

    L = eu.lib()
    acc = {}

    class Timed:  # wraps a ctypes function: host seconds per call, summed
        def __init__(self, nm, f):
            self.nm, self.f = nm, f

        def __call__(self, *a):
            t = time.perf_counter()
            r = self.f(*a)
            acc[self.nm] = acc.get(self.nm, 0.0) + time.perf_counter() - t
            return r

    for nm in ("eucalc_build_complex", "eucalc_critical_points", "eucalc_output_bound_upper", "eucalc_transforms",
               "eucalc_transforms_ht", "eucalc_destroy_critical", "eucalc_destroy_complex"):
        setattr(L, nm, Timed(nm, getattr(L, nm)))
    name = sys.argv[1] if len(sys.argv) > 1 else "config2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    w = bench.workload(name, 0)
    imgs = torch.from_numpy(np.ascontiguousarray(w["images"])).cuda()
    ht = (bench.HT_KERNEL_C2, 1.0, "f64") if name == "config2_fused_ht" else None
    for _ in range(3):
        bench.transforms_step(eu, imgs, w["dirs"], w["construction"], ht)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    for rep in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        h = [time.perf_counter()]
        ev[0].record(s)
        cx = eu.build_complex(imgs, w["construction"])
        h.append(time.perf_counter())
        ev[1].record(s)
        cr = eu.critical_points(cx)
        h.append(time.perf_counter())
        ev[2].record(s)
        r = eu.transforms(cr, w["dirs"], elem_bytes="auto", share_heights=True, ht=ht)
        h.append(time.perf_counter())
        ev[3].record(s)
        ev[3].synchronize()
        h.append(time.perf_counter())
        hd = [1e3 * (x - h[0]) for x in h]
        if rep == reps - 1:
            print("  C-call host ms (this rep):", {k: round(v * 1e3, 3) for k, v in acc.items()}, flush=True)
        acc.clear()
        gd = [ev[0].elapsed_time(e) for e in ev]
        print(f"{name} rep {rep}: host returns build {hd[1]:.3f} K1 {hd[2]:.3f} K2call {hd[3]:.3f} done {hd[4]:.3f} ms;"
              f" device marks build {gd[1]:.3f} K1 {gd[2]:.3f} K2 {gd[3]:.3f} ms", flush=True)
        del r, cr, cx


if __name__ == "__main__":
    main()
