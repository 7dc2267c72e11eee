"""Host cost of the pieces of eu.transforms() (diagnostics)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2405_02256_b200 as eu
gray, binary, dirs = bench.workload(0)
img = torch.from_numpy(gray).cuda()
cx = eu.build_complex(img, "vertex"); cr = eu.critical_points(cx); torch.cuda.synchronize()
T = {}
def t(name, f, *a, **k):
    t0 = time.perf_counter(); r = f(*a, **k); T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e6; return r
N = 50
for i in range(N + 5):
    if i == 5: T.clear()
    d = t("dirs_i32", eu._dirs_i32, dirs)
    b = t("output_bound", cr.output_bound, d)
    r = {}
    for name in ("ect", "ordinary", "classical"):
        r[name] = t("alloc_steps", eu._alloc_steps, torch, 1024 * 256, b[0], 2, "cuda", with_height=name != "classical")
    p, keep = eu._ptr(d)
    st = t("stream", eu._stream, None)
    req = ctypes.c_int64()
    sts = [r[k][1] for k in ("ect", "ordinary", "classical")]
    sts[2].height = sts[0].height
    t("c_transforms", eu.lib().eucalc_transforms, cr._h, p, 256, ctypes.byref(sts[0]), ctypes.byref(sts[1]), ctypes.byref(sts[2]), ctypes.byref(req), st)
    t("c_hybrid", eu.hybrid, cr, dirs, "sin", 1.0, "f64")
    torch.cuda.synchronize()
for k, v in T.items(): print(f"{k:14s} {v / N:8.1f} us")
