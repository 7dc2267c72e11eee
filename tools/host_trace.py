"""Host-side cost of the bench step's API calls WITHOUT synchronisation between
them (diagnostics): mean wall time of each call as issued, the enqueue total,
and the final wait for the device. Also times the raw C entry points of one
variant with ctypes directly (no Python allocation) to separate binding cost
from library cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(gray).cuda(), torch.from_numpy(binary).cuda()]
T = {}


def tic(name, f, *a, **k):
    t0 = time.perf_counter()
    r = f(*a, **k)
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


N = 20
for it in range(N + 3):
    if it == 3:
        T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cxs = [tic(f"build[{v}]", eu.build_complex, img, "vertex") for v, img in enumerate(imgs)]
    crs = [tic(f"critical[{v}]", eu.critical_points, cx) for v, cx in enumerate(cxs)]
    out = []
    for v, cr in enumerate(crs):
        r = tic(f"transforms[{v}]", eu.transforms, cr, dirs, elem_bytes="auto", share_heights=True)
        h = tic(f"hybrid[{v}]", eu.hybrid, cr, dirs, "sin", 1.0, "f64")
        out.append((r, h))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    T["enqueue_total"] = T.get("enqueue_total", 0.0) + (t1 - t0) * 1e3
    T["final_wait"] = T.get("final_wait", 0.0) + (t2 - t1) * 1e3
    tic("release", lambda: (out.clear(), crs.clear(), cxs.clear()))
for k, v in T.items():
    print(f"{k:16s} {v / N:8.3f} ms")

# sub-steps of transforms() for the gray variant
cx = eu.build_complex(imgs[0], "vertex")
cr = eu.critical_points(cx)
torch.cuda.synchronize()
S = {}
for it in range(N):
    t0 = time.perf_counter()
    b = cr.output_bound(dirs)
    t1 = time.perf_counter()
    r = eu.transforms(cr, dirs, elem_bytes=2, share_heights=True)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    S["output_bound"] = S.get("output_bound", 0) + (t1 - t0) * 1e3
    S["transforms(eb=2)"] = S.get("transforms(eb=2)", 0) + (t2 - t1) * 1e3
for k, v in S.items():
    print(f"{k:16s} {v / N:8.3f} ms")
