"""Per-call host timing of the bench step (diagnostics, not product code)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(gray).cuda(), torch.from_numpy(binary).cuda()]
T = {}


def tic(name, f, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f(*a, **k)
    torch.cuda.synchronize()
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


for it in range(6):
    if it == 1:
        T.clear()
    for v, img in enumerate(imgs):
        cx = tic(f"build[{v}]", eu.build_complex, img, "vertex")
        cr = tic(f"critical[{v}]", eu.critical_points, cx)
        tic(f"bound[{v}]", cr.output_bound, dirs)
        r = tic(f"transforms[{v}]", eu.transforms, cr, dirs, elem_bytes="auto", share_heights=True)
        h = tic(f"hybrid[{v}]", eu.hybrid, cr, dirs, "sin", 1.0, "f64")
        tic(f"del[{v}]", lambda: (r.clear(), globals().update(_x=None)))
        del cx, cr, h
for k, v in T.items():
    print(f"{k:16s} {v / 5:8.3f} ms")
mid = os.environ.get("PROFILE_ONCE")
