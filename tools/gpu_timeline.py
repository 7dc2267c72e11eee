"""Device timeline of the bench step (diagnostics): CUDA events recorded on the
stream between the API calls, L2 flushed before each step as in bench.py.
Prints, per marker, the device time since the step start (mean over steps) and
the host time at which the marker was enqueued."""
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
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
FLUSH = os.environ.get("FLUSH", "1") == "1"
N = 10
acc_dev, acc_host = {}, {}
for it in range(N + 3):
    if FLUSH:
        flush.fill_(1.0)
    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        marks.append((name, e, time.perf_counter()))

    mark("start")
    cxs = []
    for v, img in enumerate(imgs):
        cxs.append(eu.build_complex(img, "vertex"))
        mark(f"build[{v}]")
    crs = []
    for v, cx in enumerate(cxs):
        crs.append(eu.critical_points(cx))
        mark(f"critical[{v}]")
    out = []
    for v, cr in enumerate(crs):
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True)
        mark(f"transforms[{v}]")
        h = eu.hybrid(cr, dirs, "sin", 1.0, "f64")
        mark(f"hybrid[{v}]")
        out.append((r, h))
    torch.cuda.synchronize()
    if it >= 3:
        e0, h0 = marks[0][1], marks[0][2]
        for name, e, h in marks:
            acc_dev[name] = acc_dev.get(name, 0.0) + e0.elapsed_time(e)
            acc_host[name] = acc_host.get(name, 0.0) + (h - h0) * 1e3
print(f"{'marker':16s} {'device_ms':>10s} {'host_enqueued_ms':>16s}")
for k in acc_dev:
    print(f"{k:16s} {acc_dev[k] / N:10.3f} {acc_host[k] / N:16.3f}")
