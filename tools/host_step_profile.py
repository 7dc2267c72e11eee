"""Host cost of each API call of bench.py's step (diagnostics): wall time of
build_complex / critical_points / transforms per variant (GPU drained before each
call, so no call waits on earlier device work except its own K1), then a cProfile
of transforms() to split Python marshalling from the C call."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(gray).cuda(), torch.from_numpy(binary).cuda()]
T = {}
N = 30
for it in range(N + 5):
    for v, img in enumerate(imgs):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cx = eu.build_complex(img, "vertex")
        t1 = time.perf_counter()
        cr = eu.critical_points(cx)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(bench.HT_KERNEL, 1.0, "f64"))
        t4 = time.perf_counter()
        if it >= 5:
            for k, dt in (("build", t1 - t0), ("critical", t2 - t1), ("transforms(K1 done)", t4 - t3)):
                T[(v, k)] = T.get((v, k), 0.0) + dt * 1e6
for (v, k), t in T.items():
    print(f"variant {v} {k:22s} {t / N:8.1f} us")
torch.cuda.synchronize()
cx = eu.build_complex(imgs[0], "vertex")
cr = eu.critical_points(cx)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(bench.HT_KERNEL, 1.0, "f64"))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
