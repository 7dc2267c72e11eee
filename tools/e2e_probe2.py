"""e2e step timing inside a bench-like process (device-resident steps first),
per API call (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

_empty = torch.empty


def timed_empty(*a, **k):
    t0 = time.perf_counter()
    r = _empty(*a, **k)
    dt = (time.perf_counter() - t0) * 1e3
    if dt > 1.0:
        print(f"  torch.empty{tuple(a)} pin={k.get('pin_memory')} took {dt:.1f} ms")
    return r


torch.empty = timed_empty
gray, binary, dirs = bench.workload(0)
batches = bench.step_batches(gray, binary)
dev = [torch.from_numpy(x).cuda() for x in batches]
host = [torch.from_numpy(x).pin_memory() for x in batches]
if os.environ.get("DEVICE_FIRST", "1") == "1":
    for _ in range(100):
        res = bench.run_step(eu, torch, dev, dirs)
    torch.cuda.synchronize()
for it in range(int(os.environ.get('IT', '16'))):
    t0 = time.perf_counter()
    cx = eu.build_complex(host[0], "vertex")
    t1 = time.perf_counter()
    cr = eu.critical_points(cx)
    t2 = time.perf_counter()
    r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, device="cpu", ht=(bench.HT_KERNEL, 1.0, "f64"))
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.2f} critical {1e3*(t2-t1):.2f} transforms(host out) {1e3*(t3-t2):.2f} sync {1e3*(t4-t3):.2f} ms")
