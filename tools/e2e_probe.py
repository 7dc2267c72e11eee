"""Host-side cost split of bench.py's e2e step (diagnostics): pinned output
allocation vs the C call (K1/K2 + device->host copies) per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(x).pin_memory() for x in bench.step_batches(gray, binary)]
T = {}
_empty = torch.empty


def timed_empty(*a, **k):
    t0 = time.perf_counter()
    r = _empty(*a, **k)
    T["torch.empty(pinned)"] = T.get("torch.empty(pinned)", []) + [(time.perf_counter() - t0) * 1e3]
    return r


torch.empty = timed_empty
for it in range(12):
    t0 = time.perf_counter()
    bench.run_step_e2e(eu, torch, imgs, dirs)
    torch.cuda.synchronize()
    T["step"] = T.get("step", []) + [(time.perf_counter() - t0) * 1e3]
for k, v in T.items():
    print(k, " ".join(f"{x:.2f}" for x in v))
