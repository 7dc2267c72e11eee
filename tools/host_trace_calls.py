"""Host wall time of every C entry point and of torch.empty during bench.py's
step (diagnostics): the library handle is wrapped so each ctypes call is timed;
the step runs as in bench.run_step (two streams, no synchronisation between
calls except the library's own wait on K1). Prints mean us per step per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

T = {}


class Timed:
    def __init__(self, L):
        self._L = L

    def __getattr__(self, name):
        f = getattr(self._L, name)
        if not callable(f):
            return f

        def g(*a):
            t0 = time.perf_counter()
            r = f(*a)
            T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e6
            return r
        return g


real = eu.lib()
eu._lib = Timed(real)
_empty = torch.empty


def timed_empty(*a, **k):
    t0 = time.perf_counter()
    r = _empty(*a, **k)
    T["torch.empty"] = T.get("torch.empty", 0.0) + (time.perf_counter() - t0) * 1e6
    return r


torch.empty = timed_empty
gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(x).cuda() for x in bench.step_batches(gray, binary)]
N = 30
tot = 0.0
for it in range(N + 5):
    if it == 5:
        T.clear()
        tot = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = bench.run_step(eu, torch, imgs, dirs)
    tot += (time.perf_counter() - t0) * 1e6
    torch.cuda.synchronize()
    del out
print(f"run_step host total {tot / N:8.1f} us")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"{k:34s} {v / N:8.1f} us")

# one step's call sequence: (call, start, end) in us since run_step entry
SEQ = []
T0 = [0.0]


class Seq(Timed):
    def __getattr__(self, name):
        f = getattr(self._L, name)
        if not callable(f):
            return f

        def g(*a):
            t0 = time.perf_counter()
            r = f(*a)
            SEQ.append((name, (t0 - T0[0]) * 1e6, (time.perf_counter() - T0[0]) * 1e6))
            return r
        return g


eu._lib = Seq(real)
for it in range(3):
    SEQ.clear()
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    out = bench.run_step(eu, torch, imgs, dirs)
    SEQ.append(("run_step returned", (time.perf_counter() - T0[0]) * 1e6, 0.0))
    torch.cuda.synchronize()
    del out
for name, a, b in SEQ:
    print(f"{name:34s} {a:8.1f} {b:8.1f}")
