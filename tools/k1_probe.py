"""K1 only, on config k's images (diagnostics / ncu target): ITERS calls of
eucalc_critical_points, then the mean K1 time from the library's stage events.
  python tools/k1_probe.py K [variant] [construction]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_02256_b200 as eu  # noqa: E402
import synth  # noqa: E402

k = int(sys.argv[1])
variant = sys.argv[2] if len(sys.argv) > 2 else "gray"
c = synth.config_inputs(k, variant)
cons = sys.argv[3] if len(sys.argv) > 3 else c["construction"]
img = torch.from_numpy(c["images"]).cuda()
cx = eu.build_complex(img, cons)
for _ in range(2):
    eu.critical_points(cx)
torch.cuda.synchronize()
eu.profile_enable(True)
N = int(os.environ.get("ITERS", "10"))
for _ in range(N):
    cr = eu.critical_points(cx)
torch.cuda.synchronize()
ms = eu.profile_read("k1_critical")[0] / N
nv = cx.batch
for m in c["images"].shape[1:]:
    nv *= m
print(f"config {k} {variant} {cons}: K1 {ms:.4f} ms, {nv / ms * 1e3:.3e} vertices/s")
