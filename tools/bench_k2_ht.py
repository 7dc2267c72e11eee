"""K2 on bench.py's 2048-image step batch with and without the fused HT, and
per variant (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
only = os.environ.get("ONLY")
for name, imgs in (("merged", np.concatenate([gray, binary])), ("gray", gray), ("binary", binary)):
    if only and name != only:
        continue
    cr = eu.critical_points(eu.build_complex(torch.from_numpy(imgs).cuda(), "vertex"))
    for ht in (None, (bench.HT_KERNEL, 1.0, "f64")):
        for _ in range(2):
            eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=ht)
        torch.cuda.synchronize()
        eu.profile_enable(True)
        N = 10
        for _ in range(N):
            eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=ht)
        torch.cuda.synchronize()
        ms = eu.profile_read("k2_transforms")[0] / N
        eu.profile_enable(False)
        print(f"{name:7s} ht={'f64' if ht else 'none':4s} K2 {ms:.4f} ms")
