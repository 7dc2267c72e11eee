"""Config-2 binary variant diagnostics: distribution of the pair-list lengths
(the K2 warp regime's sparse path takes lists of <= 32 records) and a few K2
calls for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
for name, img in (("gray", gray), ("binary", binary)):
    cx = eu.build_complex(torch.from_numpy(img).cuda(), "vertex")
    cr = eu.critical_points(cx)
    L = cr.list_lengths()
    q = np.percentile(L, [0, 10, 50, 90, 99, 100])
    print(name, "list lengths pct 0/10/50/90/99/100:", q, "frac<=32:", float((L <= 32).mean()),
          "frac<=64:", float((L <= 64).mean()))
    if name == "binary":
        for _ in range(int(os.environ.get("ITERS", "3"))):
            eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=(bench.HT_KERNEL, 1.0, "f64"))
        torch.cuda.synchronize()
