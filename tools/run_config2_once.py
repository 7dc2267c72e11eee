"""One config-2 pass (gray then binary) for ncu captures (diagnostics, not product code)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
for it in range(int(os.environ.get("ITERS", "2"))):
    for img in (gray, binary):
        cx = eu.build_complex(torch.from_numpy(img).cuda(), "vertex")
        cr = eu.critical_points(cx)
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True)
        h = eu.hybrid(cr, dirs, "sin", 1.0, "f64")
        torch.cuda.synchronize()
print("ok")
