"""One bench step (config 2 gray + binary as bench.py's step batches and
run_step) per iteration, for ncu captures (diagnostics, not product code)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_02256_b200 as eu  # noqa: E402

gray, binary, dirs = bench.workload(0)
imgs = [torch.from_numpy(x).cuda() for x in bench.step_batches(gray, binary)]
for it in range(int(os.environ.get("ITERS", "2"))):
    bench.run_step(eu, torch, imgs, dirs)
    torch.cuda.synchronize()
print("ok")
