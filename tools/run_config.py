"""Runs one BASELINE.json config's bench step ITERS times (for ncu captures; no
timing). Same inputs and calls as bench.py.

  python tools/run_config.py config4|config2|config3|config1 [iters]
  python tools/run_config.py config5 [iters] [kernel] [precision] [algorithm]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    import paper_2405_02256_b200 as eu

    name = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = bench.workload(name, 0)
    imgs = torch.from_numpy(np.ascontiguousarray(w["images"])).cuda()
    if name == "config5":
        kern = sys.argv[3] if len(sys.argv) > 3 else "cos"
        prec = sys.argv[4] if len(sys.argv) > 4 else "f32"
        alg = sys.argv[5] if len(sys.argv) > 5 else "auto"
        param = dict(bench.C5_KERNELS)[kern]
        cx = eu.build_complex(imgs, "vertex")
        cr = eu.critical_points(cx)
        for _ in range(iters):
            eu.hybrid(cr, w["dirs"], kern, param, prec, algorithm=alg)
    else:
        ht = (bench.HT_KERNEL_C2, 1.0, "f64") if name == "config2_fused_ht" else None
        for _ in range(iters):
            bench.transforms_step(eu, imgs, w["dirs"], w["construction"], ht)
    torch.cuda.synchronize()
    print("ok", name, iters)


if __name__ == "__main__":
    main()
