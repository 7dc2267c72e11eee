"""How many K2 segments redo their fill with split bins after a checked packed
add flagged (diagnostic). EUCALC_K2_CHK_BITS=14 is the default checked range;
setting it only makes the library read the restart counter back.

  EUCALC_K2_CHK_BITS=14 python tools/restarts.py config3 config4
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("EUCALC_K2_CHK_BITS", "14")

import bench  # noqa: E402


def main():
    import torch

    import paper_2405_02256_b200 as eu

    for name in sys.argv[1:] or ["config3", "config4"]:
        w = bench.workload(name, 0)
        imgs = torch.from_numpy(np.ascontiguousarray(w["images"])).cuda()
        eu.k2_restarts(reset=True)
        cx, cr, r = bench.transforms_step(eu, imgs, w["dirs"], w["construction"])
        torch.cuda.synchronize()
        print(name, "segments", cx.batch * len(w["dirs"]), "restarts", eu.k2_restarts(), flush=True)


if __name__ == "__main__":
    main()
