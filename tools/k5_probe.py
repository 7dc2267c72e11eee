"""K5 (eucalc_transforms_real) on config 2 x 100 real directions in [0,1]^2 (the
paper's Table 1 setting; diagnostics / ncu target): prints the K5 stage time.
  python tools/k5_probe.py [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_02256_b200 as eu  # noqa: E402
import synth  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "gray"
c = synth.config_inputs(2, variant)
dirs = np.random.default_rng(3).uniform(1e-3, 1.0, size=(100, 2))
cr = eu.critical_points(eu.build_complex(torch.from_numpy(c["images"]).cuda(), "vertex"))
eu.transforms_real(cr, dirs, share_heights=True)
torch.cuda.synchronize()
eu.profile_enable(True)
N = int(os.environ.get("ITERS", "3"))
for _ in range(N):
    eu.transforms_real(cr, dirs, share_heights=True)
torch.cuda.synchronize()
ms = eu.profile_read("k5_real")[0] / N
print(f"K5 config 2 {variant} x 100 real dirs: {ms:.3f} ms, {1024 * 100 / ms * 1e3:.3e} image-dirs/s")
