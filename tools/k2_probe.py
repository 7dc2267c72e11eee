"""K2 (eucalc_transforms) only on config k's images with the first D directions
(diagnostics / ncu target): prints the mean K2 stage time.
  python tools/k2_probe.py K [variant] [D] [elem_bytes]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_02256_b200 as eu  # noqa: E402
import synth  # noqa: E402

k = int(sys.argv[1])
variant = sys.argv[2] if len(sys.argv) > 2 else "gray"
c = synth.config_inputs(k, variant)
D = int(sys.argv[3]) if len(sys.argv) > 3 else len(c["dirs"])
eb = sys.argv[4] if len(sys.argv) > 4 else "auto"
eb = eb if eb == "auto" else int(eb)
dirs = c["dirs"][:D]
cx = eu.build_complex(torch.from_numpy(c["images"]).cuda(), c["construction"])
cr = eu.critical_points(cx)
eu.transforms(cr, dirs, elem_bytes=eb, share_heights=True)
torch.cuda.synchronize()
eu.profile_enable(True)
N = int(os.environ.get("ITERS", "3"))
for _ in range(N):
    r = eu.transforms(cr, dirs, elem_bytes=eb, share_heights=True)
torch.cuda.synchronize()
ms = eu.profile_read("k2_transforms")[0] / N
print(f"config {k} {variant} D={D} eb={r['ect']['value'].element_size()}: K2 {ms:.3f} ms, {cx.batch * D / ms * 1e3:.3e} image-dirs/s")
