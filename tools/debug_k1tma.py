import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_02256_b200 as eu, synth
shape = tuple(int(x) for x in sys.argv[1].split("x"))
dt = {"u8": np.uint8, "i16": np.int16}[sys.argv[2]]
batch = int(sys.argv[3]); warm = int(sys.argv[4])
rng = np.random.default_rng(0)
if warm:
    c0 = eu.critical_points(eu.build_complex(synth.blob_images(2, 28, 1), "vertex")); torch.cuda.synchronize()
img = rng.integers(0, 256, size=(batch, *shape)).astype(dt)
cx = eu.build_complex(img, "vertex")
cr = eu.critical_points(cx)
torch.cuda.synchronize()
print("K1 ok", cr.list_lengths())
