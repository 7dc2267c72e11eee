"""Small inputs through every kernel family, for compute-sanitizer:
K1 (2-D single-region, 2-D multi-tile, 3-D; VERTEX and TOP; k1_scan/k1_copy),
K2 warp regime (count / scan / emit, sparse register sort + slab, fused HT),
K2 block regime (single window, staged multi-window with tile culling, checked
packed bins and their split restart), K3 (tabulated and per-term, f32 / f64),
K4 (evaluation, vectorisation) and K5 (warp sort, bucketed pieces).

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py
No timing, no oracle: results are only synchronised (the GPU tests check values).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    import torch

    import paper_2405_02256_b200 as eu

    rng = np.random.default_rng(5)
    cases = [
        (synth.blob_images(6, 28, 11), synth.random_directions(9, 2, 16, 1), "vertex"),      # warp regime
        (synth.binarize(synth.blob_images(6, 28, 12), 128), synth.random_directions(9, 2, 16, 2), "top"),  # sparse
        (rng.integers(0, 7, size=(2, 70, 100)).astype(np.uint8), synth.random_directions(5, 2, 6, 3), "top"),
        (synth.grf_image(160, 5)[None], np.array([[90, -89], [-90, 90], [3, 5]], np.int32), "vertex"),  # block
        (synth.smooth_volume(40, 77)[None], np.array([[400, -399, 398], [5, 7, -3]], np.int32), "vertex"),
        (rng.integers(0, 256, size=(2, 9, 11, 13)).astype(np.uint8), synth.random_directions(6, 3, 5, 4), "top"),
        (rng.integers(-40000, 40000, size=(2, 12, 11)).astype(np.int32), synth.random_directions(4, 2, 5, 8),
         "vertex"),  # int32 weights: wide records
    ]
    for k, (imgs, dirs, cons) in enumerate(cases):
        cx = eu.build_complex(np.ascontiguousarray(imgs), cons)
        cr = eu.critical_points(cx)
        cr.counts()
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True)
        eu.transforms(cr, dirs, elem_bytes=8, ht=("sin", 1.0, "f64"))
        eu.transforms(cr, dirs, elem_bytes=4, device="cpu")
        for prec in ("f32", "f64"):
            for alg in ("table", "direct"):
                eu.hybrid(cr, dirs, "cos", 64.0, prec, algorithm=alg)
        eu.vectorize(cx, dirs, -1.0, 1.0, 17, ect=r["ect"])
        eu.evaluate(cx, dirs, np.linspace(-1.0, 1.0, 9), ordinary=r["ordinary"], classical=r["classical"])
        real = rng.uniform(-1.0, 1.0, size=(3, imgs.ndim - 1))
        real[np.abs(real) < 1e-3] = 0.5
        eu.transforms_real(cr, real)
        torch.cuda.synchronize()
        print("case", k, "ok", flush=True)
    # checked packed bins forced to restart, and the bucketed K5 path
    os.environ["EUCALC_K2_CHK_BITS"] = "1"
    vol = synth.smooth_volume(48, 78)[None]
    cr = eu.critical_points(eu.build_complex(vol, "vertex"))
    eu.transforms(cr, np.array([[31, -30, 29], [-300, 200, 100]], np.int32))
    del os.environ["EUCALC_K2_CHK_BITS"]
    os.environ["EUCALC_K5_SMALL_MAX"] = "0"
    os.environ["EUCALC_K5_BUCKET"] = "16"
    img = rng.integers(0, 256, size=(1, 40, 40)).astype(np.uint8)
    cr = eu.critical_points(eu.build_complex(img, "vertex"))
    eu.transforms_real(cr, np.array([[0.3, 0.7], [-0.2, 0.9]]))
    torch.cuda.synchronize()
    print("sanitize run ok", flush=True)


if __name__ == "__main__":
    main()
