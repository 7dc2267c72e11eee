"""NEXT row f4: the shapes of the paper's §5 experiments on synthetic
stand-ins, on one B200, through the C ABI. Prints one JSON line per point.

  size      P:175-201  binary m x m images of 10 x 10 periodic squares (100 classical /
                       200 ordinary points per orthant, checked), m varied: K1 grows with
                       m^2, the transforms stay flat.
  critical  P:203-229  1000 x 1000 binary squares, number of squares varied.
  directions P:231-250 one binarised blob image (fashion-MNIST stand-in), ECT for
                       1 .. 10^4 directions with positive coordinates (the paper samples
                       [0,1]^2; integer directions in [1,16]^2 here, BJ:5).
  vectorize P:252-258  1000 x 1000 image with ~10^6 critical points, ECT vectorised on
                       10 .. 10^6 points.
  levels    P:260-272  fraction of critical vertices vs number of gray levels, uniform and
                       k^-3 Gaussian-random-field 2-D images.

Times are CUDA-event stage times on the launching stream (eucalc_profile_*),
median of 5 after 2 warm-ups.

  python tools/experiments.py [--only size,critical,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def stage_times(eu, torch, fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    acc = {}
    for _ in range(reps):
        eu.profile_enable(True)
        fn()
        torch.cuda.synchronize()
        for st in ("k1_critical", "k2_transforms", "k3_hybrid", "k4_evaluate"):
            acc.setdefault(st, []).append(eu.profile_read(st)[0])
        eu.profile_enable(False)
    return {k: float(np.median(v)) for k, v in acc.items()}


def pos_dirs(D, k, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(1, k + 1, size=(D, 2)).astype(np.int32)


def exp_size(eu, torch):
    dirs = pos_dirs(100, 16, 7)
    for m in (100, 200, 400, 800, 1600, 2000):
        s = max(2, m // 20)
        img = synth.squares_image(m, 10, s)[None]
        dev = torch.from_numpy(img).cuda()
        cx = eu.build_complex(dev, "vertex")
        cr = eu.critical_points(cx)
        cnt = cr.counts()[0]
        assert all(tuple(cnt[e]) == (100, 200) for e in range(4)), cnt

        def run():
            c = eu.critical_points(eu.build_complex(dev, "vertex"))
            eu.transforms(c, dirs, elem_bytes="auto", share_heights=True)
            eu.hybrid(c, dirs, "sin", 1.0, "f64")

        t = stage_times(eu, torch, run)
        yield dict(experiment="size", m=m, vertices=m * m, classical=100, ordinary=200, directions=100, **t)


def exp_critical(eu, torch):
    dirs = pos_dirs(100, 16, 8)
    m = 1000
    for k in (1, 4, 16, 64, 128, 250):
        s = max(1, m // (2 * k))
        img = synth.squares_image(m, k, s)[None]
        dev = torch.from_numpy(img).cuda()
        cr = eu.critical_points(eu.build_complex(dev, "vertex"))
        cnt = cr.counts()[0]

        def run():
            c = eu.critical_points(eu.build_complex(dev, "vertex"))
            eu.transforms(c, dirs, elem_bytes="auto", share_heights=True)
            eu.hybrid(c, dirs, "sin", 1.0, "f64")

        t = stage_times(eu, torch, run)
        yield dict(experiment="critical", m=m, squares=k * k, classical=int(cnt[3, 0]), ordinary=int(cnt[3, 1]),
                   directions=100, **t)


def exp_directions(eu, torch):
    img = synth.binarize(synth.blob_images(1, 28, synth.IMAGE_SEED[2]), 128)
    dev = torch.from_numpy(img).cuda()
    for D in (1, 10, 100, 1000, 10000):
        dirs = pos_dirs(D, 16, 9)

        def run():
            c = eu.critical_points(eu.build_complex(dev, "vertex"))
            eu.ect(c, dirs, elem_bytes="auto")

        t = stage_times(eu, torch, run)
        yield dict(experiment="directions", directions=D, per_direction_us=1e3 * t["k2_transforms"] / D, **t)


def exp_vectorize(eu, torch):
    img = synth.uniform_image((1000, 1000), 4, 11)[None]
    dev = torch.from_numpy(img).cuda()
    dirs = np.array([[3, 5]], np.int32)
    cx = eu.build_complex(dev, "vertex")
    cr = eu.critical_points(cx)
    ncrit = int(cr.counts()[0, 3].sum())
    r = eu.ect(cr, dirs, elem_bytes=8)
    for N in (10, 100, 1000, 10000, 100000, 1000000):
        t = stage_times(eu, torch, lambda: eu.vectorize(cx, dirs, -1.0, 1.0, N, ect=r))
        yield dict(experiment="vectorize", m=1000, critical_points=ncrit, breakpoints=int(r["offsets"][-1]),
                   points=N, **{k: v for k, v in t.items() if k == "k4_evaluate"})


def exp_levels(eu, torch):
    m = 256
    for kind in ("uniform", "grf"):
        for levels in (2, 4, 8, 16, 32, 64, 128, 256):
            if kind == "uniform":
                img = synth.uniform_image((m, m), levels, 100 + levels)
            else:
                img = synth.grf_image(m, 200 + levels, levels=levels)
            cr = eu.critical_points(eu.build_complex(img[None].astype(np.int16), "vertex"))
            cnt = cr.counts()[0]  # [4 orthants][classical, ordinary]
            V = m * m
            yield dict(experiment="levels", kind=kind, levels=levels, vertices=V,
                       classical_frac=float(cnt[:, 0].mean() / V), ordinary_frac=float(cnt[:, 1].mean() / V))


def exp_real(eu, torch):
    """Real-valued directions (K5, NEXT f3): config-2 images x 100 directions uniform in
    [0,1]^2, the paper's Table 1 setting (6e6 image-directions in 117 s
    for the ECT on an i7-4770)."""
    for variant in ("gray", "binary"):
        c = synth.config_inputs(2, variant)
        dev = torch.from_numpy(c["images"]).cuda()
        dirs = np.random.default_rng(3).uniform(1e-3, 1.0, size=(100, 2))

        def run():
            cr = eu.critical_points(eu.build_complex(dev, "vertex"))
            eu.profile_enable(True)
            eu.transforms_real(cr, dirs, share_heights=True)

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            cr = eu.critical_points(eu.build_complex(dev, "vertex"))
            torch.cuda.synchronize()
            eu.profile_enable(True)
            eu.transforms_real(cr, dirs, share_heights=True)
            torch.cuda.synchronize()
            ts.append(eu.profile_read("k5_real")[0])
            eu.profile_enable(False)
        ms = float(np.median(ts))
        yield dict(experiment="real", variant=variant, images=int(dev.shape[0]), directions=100, k5_real_ms=ms,
                   image_directions_per_s=dev.shape[0] * 100 / (ms / 1e3))


def exp_real_large(eu, torch):
    """Real-valued directions on long lists (K5 bucketed path): config 3 (2048^2 GRF) and
    config 4 (256^3) with directions uniform in [0,1]^n; and the paper's §5 size
    experiment shape (1000 x 1000 image) with 100 such directions."""
    cases = [("config3", synth.config_inputs(3, "gray")["images"], 2, 256),
             ("config4", synth.config_inputs(4, "gray")["images"], 3, 64),
             ("squares1000", synth.squares_image(1000, 250, 2)[None], 2, 100)]
    for name, img, n, D in cases:
        dev = torch.from_numpy(img).cuda()
        dirs = np.random.default_rng(5).uniform(1e-3, 1.0, size=(D, n))
        cr = eu.critical_points(eu.build_complex(dev, "vertex"))
        recs = int(cr.counts().max())
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            eu.profile_enable(True)
            eu.transforms_real(cr, dirs, share_heights=True)
            torch.cuda.synchronize()
            if it:
                ts.append(eu.profile_read("k5_real")[0])
            eu.profile_enable(False)
        ms = float(np.median(ts))
        yield dict(experiment="real_large", input=name, directions=D, max_list=recs, k5_real_ms=ms,
                   directions_per_s=img.shape[0] * D / (ms / 1e3), records_per_s=recs * D / (ms / 1e3))


EXPS = {"size": exp_size, "critical": exp_critical, "directions": exp_directions, "vectorize": exp_vectorize,
        "levels": exp_levels, "real": exp_real,
        "real_large": exp_real_large}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(EXPS))
    args = ap.parse_args()
    import torch

    import paper_2405_02256_b200 as eu

    for name in args.only.split(","):
        for line in EXPS[name](eu, torch):
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
