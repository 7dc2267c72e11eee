"""Per-config stage measurements for all five BASELINE.json configs (diagnostics;
bench.py stays the contract's single-line benchmark on configs[1]).

For each config: device-resident inputs, W warm-up passes, then K timed passes;
each stage timed with the library's CUDA events on the launching stream
(eucalc_profile_*). Prints one JSON line per (config, variant, stage group):
image-directions/s, critical points/s (sum over segments of the pair-list
length / K2 time), algorithmic bytes / time against the HBM peak, and for the
HT terms/s.

  python tools/bench_configs.py [--configs 1,2,3,4,5] [--steps K] [--warmup W] [--construction vertex]
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


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p)).get("hbm_gbs", 6650.0))
    return 6650.0


def pair_of(dirs):
    n = dirs.shape[1]
    full = (1 << n) - 1
    e = ((dirs > 0).astype(np.int64) << np.arange(n)).sum(1)
    return np.where((e >> (n - 1)) & 1, e ^ full, e)


def run(eu, torch, k, variant, construction, steps, warmup, ht_kernels, out):
    c = synth.config_inputs(k, variant)
    imgs = torch.from_numpy(np.ascontiguousarray(c["images"])).cuda()
    dirs = c["dirs"]
    cons = construction or c["construction"]
    D = len(dirs)
    B = imgs.shape[0]
    do_tr = k != 5
    rec = {}

    def one():
        cx = eu.build_complex(imgs, cons)
        cr = eu.critical_points(cx)
        r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True) if do_tr else None
        hts = {}
        for kern, param, prec in ht_kernels[:1] if k == 5 else ():
            hts[(kern, prec)] = eu.hybrid(cr, dirs, kern, param, prec)
        return cx, cr, r, hts

    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    stage = {}
    ev = []
    for _ in range(steps):
        eu.profile_enable(True)
        cx, cr, r, hts = one()
        torch.cuda.synchronize()
        for st in ("k1_critical", "k2_transforms", "k3_hybrid"):
            ms, n = eu.profile_read(st)
            stage[st] = stage.get(st, 0.0) + ms
        eu.profile_enable(False)
    for st in stage:
        stage[st] /= steps
    lens = cr.list_lengths()  # [B, Q]
    q = pair_of(dirs)
    npair = int(lens[:, q].sum())  # sum over segments of the pair-list length
    nvert = int(np.prod([s + (1 if cons == "top" else 0) for s in imgs.shape[1:]])) * B
    peak = hbm_peak()
    base = {"config": k, "variant": variant, "construction": cons, "batch": B, "directions": D,
            "steps": steps}
    # K1: image read + records written (8 B per kept vertex per pair)
    rb = 8 if not getattr(cr, "wide", False) else 12
    k1_bytes = imgs.numel() * imgs.element_size() + int(lens.sum()) * rb
    out.append(dict(base, stage="k1_critical", ms=stage["k1_critical"], vertices=nvert,
                    vertices_per_s=nvert / (stage["k1_critical"] / 1e3),
                    algorithmic_bytes=k1_bytes,
                    gbs=k1_bytes / (stage["k1_critical"] / 1e3) / 1e9,
                    hbm_frac=k1_bytes / (stage["k1_critical"] / 1e3) / 1e9 / peak))
    if do_tr:
        S = B * D
        ne = int(r["ect"]["offsets"][S])
        no = int(r["ordinary"]["offsets"][S])
        eb = r["ect"]["value"].element_size()
        k2_bytes = npair * 8 + ne * 2 * eb + no * 2 * eb + ne * eb + 3 * (S + 1) * 8
        t = stage["k2_transforms"] / 1e3
        out.append(dict(base, stage="k2_transforms", ms=stage["k2_transforms"],
                        image_directions_per_s=S / t, critical_points_per_s=npair / t,
                        entries_ect=ne, entries_ordinary=no, elem_bytes=eb,
                        algorithmic_bytes=k2_bytes, gbs=k2_bytes / t / 1e9, hbm_frac=k2_bytes / t / 1e9 / peak))
    if k == 5:
        # per (kernel, precision) timing, one call each
        cnt = cr.counts()  # [B, 2^n, 2]
        full = (1 << dirs.shape[1]) - 1
        e = ((dirs > 0).astype(np.int64) << np.arange(dirs.shape[1])).sum(1)
        nterms = int(cnt[:, e, 1].sum())  # ordinary points summed over (image, direction)
        nrec = npair
        for (kern, param, prec), alg in [(h, a) for h in ht_kernels for a in ("direct", "table")]:
            for _ in range(2):
                eu.hybrid(cr, dirs, kern, param, prec, algorithm=alg)
            torch.cuda.synchronize()
            eu.profile_enable(True)
            for _ in range(steps):
                eu.hybrid(cr, dirs, kern, param, prec, algorithm=alg)
            torch.cuda.synchronize()
            ms, _ = eu.profile_read("k3_hybrid")
            eu.profile_enable(False)
            ms /= steps
            out.append(dict(base, stage=f"k3_hybrid[{kern},{prec},{alg}]", ms=ms,
                            image_directions_per_s=B * D / (ms / 1e3),
                            ordinary_terms=nterms, records_evaluated=nrec,
                            terms_per_s=nterms / (ms / 1e3), records_per_s=nrec / (ms / 1e3)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--construction", default=None)
    args = ap.parse_args()
    import torch

    import paper_2405_02256_b200 as eu

    ht = [("gauss", 1.0, "f64"), ("gauss", 1.0, "f32"), ("cos", 64.0, "f64"), ("cos", 64.0, "f32")]
    for k in [int(x) for x in args.configs.split(",")]:
        variants = ["gray", "binary"] if k in (2, 4) else ["gray"]
        for v in variants:
            out = []
            run(eu, torch, k, v, args.construction, args.steps, args.warmup, ht, out)
            for line in out:
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
