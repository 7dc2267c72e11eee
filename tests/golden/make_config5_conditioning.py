"""Writes tests/golden/config5_cos_conditioning.json: the (volume, direction)
pairs of BASELINE.json config 5 (BJ:11) whose hybrid transform with the cos
kernel (kappa(t) = cos(2 pi t / 64), E11) is worst conditioned, ranked by

    cond(b, d) = sum_x |J(x) kbar(t(x))| / |HT(b, d)|,   HT = -sum_x J(x) kbar(t(x))

over the ordinary points x of the direction's orthant (Lemma 2, sign
E1; kbar(t) = 64/(2 pi) sin(2 pi t / 64)). A large cond means heavy
cancellation: those pairs stress the fp32 HT path (SURVEY.md 8(c) "HT
numerics", measured up to 3.9e4). The GPU parity test checks them against the
oracle's quadrature (oracle.Grid.ht_quad); this file only SELECTS the pairs, it
stores no expected value. It calls only oracle/ (critical tables) and numpy.

  python tests/golden/make_config5_conditioning.py [--top 16]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

PERIOD = 64.0
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config5_cos_conditioning.json")


def volume_conditioning(j: int):
    c = synth.config_inputs(5)
    vol, dirs = c["images"][j], c["dirs"]
    g = oracle.Grid(vol, "vertex")
    M = [int(x) for x in g.M]
    e_of = ((dirs > 0).astype(np.int64) << np.arange(3)).sum(1)
    cond = np.empty(len(dirs))
    ht = np.empty(len(dirs))
    for e in range(8):
        _, _, o, jj = g.critical_table(e)
        coords = np.array(np.unravel_index(o, M)).T.astype(np.int64)
        aj = np.abs(jj).astype(np.float64)
        for d in np.nonzero(e_of == e)[0]:
            xs = g.xs(dirs[d])
            H = coords @ xs
            lo = int(H.min())
            hsum = np.bincount(H - lo, weights=jj.astype(np.float64))
            habs = np.bincount(H - lo, weights=aj)
            Hs = np.arange(lo, lo + len(hsum), dtype=np.float64)
            t = (2.0 * Hs - g.L * g.csum(dirs[d])) / (2.0 * g.L)
            kbar = PERIOD / (2 * math.pi) * np.sin(2 * math.pi * t / PERIOD)
            val = -float(np.dot(hsum, kbar))
            ht[d] = val
            cond[d] = float(np.dot(habs, np.abs(kbar))) / max(abs(val), 1e-300)
    return j, cond, ht


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--top", type=int, default=16)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    rows = []
    with ProcessPoolExecutor(args.workers) as ex:
        for j, cond, ht in ex.map(volume_conditioning, range(16)):
            for d in range(len(cond)):
                rows.append((float(cond[d]), j, d, float(ht[d])))
            print(f"volume {j}: max cond {cond.max():.4g}, median {np.median(cond):.4g}", flush=True)
    rows.sort(reverse=True)
    conds = np.array([r[0] for r in rows])
    out = {
        "what": "config 5 (BJ:11) (volume, direction) pairs with the largest sum|J kbar| / |HT| for the cos kernel "
                "(period 64, E11), VERTEX construction; selection only, no expected values",
        "script": "tests/golden/make_config5_conditioning.py (oracle critical tables + numpy)",
        "cite": "Lemma 2 P:99-101 (HT = -sum J kbar, sign E1); SURVEY.md 8(c) HT numerics",
        "pairs": [[j, d] for _, j, d, _ in rows[:args.top]],
        "cond": [c for c, _, _, _ in rows[:args.top]],
        "cond_median_all": float(np.median(conds)),
        "cond_max_all": float(conds.max()),
    }
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("pairs", "cond", "cond_median_all")}))


if __name__ == "__main__":
    main()
