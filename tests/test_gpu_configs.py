"""GPU parity at the FULL sizes of BASELINE.json configs 3-5 (BJ:9-11), in the
launch configuration bench.py times (every direction of the config in one call,
narrowest exact output width, classical heights shared with the ECT), on
stated seeded samples that the oracle computes one by one:

  config 3 (2048^2 i16, 4096 dirs): 64 directions, 32 from each antipodal pair
      list, + the first and last direction; VERTEX and TOP; the full critical
      tables of the image (4 orthants).
  config 4 (256^3 u8, 1024 Fibonacci dirs): 8 directions per orthant (64),
      including >= 8 whose rounded zero component was fixed (E12); gray and
      binary (v > median, P:146 / E15) x VERTEX and TOP; the full critical
      tables of the volume (8 orthants).
  config 5 (16 x 128^3, 10^4 dirs): 2 directions per (volume, orthant) = 256
      pairs over all 16 volumes and 8 orthants, + the 16 pairs worst
      conditioned for the fp32 cos HT (tests/golden/config5_cos_conditioning.json,
      written by a script that calls only oracle/); kernels exp(-t^2/2) and
      cos(2 pi t/64) (BJ:11) x fp32/fp64 x per-term/tabulated kbar (K3) and the
      histogram-fused HT (f2); TOP on 64 pairs.

ECT/Radon/critical tables bit-exact; HT within 1e-9 (fp64) / 1e-4 (fp32) of
max(|ref|, 1) (BJ:5, E18), against the oracle's quadrature of the Radon
transform.
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_02256_b200 as eu  # noqa: E402

HT_TOL = {"f64": 1e-9, "f32": 1e-4}
NAMES = {"ect": ("T", "E"), "ordinary": ("To", "Eo"), "classical": ("Tc", "Ec")}
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THREADS = os.cpu_count() or 1


def orthant_of(dirs):
    return ((np.asarray(dirs) > 0).astype(np.int64) << np.arange(dirs.shape[1])).sum(1)


def pair_of(dirs):
    n = dirs.shape[1]
    e = orthant_of(dirs)
    return np.where((e >> (n - 1)) & 1, e ^ ((1 << n) - 1), e)


class Oracle:
    """Oracle grids of a batch, materialised once (in parallel), shared by the
    transforms, HT and critical-table checks of one test."""

    def __init__(self, images, construction, need):
        self.images, self.construction = images, construction
        with ThreadPoolExecutor(min(THREADS, len(need))) as ex:
            self.grids = dict(zip(need, ex.map(lambda b: oracle.Grid(images[b], construction), need)))

    def transforms(self, dirs, pairs):
        with ThreadPoolExecutor(THREADS) as ex:
            return dict(zip(pairs, ex.map(lambda bd: self.grids[bd[0]].transforms(dirs[bd[1]]), pairs)))

    def ht(self, dirs, pairs, kernel, param):
        with ThreadPoolExecutor(THREADS) as ex:
            return dict(zip(pairs, ex.map(lambda bd: self.grids[bd[0]].ht_quad(dirs[bd[1]], kernel, param), pairs)))


def gpu_segments(res, ids):
    """{stream: {s: (heights, values)}} of the listed segments only (device -> host)."""
    out = {}
    for k, st in res.items():
        if k == "ht":
            continue
        off = st["offsets"].cpu().numpy()
        out[k] = {}
        for s in ids:
            a, b = int(off[s]), int(off[s + 1])
            out[k][s] = (st["height"][a:b].cpu().numpy().astype(np.int64),
                         st["value"][a:b].cpu().numpy().astype(np.int64))
    return out


def check_transforms(ref, got, D):
    for (b, d), want in ref.items():
        s = b * D + d
        for k, (tn, en) in NAMES.items():
            h, v = got[k][s]
            np.testing.assert_array_equal(h, want[tn], err_msg=f"{k} heights b={b} d={d}")
            np.testing.assert_array_equal(v, want[en], err_msg=f"{k} values b={b} d={d}")


def check_critical_full(orc, cr, b):
    """Every orthant's critical table of image b (kept vertices, Delta^-, J) vs the
    oracle's star sums, orthants in parallel."""
    g = orc.grids[b]
    n = g.n

    def one(e):
        odm, oep = g.critical(e)
        keep = np.nonzero((odm != 0) | (oep != 0))[0]
        return e, keep, odm[keep], (odm - oep)[keep]

    with ThreadPoolExecutor(min(THREADS, 1 << n)) as ex:
        for e, keep, dm, j in ex.map(one, range(1 << n)):
            v, gdm, gj = cr.export(b, e)
            np.testing.assert_array_equal(v, keep, err_msg=f"kept vertices b={b} e={e}")
            np.testing.assert_array_equal(gdm, dm, err_msg=f"Delta^- b={b} e={e}")
            np.testing.assert_array_equal(gj, j, err_msg=f"J b={b} e={e}")


def bench_launch(images, dirs, construction):
    cx = eu.build_complex(images, construction)
    cr = eu.critical_points(cx)
    r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True)
    torch.cuda.synchronize()
    return cx, cr, r


# ----------------------------------------------------------------------------- config 3

@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_config3_full_size(construction):
    c = synth.config_inputs(3)
    img, dirs = c["images"], c["dirs"]
    D = len(dirs)
    cx, cr, r = bench_launch(img, dirs, construction)
    q = pair_of(dirs)
    rng = np.random.default_rng(3003)
    sel = set(rng.choice(np.nonzero(q == 0)[0], 32, replace=False).tolist())
    sel |= set(rng.choice(np.nonzero(q == 1)[0], 32, replace=False).tolist())
    sel |= {0, D - 1}
    pairs = [(0, int(d)) for d in sorted(sel)]
    orc = Oracle(img, construction, [0])
    check_transforms(orc.transforms(dirs, pairs), gpu_segments(r, [d for _, d in pairs]), D)
    check_critical_full(orc, cr, 0)


# ----------------------------------------------------------------------------- config 4

def config4_sample(dirs):
    """8 directions per orthant, at least one with a fixed zero component (E12)
    in each orthant that has one; >= 8 fixed directions overall."""
    fixed = synth.fibonacci_zero_fixed(len(dirs), 32.0)
    e = orthant_of(dirs)
    rng = np.random.default_rng(4004)
    sel = []
    for o in range(8):
        idx = np.nonzero(e == o)[0]
        fx = idx[fixed[idx]]
        take = list(rng.choice(fx, min(len(fx), 2), replace=False)) if len(fx) else []
        rest = np.setdiff1d(idx, take)
        take += list(rng.choice(rest, 8 - len(take), replace=False))
        sel += [int(x) for x in take]
    assert int(fixed[sel].sum()) >= 8 and len(set(e[sel])) == 8
    return sorted(sel)


@pytest.mark.parametrize("construction", ["vertex", "top"])
@pytest.mark.parametrize("variant", ["gray", "binary"])
def test_config4_full_size(variant, construction):
    c = synth.config_inputs(4, variant)
    vol, dirs = c["images"], c["dirs"]
    D = len(dirs)
    cx, cr, r = bench_launch(vol, dirs, construction)
    sel = config4_sample(dirs)
    pairs = [(0, d) for d in sel]
    orc = Oracle(vol, construction, [0])
    check_transforms(orc.transforms(dirs, pairs), gpu_segments(r, sel), D)
    check_critical_full(orc, cr, 0)


# ----------------------------------------------------------------------------- config 5

def config5_pairs(dirs, per=2, seed=5005, volumes=range(16)):
    e = orthant_of(dirs)
    rng = np.random.default_rng(seed)
    pairs = []
    for j in volumes:
        for o in range(8):
            idx = np.nonzero(e == o)[0]
            pairs += [(j, int(d)) for d in rng.choice(idx, per, replace=False)]
    return pairs


def worst_conditioned():
    g = json.load(open(os.path.join(GOLDEN, "config5_cos_conditioning.json")))
    return [tuple(p) for p in g["pairs"]]


def check_ht_values(out, ref, tol, label):
    bad = []
    for (b, d), want in ref.items():
        got = float(out[b, d])
        if not abs(got - want) <= tol * max(abs(want), 1.0):
            bad.append((b, d, got, want))
    assert not bad, (label, len(bad), bad[:5])


@pytest.fixture(scope="module")
def config5():
    c = synth.config_inputs(5)
    vols, dirs = c["images"], c["dirs"]
    cx = eu.build_complex(vols, "vertex")
    cr = eu.critical_points(cx)
    orc = Oracle(vols, "vertex", list(range(16)))
    return vols, dirs, cx, cr, orc


@pytest.mark.parametrize("kernel,param", [("gauss", 1.0), ("cos", 64.0)])
def test_config5_ht_full_size(config5, kernel, param):
    vols, dirs, cx, cr, orc = config5
    pairs = config5_pairs(dirs)
    if kernel == "cos":
        pairs += [p for p in worst_conditioned() if p not in pairs]
    assert len({j for j, _ in pairs}) == 16 and len(set(orthant_of(dirs[[d for _, d in pairs]]))) == 8
    ref = orc.ht(dirs, pairs, kernel, param)
    for precision in ("f64", "f32"):
        for alg in ("direct", "table"):
            out = eu.hybrid(cr, dirs, kernel, param, precision, algorithm=alg).cpu().numpy()
            check_ht_values(out, ref, HT_TOL[precision], (kernel, precision, alg))
    # histogram-fused HT (f2) over the sampled directions, all 16 volumes
    dsel = sorted({d for _, d in pairs})
    pos = {d: i for i, d in enumerate(dsel)}
    sub = np.ascontiguousarray(dirs[dsel])
    for precision in ("f64", "f32"):
        fused = eu.transforms(cr, sub, elem_bytes="auto", share_heights=True, ht=(kernel, param, precision))
        out = fused["ht"].cpu().numpy()
        check_ht_values(out, {(b, pos[d]): v for (b, d), v in ref.items()}, HT_TOL[precision],
                        (kernel, precision, "fused"))
        del fused


def test_config5_worst_conditioned_fp32_cos(config5):
    """The 16 pairs with the largest sum|J kbar| / |HT| (cos kernel) hold 1e-4 in fp32."""
    vols, dirs, cx, cr, orc = config5
    pairs = worst_conditioned()
    g = json.load(open(os.path.join(GOLDEN, "config5_cos_conditioning.json")))
    assert len(pairs) == 16 and min(g["cond"]) > g["cond_median_all"]
    ref = orc.ht(dirs, pairs, "cos", 64.0)
    for alg in ("direct", "table"):
        out = eu.hybrid(cr, dirs, "cos", 64.0, "f32", algorithm=alg).cpu().numpy()
        check_ht_values(out, ref, 1e-4, ("cos", "f32", alg, "worst"))


def test_config5_top_sampled():
    c = synth.config_inputs(5)
    vols, dirs = c["images"], c["dirs"]
    cx = eu.build_complex(vols, "top")
    cr = eu.critical_points(cx)
    # 64 pairs: 4 orthants per volume (even orthants for even volumes, odd for odd)
    e = orthant_of(dirs)
    rng = np.random.default_rng(5006)
    pairs = [(j, int(rng.choice(np.nonzero(e == o)[0]))) for j in range(16) for o in range(j % 2, 8, 2)]
    assert len(pairs) == 64 and len(set(orthant_of(dirs[[d for _, d in pairs]]))) == 8
    orc = Oracle(vols, "top", sorted({j for j, _ in pairs}))
    for kernel, param in (("gauss", 1.0), ("cos", 64.0)):
        ref = orc.ht(dirs, pairs, kernel, param)
        for precision in ("f64", "f32"):
            for alg in ("direct", "table"):
                out = eu.hybrid(cr, dirs, kernel, param, precision, algorithm=alg).cpu().numpy()
                check_ht_values(out, ref, HT_TOL[precision], (kernel, precision, alg, "top"))
