"""GPU parity of evaluation / vectorisation (K4, NEXT row f1) against the oracle's
definition-level evaluation at the same double t (E7, E20)."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_02256_b200 as eu  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))


def reps(images, dirs, construction, elem_bytes=8, share=True):
    cx = eu.build_complex(np.ascontiguousarray(images), construction)
    cr = eu.critical_points(cx)
    r = eu.transforms(cr, dirs, elem_bytes=elem_bytes, share_heights=share)
    return cx, cr, r


def test_ex4_golden_eval_vectorize():
    img = synth.EX4[None]
    xi = np.array([GOLD["xi"]], np.int32)
    cx, cr, r = reps(img, xi, "vertex")
    ts = [t for t, _ in GOLD["evaluate"]["ect_at"]]
    got = eu.evaluate(cx, xi, ts, ect=r["ect"]).cpu().numpy()[0]
    assert got.tolist() == [v for _, v in GOLD["evaluate"]["ect_at"]]
    vz = GOLD["vectorize"]
    got = eu.vectorize(cx, xi, vz["a"], vz["b"], vz["N"], ect=r["ect"]).cpu().numpy()[0]
    assert got.tolist() == vz["values"]
    # Radon: E_c = [1,2,1] at T_c = [-2,-2/3,0], E' = [2,1,0] after [-2/3,2/3,4/3] (E1, E3)
    tr = [-2.0, -1.5, -0.5, 0.0, 0.5, 1.0, 1.5, math.inf, -math.inf, math.nan]
    got = eu.evaluate(cx, xi, tr, ordinary=r["ordinary"], classical=r["classical"]).cpu().numpy()[0]
    assert got.tolist() == [1, 0, 2, 1, 2, 1, 0, 0, 0, 0]


def queries_for(images, dirs, construction, pairs, rng):
    """Doubles that hit breakpoints of the sampled segments exactly, their
    neighbours, midpoints, random points and the infinities."""
    qs = [-math.inf, math.inf, -1e300, 1e300, 0.0, -0.0, 0.25, 1e-300]
    for b, d in pairs:
        g = oracle.Grid(images[b], construction)
        r = g.transforms(dirs[d])
        for h in list(r["T"][:6]) + list(r["To"][-6:]):
            t = float(g.t_of(h, dirs[d]))
            qs += [t, float(np.nextafter(t, -np.inf)), float(np.nextafter(t, np.inf))]
    qs += list(rng.uniform(-1.5, 1.5, 40))
    return np.array(qs, np.float64)


def check(images, dirs, construction, r, cx, qs, pairs, out_eb=8, device="cuda"):
    D = len(dirs)
    e = eu.evaluate(cx, dirs, qs, ect=r["ect"], out_elem_bytes=out_eb, device=device).cpu().numpy()
    o = eu.evaluate(cx, dirs, qs, ordinary=r["ordinary"], classical=r["classical"], out_elem_bytes=out_eb,
                    device=device).cpu().numpy()
    grids = {}
    for b, d in pairs:
        g = grids.setdefault(b, oracle.Grid(images[b], construction))
        want_e = [g.ect_eval(dirs[d], float(t)) for t in qs]
        want_o = [g.radon_eval(dirs[d], float(t)) for t in qs]
        np.testing.assert_array_equal(e[b * D + d], want_e, err_msg=f"ECT eval b={b} d={d}")
        np.testing.assert_array_equal(o[b * D + d], want_o, err_msg=f"Radon eval b={b} d={d}")


CASES = [((9, 13), 3, "vertex", 256, 8, 7), ((9, 13), 3, "top", 5, 8, 7), ((6, 7, 5), 2, "vertex", 256, 5, 6),
         ((5, 4, 6), 2, "top", 3, 4, 5), ((1, 9), 2, "vertex", 5, 4, 3)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}")
def test_eval_parity(case):
    shape, batch, construction, levels, k, nd = case
    rng = np.random.default_rng(abs(hash(case)) & 0xFFFF)
    images = rng.integers(0, levels, size=(batch, *shape)).astype(np.uint8)
    dirs = synth.random_directions(nd, len(shape), k, 7)
    cx, cr, r = reps(images, dirs, construction)
    pairs = [(b, d) for b in range(batch) for d in range(nd)]
    qs = queries_for(images, dirs, construction, pairs[:4], rng)
    check(images, dirs, construction, r, cx, qs, pairs)


@pytest.mark.parametrize("elem_bytes,out_eb", [(2, 4), (4, 4), (4, 8), (8, 8)])
def test_eval_widths_and_host_buffers(elem_bytes, out_eb):
    images = synth.blob_images(3, 28, 5)
    dirs = synth.random_directions(6, 2, 16, 6)
    cx, cr, r = reps(images, dirs, "vertex", elem_bytes=elem_bytes)
    rng = np.random.default_rng(1)
    pairs = [(0, 0), (2, 5), (1, 3)]
    qs = queries_for(images, dirs, "vertex", pairs, rng)
    check(images, dirs, "vertex", r, cx, qs, pairs, out_eb=out_eb)
    # host representations and host output through the same ABI
    rh = {k: {kk: (vv.cpu() if vv is not None else None) for kk, vv in v.items()} for k, v in r.items()}
    rh["classical"]["height"] = rh["ect"]["height"]
    check(images, dirs, "vertex", rh, cx, qs, pairs, out_eb=out_eb, device="cpu")


def test_vectorize_config2_sampled():
    """Config 2 at full size in the bench's launch configuration (int16 representations,
    shared heights), vectorised on [-1, 1] with N = 100 (demeter's T = 100)."""
    c = synth.config_inputs(2, "gray")
    imgs, dirs = c["images"], c["dirs"]
    cx, cr, r = reps(imgs, dirs, "vertex", elem_bytes="auto")
    ve = eu.vectorize(cx, dirs, -1.0, 1.0, 100, ect=r["ect"]).cpu().numpy()
    vr = eu.vectorize(cx, dirs, -1.0, 1.0, 100, ordinary=r["ordinary"], classical=r["classical"]).cpu().numpy()
    rng = np.random.default_rng(3)
    D = len(dirs)
    for b, d in [(0, 0), (1023, 255)] + [(int(x), int(y)) for x, y in zip(rng.integers(0, 1024, 6),
                                                                          rng.integers(0, 256, 6))]:
        g = oracle.Grid(imgs[b], "vertex")
        np.testing.assert_array_equal(ve[b * D + d], g.vectorize(dirs[d], -1.0, 1.0, 100, "ect"))
        np.testing.assert_array_equal(vr[b * D + d], g.vectorize(dirs[d], -1.0, 1.0, 100, "radon"))


def test_eval_errors():
    images = synth.blob_images(2, 28, 3)
    dirs = synth.random_directions(3, 2, 8, 1)
    cx, cr, r = reps(images, dirs, "vertex", elem_bytes=8)
    with pytest.raises(eu.EucalcError) as ei:
        eu.evaluate(cx, dirs, [0.0], ect=r["ect"], out_elem_bytes=4)  # int64 rep -> int32 out refused
    assert ei.value.status == eu.E_ARG
    bad = np.array([[1, 0], [1, 1], [2, 2]], np.int32)
    with pytest.raises(eu.EucalcError) as ei:
        eu.evaluate(cx, bad, [0.0], ect=r["ect"])
    assert ei.value.status == eu.E_NONGENERIC
