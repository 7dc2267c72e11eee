"""Oracle pins for real-valued directions (NEXT row f3, E22).

The real-direction oracle sweeps the cell sums over the distinct double vertex
heights <xi, x> (P:116 embedding, left-to-right, no FMA). It is pinned
  * to the integer-lattice oracle where every dot is exact in double (vertex
    spacing 1/(M-1) dyadic, small integer xi): same breakpoints (as exact
    paper heights t(H)) and values — an independent code path;
  * to Lemma 2 (sign E1) evaluated on the oracle's critical tables
    with heights computed here by numpy in the same order — a different formula;
  * to the Appendix A evaluations and vectorisation.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import evaluate_ect, lemma2_transforms

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))


def vertex_heights(g, xi):
    """<xi, x> for every vertex (row-major ids), x_i = p_i/(M_i-1) - 0.5, summed left to right."""
    M = [int(v) for v in g.M]
    coords = np.array(np.unravel_index(np.arange(int(np.prod(M))), M), dtype=np.float64)
    h = None
    for i in range(g.n):
        x = coords[i] / float(M[i] - 1) - 0.5 if M[i] > 1 else np.zeros(coords.shape[1])
        t = float(xi[i]) * x
        h = t if h is None else h + t
    return h + 0.0


@pytest.mark.parametrize("shape,construction", [((9, 9), "vertex"), ((5, 5, 5), "vertex"), ((8, 8), "top"),
                                                ((1, 9), "vertex"), ((4, 4, 4), "top")])
def test_real_equals_lattice_when_exact(shape, construction):
    rng = np.random.default_rng(len(shape) * 7 + shape[0])
    for trial in range(6):
        img = rng.integers(-2, 6, size=shape).astype(np.int32)
        g = oracle.Grid(img, construction)
        xi = synth.random_directions(1, len(shape), 5, 40 + trial)[0]
        ri = g.transforms(xi)
        rr = g.transforms_real(xi.astype(np.float64))
        for hk, vk in (("T", "E"), ("To", "Eo"), ("Tc", "Ec")):
            np.testing.assert_array_equal(rr[hk], g.t_of(ri[hk], xi))
            np.testing.assert_array_equal(rr[vk], ri[vk])


@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_real_equals_lemma2(construction):
    rng = np.random.default_rng(5)
    for trial in range(10):
        shape = tuple(rng.integers(2, 7, size=rng.integers(2, 4)))
        img = rng.integers(0, 5, size=shape).astype(np.int32)
        g = oracle.Grid(img, construction)
        xi = rng.uniform(0.05, 1.0, size=len(shape)) * rng.choice([-1.0, 1.0], size=len(shape))
        e = int(sum(1 << i for i, v in enumerate(xi) if v > 0))
        c, dm, o, j = g.critical_table(e)
        h = vertex_heights(g, xi)
        want = lemma2_transforms(h[c], dm, h[o], j)
        got = g.transforms_real(xi)
        for k in ("T", "To", "Tc"):
            np.testing.assert_array_equal(got[k], np.asarray(want[k], dtype=np.float64), err_msg=f"{k} {trial}")
        for k in ("E", "Eo", "Ec"):
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"{k} {trial}")
        assert got["E"][-1] == g.euler() and (len(got["Eo"]) == 0 or got["Eo"][-1] == 0)


def test_real_appendix_evaluations():
    """P:337 ECT(xi,-0.3) = 3, ECT(xi,1) = 2 and P:341 [1,1,2,2,2] with xi = (2,2) as reals."""
    g = oracle.Grid(synth.EX4, "vertex")
    r = g.transforms_real(np.array(GOLD["xi"], dtype=np.float64))
    for t, v in GOLD["evaluate"]["ect_at"]:
        assert evaluate_ect(r["T"], r["E"], t) == v
    vz = GOLD["vectorize"]
    ts = g.sample_points(vz["a"], vz["b"], vz["N"])
    assert [evaluate_ect(r["T"], r["E"], t) for t in ts] == vz["values"]
