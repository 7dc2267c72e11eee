"""Oracle pins for evaluation and vectorisation at real t (NEXT row f1).

The oracle evaluates the DEFINITIONS (cell sums of ECT(xi,t) = chi[phi_{xi<=t}]
and Radon(xi,t) = chi[phi_{xi=t}]) at the exact rational image of a double t.
It is pinned against the paper's printed evaluation and vectorisation values
 and against the binary-search evaluation of the canonical arrays
(tests/helpers.py, strict rule E7) — a different code path —
at breakpoints, between them and outside the support.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import evaluate_ect, evaluate_radon

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))


def test_appendix_evaluation_definition():
    """ECT(xi,-0.3) = 3, ECT(xi,1) = 2; vectorisation on [-2,2], N=5 -> [1,1,2,2,2]."""
    g = oracle.Grid(synth.EX4, "vertex")
    xi = GOLD["xi"]
    for t, v in GOLD["evaluate"]["ect_at"]:
        assert g.ect_eval(xi, t) == v
    vz = GOLD["vectorize"]
    assert g.vectorize(xi, vz["a"], vz["b"], vz["N"]).tolist() == vz["values"]
    assert g.sample_points(vz["a"], vz["b"], vz["N"]) == [-2.0, -1.0, 0.0, 1.0, 2.0]


def test_appendix_radon_evaluation():
    """Radon of EX4 along (2,2): E_c = [1,2,1] at T_c = [-2,-2/3,0] (E3) and
    E' = [0,2,1,0] after T = [-2/3, 2/3, 4/3] (sign E1); -2 is classical but
    not ordinary, so Radon(-2) = 1 and Radon = 0 just after it."""
    g = oracle.Grid(synth.EX4, "vertex")
    xi = GOLD["xi"]
    assert g.radon_eval(xi, -2.0) == 1
    assert g.radon_eval(xi, -1.5) == 0
    assert g.radon_eval(xi, -0.5) == 2
    assert g.radon_eval(xi, 0.0) == 1
    assert g.radon_eval(xi, 0.5) == 2
    assert g.radon_eval(xi, 1.0) == 1
    assert g.radon_eval(xi, 1.5) == 0
    assert g.radon_eval(xi, math.inf) == 0 and g.ect_eval(xi, math.inf) == 2 and g.ect_eval(xi, -math.inf) == 0
    # far outside the support (beyond int64 in doubled lattice units): ECT(+-oo) limits
    assert g.ect_eval(xi, 1e300) == g.euler() == 2 and g.ect_eval(xi, -1e300) == 0
    assert g.radon_eval(xi, 1e300) == 0 and g.radon_eval(xi, -1e300) == 0


def _queries(g, xi, r, rng):
    """Doubles: exact breakpoints (when representable), their neighbours, midpoints, outside."""
    L, cs = g.L, g.csum(xi)
    hs = sorted(set(r["T"].tolist()) | set(r["To"].tolist()))
    qs = [-1e9, 1e9, -0.75, 0.0, 0.5]
    for h in hs:
        t = (2 * h - L * cs) / (2 * L)
        qs += [t, np.nextafter(t, -np.inf), np.nextafter(t, np.inf), t + 0.5 / L]
    qs += list(rng.uniform(-3, 3, 20))
    return [float(q) for q in qs]


@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_eval_matches_search_on_canonical_arrays(construction):
    rng = np.random.default_rng(11)
    for trial in range(12):
        shape = tuple(rng.integers(1, 6, size=rng.integers(2, 4)))
        img = rng.integers(-2, 5, size=shape).astype(np.int32)
        g = oracle.Grid(img, construction)
        xi = [int(v) for v in synth.random_directions(1, len(shape), 4, 100 + trial)[0]]
        r = g.transforms(xi)
        for t in _queries(g, xi, r, rng):
            h = Fraction(t) * g.L + Fraction(g.L * g.csum(xi), 2)  # exact lattice height of t
            assert g.ect_eval(xi, t) == evaluate_ect(r["T"], r["E"], h), (trial, t)
            assert g.radon_eval(xi, t) == evaluate_radon(r["To"], r["Eo"], r["Tc"], r["Ec"], h), (trial, t)


def test_sample_points_order_of_operations():
    """E20: t_i = a + (i*(b-a))/(N-1) in double; N = 1 gives [a]; endpoints exact for these."""
    assert oracle.Grid.sample_points(0.1, 0.7, 1) == [0.1]
    pts = oracle.Grid.sample_points(-0.5, 0.5, 101)
    assert pts[0] == -0.5 and pts[-1] == 0.5 and pts[50] == 0.0
    assert pts[3] == -0.5 + (3 * 1.0) / 100
