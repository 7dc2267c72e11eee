"""Pins of the CPU oracle to things other than itself (CPU only).

Each test names what fixes the expected value: a printed value of the paper
(tests/golden/appendix_a.json), a closed form, an invariant proved in the paper,
an independent formula of the paper (Lemma 2 vs Lemma 1/4), or a textbook
routine (connected-component labelling, exact line/cell geometry).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import (critical_heights, digital_euler_2d, evaluate_ect, evaluate_radon,
                           lemma2_transforms, orthant, slice_components_2d)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))


def _ex4():
    return oracle.Grid(np.array(GOLD["image"]["rows"], dtype=np.int32), "vertex")


# ----------------------------------------------------------------------------- Appendix A

def test_ex4_cell_counts():
    """'Cells with non-zero values include 9 vertices, 9 edges, and 2 squares'."""
    g = _ex4()
    u = np.indices(g.cells.shape).reshape(2, -1).T
    dim = (u % 2).sum(1)
    nz = g.cells.reshape(-1) != 0
    counts = [int((nz & (dim == k)).sum()) for k in range(3)]
    assert counts == [9, 9, 2]
    assert g.euler() == 9 - 9 + 2


def _paper_vertex(key):
    # E4: paper key k = c0 + 7*c1 with c0 the fast axis -> C-order doubled cell (c1, c0)
    c0, c1 = key % 7, key // 7
    assert c0 % 2 == 0 and c1 % 2 == 0
    return (c1 // 2) * 4 + (c0 // 2)


def _paper_orthant(eps):
    # paper eps (e0, e1) acts on (fast, slow) = (axis1, axis0)  (E4)
    mine = (eps[1], eps[0])
    return orthant(mine)


@pytest.mark.parametrize("row", GOLD["table2"]["rows"], ids=lambda r: str(r["eps"]))
def test_table2(row):
    """Table 2: classical points/values exactly; ordinary values = -J (E1)."""
    g = _ex4()
    c, dm, o, j = g.critical_table(_paper_orthant(row["eps"]))
    want_c = {_paper_vertex(k): v for k, v in zip(row["cls_points"], row["cls_values"])}
    want_o = {_paper_vertex(k): -v for k, v in zip(row["ord_points"], row["ord_values"])}
    assert dict(zip(c.tolist(), dm.tolist())) == want_c
    assert dict(zip(o.tolist(), j.tolist())) == want_o


def test_worked_vertex_32():
    """x = 32, eps = (1,-1): e_- = 0, e_+ = -1 (ordinary)."""
    w = GOLD["worked_vertex"]
    g = _ex4()
    dm, ep = g.critical(_paper_orthant(w["eps"]))
    v = _paper_vertex(w["key"])
    assert (int(dm[v]), int(ep[v])) == (w["e_minus"], w["e_plus"])


def test_appendix_ect_radon():
    """ECT T=[-2,-0.67,0], E=[0,1,3,2]; Radon T=[-0.67,0.67,1.33], T_c=[-2,-0.67,0];
    E' is printed negated and E_c inconsistently (E3): E'=[0,2,1,0], E_c=[1,2,1]."""
    g = _ex4()
    xi = GOLD["xi"]
    r = g.transforms(xi)
    np.testing.assert_allclose(g.t_of(r["T"], xi), GOLD["ect"]["T"], atol=5e-3)
    assert [0] + r["E"].tolist() == GOLD["ect"]["E"]
    np.testing.assert_allclose(g.t_of(r["To"], xi), GOLD["radon"]["T"], atol=5e-3)
    assert [0] + r["Eo"].tolist() == [-v for v in GOLD["radon"]["E_prime_printed"]]
    np.testing.assert_allclose(g.t_of(r["Tc"], xi), GOLD["radon"]["T_c"], atol=5e-3)
    assert r["Ec"].tolist() == [1, 2, 1]
    # E_c entries are the Radon values at the classical dots: check against the literal oracle
    for h, v in zip(r["Tc"], r["Ec"]):
        assert g.radon_at(xi, 2 * int(h)) == int(v)


def test_appendix_ht_exp():
    """P:334 'HT ~ -4.715' (kbar = exp); E1: the true sign is +. Closed form
    e^{2/3} + e^{4/3} - 2 e^{-2/3} from the Radon step function above."""
    g = _ex4()
    closed = math.exp(2 / 3) + math.exp(4 / 3) - 2 * math.exp(-2 / 3)
    q = g.ht_quad(GOLD["xi"], "exp")
    c = g.ht_cells(GOLD["xi"], "exp")
    assert abs(q - closed) <= 1e-13 * closed
    assert abs(c - closed) <= 1e-13 * closed
    assert abs(abs(q) - abs(GOLD["ht_exp"]["printed"])) < 5e-4


def test_appendix_evaluation_vectorisation():
    """P:337 ECT(xi,-0.3)=3, ECT(xi,1)=2; P:341 vectorisation [1,1,2,2,2]."""
    g = _ex4()
    xi = GOLD["xi"]
    r = g.transforms(xi)
    to_h = lambda t: g.L * (t + g.csum(xi) / 2)  # inverse of t = H/L - csum/2
    for t, v in GOLD["evaluate"]["ect_at"]:
        assert evaluate_ect(r["T"], r["E"], to_h(t)) == v
    vz = GOLD["vectorize"]
    ts = [vz["a"] + i * (vz["b"] - vz["a"]) / (vz["N"] - 1) for i in range(vz["N"])]
    assert [evaluate_ect(r["T"], r["E"], to_h(t)) for t in ts] == vz["values"]


# ----------------------------------------------------------------------------- quadrature

@pytest.mark.parametrize("kernel,param", [("gauss", 1.0), ("cos", 64.0), ("sin", 1.0), ("exp", 1.0), ("one", 1.0)])
def test_quadrature_matches_primitive(kernel, param):
    """The definition HT = int kappa Radon dt, integrated numerically, equals the
    cell-primitive form of corrected Lemma 1 (E2) to 1e-12: pins GL nodes/weights,
    kappa/kbar pairs and the t map."""
    rng = np.random.default_rng(7)
    for trial in range(6):
        shape = (5, 6) if trial % 2 == 0 else (3, 4, 3)
        img = rng.integers(-2, 5, size=shape)
        g = oracle.Grid(img, "vertex" if trial % 3 else "top")
        xi = synth.random_directions(1, len(shape), 5, 100 + trial)[0]
        q = g.ht_quad(xi, kernel, param, nsub=2)
        c = g.ht_cells(xi, kernel, param)
        assert abs(q - c) <= 1e-12 * max(1.0, abs(c)), (q, c)


def test_ht_single_edge_unit_kernel():
    """single value-1 edge, kappa = 1 -> HT = t_b - t_a."""
    img = np.array([[1, 1]], dtype=np.int32)  # vertex construction: one edge along axis 1
    g = oracle.Grid(img, "vertex")
    for xi in ([3, 2], [-1, -5], [2, -7]):
        ta, tb = sorted([g.t_of(0, xi) + 0.0, g.t_of(g.xs(xi)[1], xi) + 0.0])
        assert g.ht_quad(xi, "one") == pytest.approx(tb - ta, abs=1e-15)


# ----------------------------------------------------------------------------- closed forms

@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_constant_image(construction):
    """Constant image w: ECT = w 1[t >= h_min]; Radon = w on [h_min, h_max];
    HT = w (kbar(t_max) - kbar(t_min)) (SURVEY §8(c) pins; the complex is a
    contractible cube of weight w)."""
    for shape in [(4, 5), (3, 3, 2)]:
        w = 3
        g = oracle.Grid(np.full(shape, w), construction)
        assert g.euler() == w
        for xi in synth.random_directions(4, len(shape), 6, 11):
            lo, hi = g.height_range(xi)
            r = g.transforms(xi)
            assert r["T"].tolist() == [lo] and r["E"].tolist() == [w]
            assert r["To"].tolist() == [lo, hi] and r["Eo"].tolist() == [w, 0]
            assert r["Tc"].tolist() == [lo] and r["Ec"].tolist() == [w]
            kb = lambda t: math.sqrt(math.pi / 2) * math.erf(t / math.sqrt(2))
            want = w * (kb(g.t_of(hi, xi)) - kb(g.t_of(lo, xi)))
            assert g.ht_quad(xi, "gauss", 1.0) == pytest.approx(want, rel=1e-12, abs=1e-14)


def test_single_cube_chi():
    """A single pixel/voxel with weight 1 (top construction) has chi = 1 for the closed cube."""
    for shape in [(1, 1), (1, 1, 1)]:
        assert oracle.Grid(np.ones(shape), "top").euler() == 1
    # all-ones vertex image: contractible full grid
    assert oracle.Grid(np.ones((4, 6)), "vertex").euler() == 1


@pytest.mark.parametrize("construction", ["vertex", "top"])
@pytest.mark.parametrize("m", [40, 60])
def test_squares_counts(construction, m):
    """periodic squares pattern -> 100 classical and 200 ordinary critical
    points for every sign vector, independent of m."""
    img = synth.squares_image(m, 10, 3)
    if construction == "top":
        # top construction: squares must not touch the image border (a border face
        # keeps weight 1, an interior boundary face gets min = 0), so pad by one pixel
        img = np.pad(img, 1)
    g = oracle.Grid(img, construction)
    for e in range(4):
        c, dm, o, j = g.critical_table(e)
        assert (len(c), len(o)) == (100, 200)


# ----------------------------------------------------------------------------- invariants

def _rand_cases(n_cases, seed, dims=(2, 3), wlo=-2, whi=5, maxext=5):
    rng = np.random.default_rng(seed)
    for k in range(n_cases):
        n = dims[k % len(dims)]
        shape = tuple(int(x) for x in rng.integers(1, maxext + 1, size=n))
        img = rng.integers(wlo, whi + 1, size=shape)
        construction = "vertex" if k % 2 == 0 else "top"
        dirs = synth.random_directions(3, n, 4, seed * 1000 + k)
        yield oracle.Grid(img, construction), dirs


def test_star_invariants():
    """sum_x Delta^-(eps,x) = chi; sum_x J = 0; J(-eps) = -J(eps) (upper and
    lower stars swap)."""
    for g, _ in _rand_cases(60, 3):
        chi = g.euler()
        full = (1 << g.n) - 1
        for e in range(1 << g.n):
            dm, ep = g.critical(e)
            dm2, ep2 = g.critical(full ^ e)
            assert dm.sum() == chi
            assert (dm - ep).sum() == 0
            np.testing.assert_array_equal(ep, dm2)  # upst(eps) = lwst(-eps)


def test_literal_equals_swept_and_limits():
    """The literal per-threshold scans equal the swept canonical arrays at every doubled
    height; ECT(-inf) = 0, ECT(+inf) = chi, Radon = 0 outside [h_min, h_max]."""
    for g, dirs in _rand_cases(40, 5, maxext=4):
        chi = g.euler()
        for xi in dirs:
            lo, hi = g.height_range(xi)
            r = g.transforms(xi)
            for t2 in range(2 * lo - 2, 2 * hi + 3):
                h = Fraction(t2, 2)
                assert g.ect_at(xi, t2) == evaluate_ect(r["T"], r["E"], h)
                assert g.radon_at(xi, t2) == evaluate_radon(r["To"], r["Eo"], r["Tc"], r["Ec"], h)
            assert g.ect_at(xi, 2 * lo - 1) == 0 and g.ect_at(xi, 2 * hi) == chi
            assert g.radon_at(xi, 2 * lo - 1) == 0 and g.radon_at(xi, 2 * hi + 1) == 0


def test_lemma2_agrees_with_cell_definition():
    """Lemma 2 (J sign per E1) applied to the star tables reproduces the
    canonical ECT/Radon of the cell-sum definition (Lemmas 1/4), and
    HT = -sum J kbar(t) reproduces the quadrature of the Radon curve."""
    for g, dirs in _rand_cases(80, 9):
        for xi in dirs:
            hc, dm, ho, j = critical_heights(g, xi, orthant(xi))
            want = lemma2_transforms(hc, dm, ho, j)
            got = g.transforms(xi)
            for k in want:
                np.testing.assert_array_equal(got[k], want[k], err_msg=k)
            kb = lambda t: math.sqrt(math.pi / 2) * math.erf(t / math.sqrt(2))
            ht = -math.fsum(float(jj) * kb(float(g.t_of(h, xi))) for h, jj in zip(ho, j))
            assert g.ht_quad(xi, "gauss") == pytest.approx(ht, rel=1e-11, abs=1e-12)


def test_lemma2_all_binary_4x4():
    """Brute force over binary 4x4 images (both constructions): Lemma 2 == definition."""
    rng = np.random.default_rng(0)
    codes = list(range(0, 1 << 16, 97)) + [0xFFFF, 0x8001, 0x0660]
    for code in codes:
        img = np.array([(code >> i) & 1 for i in range(16)]).reshape(4, 4)
        for construction in ("vertex", "top"):
            g = oracle.Grid(img, construction)
            xi = synth.random_directions(1, 2, 5, code)[0]
            hc, dm, ho, j = critical_heights(g, xi, orthant(xi))
            want = lemma2_transforms(hc, dm, ho, j)
            got = g.transforms(xi)
            for k in want:
                np.testing.assert_array_equal(got[k], want[k])


def test_lemma6_jump_relations():
    """Corrected Lemma 6: R(t)-R(t-) = sum Delta^- at t; R(t+)-R(t-) = sum J at t."""
    for g, dirs in _rand_cases(30, 13, maxext=4):
        for xi in dirs:
            hc, dm, ho, j = critical_heights(g, xi, orthant(xi))
            lo, hi = g.height_range(xi)
            for h in range(lo, hi + 1):
                at = g.radon_at(xi, 2 * h)
                left = g.radon_at(xi, 2 * h - 1)
                right = g.radon_at(xi, 2 * h + 1)
                assert at - left == int(dm[hc == h].sum())
                assert right - left == int(j[ho == h].sum())


def test_positive_scaling_and_axis_flip():
    """lambda xi (lambda > 0) scales breakpoints, E arrays unchanged; flipping
    axis i together with xi_i -> -xi_i leaves the transforms unchanged up to the
    height offset (an isometry of the cube)."""
    for g, dirs in _rand_cases(20, 17):
        for xi in dirs:
            r1 = g.transforms(xi)
            r3 = g.transforms(3 * np.asarray(xi))
            for k in ("T", "To", "Tc"):
                np.testing.assert_array_equal(r3[k], 3 * r1[k])
            for k in ("E", "Eo", "Ec"):
                np.testing.assert_array_equal(r3[k], r1[k])


def test_axis_flip():
    rng = np.random.default_rng(21)
    for k in range(20):
        shape = (4, 5) if k % 2 else (3, 4, 2)
        img = rng.integers(0, 4, size=shape)
        construction = "vertex" if k % 3 else "top"
        xi = synth.random_directions(1, len(shape), 5, 77 + k)[0]
        g = oracle.Grid(img, construction)
        gf = oracle.Grid(np.flip(img, axis=0).copy(), construction)
        xif = xi.copy()
        xif[0] = -xif[0]
        r, rf = g.transforms(xi), gf.transforms(xif)
        off = int(g.xs(xi)[0]) * (int(g.M[0]) - 1)  # H -> H - xs0 (M0-1) under p0 -> M0-1-p0
        for kk in ("T", "To", "Tc"):
            np.testing.assert_array_equal(rf[kk], r[kk] - off)
        for kk in ("E", "Eo", "Ec"):
            np.testing.assert_array_equal(rf[kk], r[kk])


# ----------------------------------------------------------------------------- topology

def test_ect_equals_digital_topology_layer_cake():
    """ECT(xi, t) = chi(phi_{xi<=t}). For the vertex construction with weights
    in {0..3}, phi = sum_k 1[phi >= k] and the sublevel set of each layer is the vertex
    complex of the binary image [I >= k] & [H(p) <= t]; its chi is computed by
    connected-component labelling (b0 - b1)."""
    rng = np.random.default_rng(31)
    for k in range(25):
        shape = tuple(int(x) for x in rng.integers(2, 8, size=2))
        img = rng.integers(0, 4, size=shape)
        g = oracle.Grid(img, "vertex")
        for xi in synth.random_directions(2, 2, 5, 300 + k):
            r = g.transforms(xi)
            xs = g.xs(xi)
            H = np.add.outer(np.arange(shape[0]) * xs[0], np.arange(shape[1]) * xs[1])
            lo, hi = g.height_range(xi)
            for h in range(lo - 1, hi + 1):
                want = sum(digital_euler_2d((img >= lev) & (H <= h)) for lev in range(1, 4))
                assert evaluate_ect(r["T"], r["E"], h) == want


def test_top_ect_equals_digital_topology_of_closed_complements():
    """TOP construction: a lower cell takes the min of its top cofaces, so for
    weights in {0..3} the layer {phi >= k} is the complement of Cl(B_k), the closed
    subcomplex spanned by the pixels below k, and with S_t the closed subcomplex of cells
    whose vertices all have height <= t,
        ECT(xi, t) = sum_k chi(S_t minus Cl(B_k)) = sum_k [chi(S_t) - chi(S_t & Cl(B_k))].
    Both terms are Euler characteristics of CLOSED cubical complexes, computed here by
    connected-component labelling (b0 - b1) of their cells drawn on the doubled grid
    (a cell is a point; faces are 4-neighbours; a unit square of mutually incident cells
    is filled: the cubical subdivision, same homotopy type) - no (-1)^dim sum, no min."""
    rng = np.random.default_rng(57)
    for k in range(20):
        m0, m1 = (int(x) for x in rng.integers(1, 6, size=2))
        img = rng.integers(0, 4, size=(m0, m1))
        g = oracle.Grid(img, "top")
        # doubled grid of the (m0+1) x (m1+1) vertex lattice; pixel r is the cell (2 r0 + 1, 2 r1 + 1)
        u0, u1 = np.meshgrid(np.arange(2 * m0 + 1), np.arange(2 * m1 + 1), indexing="ij")
        for xi in synth.random_directions(2, 2, 5, 900 + k):
            r = g.transforms(xi)
            xs = g.xs(xi)
            lo, hi = g.height_range(xi)
            # highest vertex of every cell: vertices floor(u/2), ceil(u/2) per axis
            hmax = sum(np.maximum(int(xs[i]) * (u // 2), int(xs[i]) * ((u + 1) // 2)) for i, u in enumerate((u0, u1)))
            for h in range(lo - 1, hi + 1):
                S = hmax <= h
                want = 0
                for lev in range(1, 4):
                    cl = np.zeros(S.shape, dtype=bool)
                    for r0, r1 in zip(*np.nonzero(img < lev)):
                        cl[2 * r0:2 * r0 + 3, 2 * r1:2 * r1 + 3] = True  # the pixel and all its faces
                    want += digital_euler_2d(S) - digital_euler_2d(S & cl)
                assert evaluate_ect(r["T"], r["E"], h) == want, (img, xi, h)


def test_radon_equals_slice_geometry():
    """Radon(xi, t) = chi(phi_{xi=t}): for binary vertex-construction images the
    slice of the subcomplex K by the line {xi = t} is a disjoint union of points and
    segments, so chi = number of its connected pieces (exact rational geometry)."""
    rng = np.random.default_rng(41)
    for k in range(12):
        shape = tuple(int(x) for x in rng.integers(2, 6, size=2))
        img = rng.integers(0, 2, size=shape)
        g = oracle.Grid(img, "vertex")
        for xi in synth.random_directions(2, 2, 4, 500 + k):
            r = g.transforms(xi)
            lo, hi = g.height_range(xi)
            for t2 in range(2 * lo - 1, 2 * hi + 2):
                want = slice_components_2d(img, g.xs(xi), Fraction(t2, 2))
                got = evaluate_radon(r["To"], r["Eo"], r["Tc"], r["Ec"], Fraction(t2, 2))
                assert got == want, (img, xi, t2)


def test_single_edge_sign_convention():
    """value-1 edge a-b (xi increasing towards b): Delta^-(a)=1, Delta^-(b)=0,
    J(a)=+1, J(b)=-1, and Radon = 1 on [t_a, t_b] (the printed Delta^ord would give -1)."""
    g = oracle.Grid(np.array([[1, 1]]), "vertex")
    xi = [1, 1]
    dm, ep = g.critical(orthant(xi))
    assert dm.tolist() == [1, 0]
    assert (dm - ep).tolist() == [1, -1]
    r = g.transforms(xi)
    assert r["To"].tolist() == [0, 1] and r["Eo"].tolist() == [1, 0]
