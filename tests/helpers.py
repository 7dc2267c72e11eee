"""Test-side helpers (no product code, no oracle arithmetic).

* ``lemma2_transforms``: ECT/Radon canonical arrays from critical tables via the
  paper's Lemma 2 (ordinary sign corrected: E1). It is a DIFFERENT
  formula from the oracle's cell sums (Lemma 1/Lemma 4), so agreement pins both.
* ``evaluate_ect`` / ``evaluate_radon``: binary-search evaluation (P:135, P:137,
  strict rule E7).
* ``digital_euler_2d``: Euler characteristic of the cubical complex of a binary
  image under the vertex construction, by connected-component labelling
  (b0 - b1 with 4-connected foreground / 8-connected background).
* ``slice_components_2d``: chi of K cap {xi = t} for the vertex-construction
  complex K of a binary image, by exact geometry (Fractions): the number of
  connected pieces of the slice.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def lemma2_transforms(heights_c, dminus, heights_o, jump):
    """Canonical (T,E), (To,Eo), (Tc,Ec) from classical (h, Delta^-) and ordinary (h, J)."""
    from collections import defaultdict

    wc = defaultdict(int)
    wj = defaultdict(int)
    key = lambda h: h.item() if hasattr(h, "item") else h  # int lattice heights or float heights (f3)
    for h, w in zip(heights_c, dminus):
        wc[key(h)] += int(w)
    for h, w in zip(heights_o, jump):
        wj[key(h)] += int(w)
    keys = sorted(set(wc) | set(wj))
    T, E, To, Eo, Tc, Ec = [], [], [], [], [], []
    e = 0
    r = 0
    for h in keys:
        if wc.get(h, 0) != 0:
            e += wc[h]
            T.append(h)
            E.append(e)
            Tc.append(h)
            Ec.append(r + wc[h])
        if wj.get(h, 0) != 0:
            r += wj[h]
            To.append(h)
            Eo.append(r)
    a = lambda x: np.array(x, dtype=np.int64)
    hdt = np.float64 if any(isinstance(k, float) for k in keys) else np.int64
    ah = lambda x: np.array(x, dtype=hdt)
    return dict(T=ah(T), E=a(E), To=ah(To), Eo=a(Eo), Tc=ah(Tc), Ec=a(Ec))


def evaluate_ect(T, E, h):
    """ECT at height h: E[i], i = number of breakpoints <= h (right-continuous)."""
    i = int(np.searchsorted(np.asarray(T), h, side="right"))
    return 0 if i == 0 else int(E[i - 1])


def evaluate_radon(To, Eo, Tc, Ec, h):
    """Radon at h: E_c if h in T_c, else E' over ordinary breakpoints strictly below h (E7)."""
    Tc = np.asarray(Tc)
    j = int(np.searchsorted(Tc, h, side="left"))
    if j < len(Tc) and Tc[j] == h:
        return int(Ec[j])
    i = int(np.searchsorted(np.asarray(To), h, side="left"))
    return 0 if i == 0 else int(Eo[i - 1])


def digital_euler_2d(b: np.ndarray) -> int:
    from scipy import ndimage

    b = np.asarray(b, dtype=bool)
    four = ndimage.generate_binary_structure(2, 1)
    eight = ndimage.generate_binary_structure(2, 2)
    _, b0 = ndimage.label(b, structure=four)
    pad = np.pad(~b, 1, constant_values=True)
    _, nbg = ndimage.label(pad, structure=eight)
    return int(b0 - (nbg - 1))


def slice_components_2d(b: np.ndarray, xs, t) -> int:
    """Number of connected components of K cap {xs0*y + xs1*x = t}, K the vertex-
    construction complex of binary image b (cells whose vertices are all 1), in
    lattice coordinates (y, x) = vertex indices; xs both nonzero; t a Fraction."""
    b = np.asarray(b, dtype=bool)
    a0, a1 = int(xs[0]), int(xs[1])
    t = Fraction(t)
    m0, m1 = b.shape
    ivs = []  # closed intervals in the x-parameter of the line

    def y_of(x):
        return (t - a1 * x) / a0

    # vertices
    for y in range(m0):
        for x in range(m1):
            if b[y, x] and a0 * y + a1 * x == t:
                ivs.append((Fraction(x), Fraction(x)))
    # edges along x (y fixed): points (y, x..x+1)
    for y in range(m0):
        for x in range(m1 - 1):
            if b[y, x] and b[y, x + 1]:
                # a0*y + a1*s = t -> s = (t - a0*y)/a1
                s = (t - a0 * y) / a1
                if x <= s <= x + 1:
                    ivs.append((s, s))
    # edges along y (x fixed)
    for y in range(m0 - 1):
        for x in range(m1):
            if b[y, x] and b[y + 1, x]:
                yy = y_of(Fraction(x))
                if y <= yy <= y + 1:
                    ivs.append((Fraction(x), Fraction(x)))
    # squares
    for y in range(m0 - 1):
        for x in range(m1 - 1):
            if b[y, x] and b[y + 1, x] and b[y, x + 1] and b[y + 1, x + 1]:
                # x-range of the line inside [x,x+1] x [y,y+1]
                lo, hi = Fraction(x), Fraction(x + 1)
                # y_of(s) in [y, y+1]: linear in s
                s_a = (t - a0 * y) / a1
                s_b = (t - a0 * (y + 1)) / a1
                lo = max(lo, min(s_a, s_b))
                hi = min(hi, max(s_a, s_b))
                if lo <= hi:
                    ivs.append((lo, hi))
    if not ivs:
        return 0
    ivs.sort()
    comps = 1
    cur_hi = ivs[0][1]
    for lo, hi in ivs[1:]:
        if lo > cur_hi:
            comps += 1
            cur_hi = hi
        else:
            cur_hi = max(cur_hi, hi)
    return comps


def critical_heights(grid, xi, e):
    """Heights (lattice units) of the orthant-e critical points of an oracle Grid."""
    c, dm, o, j = grid.critical_table(e)
    M = [int(x) for x in grid.M]
    xs = grid.xs(xi)

    def h(ids):
        coords = np.array(np.unravel_index(ids, M)).T if len(ids) else np.zeros((0, grid.n), dtype=np.int64)
        return coords.astype(np.int64) @ xs

    return h(c), dm, h(o), j


def orthant(xi) -> int:
    return int(sum(1 << i for i, v in enumerate(xi) if v > 0))
