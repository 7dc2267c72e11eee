"""NEXT row f4 on the GPU: the critical-point counts of the paper's section-5
experiments, computed by K1 (eucalc_critical_points / eucalc_critical_counts).

* P:175 "Size of images": binary m x m images of a periodic pattern of 10 x 10
  squares have exactly 100 classical and 200 ordinary critical points for every
  sign vector, independent of m — at m in {100, 1000, 2000}, both
  constructions (TOP: the pattern kept off the image border, DESIGN.md
  "Top-construction squares").
* P:263 "Average number of critical points": uniform random 2-D images; K1's
  per-orthant counts equal the oracle's star sums exactly, and the classical
  fraction is about half the vertices above 10 gray levels and lower for binary
  images (the paper prints no values, only the figure: the bounds below are
  loose readings of its sentence, the exact check is against the oracle).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_02256_b200 as eu  # noqa: E402


@pytest.mark.parametrize("construction", ["vertex", "top"])
@pytest.mark.parametrize("m", [100, 1000, 2000])
def test_squares_100_200(m, construction):
    for s in sorted({3, max(2, m // 20)}):
        img = synth.squares_image(m, 10, s)
        if construction == "top":
            img = np.pad(img, 1)
        cr = eu.critical_points(eu.build_complex(img[None], construction))
        cnt = cr.counts()[0]
        for e in range(4):
            assert tuple(cnt[e]) == (100, 200), (m, s, construction, e, cnt[e])


@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_uniform_levels_fractions(construction):
    m = 256
    fr = {}
    for levels in (2, 4, 16, 64, 256):
        img = synth.uniform_image((m, m), levels, 7000 + levels)
        cr = eu.critical_points(eu.build_complex(img[None], construction))
        cnt = cr.counts()[0]
        g = oracle.Grid(img, construction)
        nv = int(np.prod(g.M))
        for e in range(4):
            c, _, o, _ = g.critical_table(e)
            assert tuple(cnt[e]) == (len(c), len(o)), (levels, e)
        fr[levels] = (cnt[:, 0].mean() / nv, cnt[:, 1].mean() / nv)
    # about half the vertices above 10 levels; fewer for binary images
    for levels in (16, 64, 256):
        assert 0.4 <= fr[levels][0] <= 0.6, fr
    assert fr[2][0] < fr[16][0] and fr[2][1] < fr[16][1], fr
    assert 0.1 <= fr[2][0] <= 0.3, fr
