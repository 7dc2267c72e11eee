"""GPU parity of real-valued directions (K5, NEXT row f3) against the oracle's
cell sums over the double vertex heights (E22): heights and values
bit-exact."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_02256_b200 as eu  # noqa: E402


def check(images, dirs, construction, pairs=None):
    cx = eu.build_complex(np.ascontiguousarray(images), construction)
    cr = eu.critical_points(cx)
    r = eu.transforms_real(cr, dirs, share_heights=True)
    res = {k: {kk: vv.cpu().numpy() for kk, vv in v.items()} for k, v in r.items()}
    ref = oracle.transforms_real_batch(images, dirs, construction, pairs=pairs)
    D = len(dirs)
    for (b, d), want in ref.items():
        s = b * D + d
        for k, (hn, vn) in (("ect", ("T", "E")), ("ordinary", ("To", "Eo")), ("classical", ("Tc", "Ec"))):
            o = res[k]["offsets"]
            lo, hi = o[s], o[s + 1]
            np.testing.assert_array_equal(res[k]["height"][lo:hi], want[hn], err_msg=f"{k} heights b={b} d={d}")
            np.testing.assert_array_equal(res[k]["value"][lo:hi], want[vn], err_msg=f"{k} values b={b} d={d}")
    return res


def test_ex4_real():
    check(synth.EX4[None], np.array([[2.0, 2.0], [0.3, 0.7], [-1.0, 0.25]]), "vertex")


CASES = [((9, 13), 3, "vertex", 256), ((9, 13), 3, "top", 5), ((6, 7, 5), 2, "vertex", 256),
         ((5, 4, 6), 2, "top", 3), ((1, 9), 2, "vertex", 5), ((40, 40), 1, "vertex", 256)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}")
def test_real_parity(case):
    shape, batch, construction, levels = case
    rng = np.random.default_rng(abs(hash(case)) & 0xFFFF)
    images = rng.integers(0, levels, size=(batch, *shape)).astype(np.uint8)
    n = len(shape)
    dirs = np.concatenate([rng.uniform(0.0, 1.0, size=(6, n)) + 1e-3,  # the paper's [0,1]^n
                           rng.uniform(-2.0, 2.0, size=(6, n))])
    dirs[dirs == 0] = 0.5
    check(images, dirs, construction)


def test_real_config2_sample():
    """Config 2 images (fashion-MNIST stand-in) with 100 directions uniform in [0,1]^2."""
    c = synth.config_inputs(2, "gray", small=True)
    imgs = c["images"][:32]
    dirs = np.random.default_rng(1).uniform(1e-3, 1.0, size=(100, 2))
    check(imgs, dirs, "vertex", pairs=[(0, 0), (7, 33), (31, 99)] + [(b, 5) for b in range(0, 32, 4)])


def test_real_equals_integer_path_when_exact():
    """Dyadic vertex spacing and small integer directions: every dot is exact, so the
    real path reproduces the integer path at the exact paper heights t(H)."""
    rng = np.random.default_rng(9)
    images = rng.integers(0, 9, size=(3, 17, 9)).astype(np.uint8)  # M-1 = 16, 8
    dirs = synth.random_directions(7, 2, 6, 3)
    cx = eu.build_complex(images, "vertex")
    cr = eu.critical_points(cx)
    ri = eu.transforms(cr, dirs, elem_bytes=8)
    rr = eu.transforms_real(cr, dirs.astype(np.float64))
    for k in ("ect", "ordinary", "classical"):
        assert torch.equal(ri[k]["offsets"], rr[k]["offsets"])
        assert torch.equal(ri[k]["value"][: int(ri[k]["offsets"][-1])], rr[k]["value"][: int(rr[k]["offsets"][-1])])
    for s in range(images.shape[0] * len(dirs)):
        d = s % len(dirs)
        L, cs = cx.height_map(dirs[d])
        a, b = int(ri["ect"]["offsets"][s]), int(ri["ect"]["offsets"][s + 1])
        H = ri["ect"]["height"][a:b].cpu().numpy()
        np.testing.assert_array_equal(rr["ect"]["height"][a:b].cpu().numpy(), (2.0 * H - L * cs) / (2.0 * L))


def test_real_errors():
    cx = eu.build_complex(synth.blob_images(2, 28, 1), "vertex")
    cr = eu.critical_points(cx)
    with pytest.raises(eu.EucalcError) as ei:
        eu.transforms_real(cr, np.array([[0.5, 0.25], [0.0, 1.0]]))
    assert ei.value.status == eu.E_NONGENERIC and ei.value.bad_index == 1


# Bucketed path for long lists (> 4096 records; forced on smaller ones through the
# EUCALC_K5_SMALL_MAX / EUCALC_K5_BUCKET hooks): value buckets -> pieces, warp
# sorts, CTA sorts of oversize pieces (bitonic tiles of 8192 + merge passes).
BIG_CASES = [
    # (shape, levels, construction, dirs kind, bucket target)
    ((40, 40), 256, "vertex", "unit", 4),        # many small pieces, empty buckets
    ((40, 40), 256, "top", "signed", 128),       # default bucket target
    ((40, 40), 256, "vertex", "unit", 100000),   # one oversize piece (CTA bitonic)
    ((160, 160), 256, "vertex", "unit", 100000),  # oversize > 8192: merge passes
    ((65, 65), 7, "vertex", "ties", 1),          # dyadic spacing: exact ties across records
    ((65, 65), 7, "vertex", "ties", 100000),
    ((17, 17, 17), 5, "vertex", "ties", 16),
    ((9, 11, 13), 256, "top", "signed", 3),
]


@pytest.mark.parametrize("case", BIG_CASES, ids=lambda c: f"{c[0]}-{c[2]}-{c[3]}-b{c[4]}")
def test_real_bucketed_forced(case, monkeypatch):
    shape, levels, construction, kind, bucket = case
    monkeypatch.setenv("EUCALC_K5_SMALL_MAX", "0")
    monkeypatch.setenv("EUCALC_K5_BUCKET", str(bucket))
    rng = np.random.default_rng(sum(shape) + bucket)
    images = rng.integers(0, levels, size=(2, *shape)).astype(np.uint8)
    n = len(shape)
    if kind == "unit":
        dirs = rng.uniform(1e-3, 1.0, size=(4, n))
    elif kind == "signed":
        dirs = rng.uniform(-2.0, 2.0, size=(4, n))
        dirs[np.abs(dirs) < 1e-3] = 0.5
    else:  # exact ties: dyadic coordinates x = p/64 - 1/2 (or 1/16) and small dyadic directions
        dirs = np.array([[1.0] * n, [0.5] + [0.25] * (n - 1), [-1.0] + [2.0] * (n - 1), [0.75] * n])
    pairs = [(b, d) for b in range(2) for d in range(len(dirs))]
    if shape == (160, 160):
        pairs = [(0, 0), (1, 3)]
    check(images, dirs, construction, pairs=pairs)


def test_real_long_lists_default():
    """Lists over 4096 records take the bucketed path by default."""
    img = synth.uniform_image((128, 128), 256, 3)[None]
    cr = eu.critical_points(eu.build_complex(img, "vertex"))
    assert int(cr.counts().max()) > 4096
    check(img, np.array([[0.5, 0.25], [-0.3, 0.9]]), "vertex")


def test_real_config3_sampled():
    """Config 3 (2048^2 GRF, 1.75 M-record lists) with real directions: sampled pairs vs the oracle."""
    c = synth.config_inputs(3, "gray")
    img = c["images"]
    dirs = np.array([[0.61, 0.23], [-0.17, 0.94], [0.5, -0.5]])
    check(img, dirs, "vertex", pairs=[(0, 0), (0, 2)])
