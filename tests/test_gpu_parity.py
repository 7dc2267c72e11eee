"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

ECT/Radon representations and critical tables must be bit-exact (integers,
SURVEY 8(c) E18); HT within 1e-9 (fp64) / 1e-4 (fp32) relative to max(|ref|,1)
(BASELINE.json north_star). Inputs are the seeded generators of synth/.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import orthant

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_02256_b200 as eu  # noqa: E402

HT_TOL = {"f64": 1e-9, "f32": 1e-4}


def to_np(steps):
    if steps is None:
        return None
    return {k: (v.cpu().numpy().astype(np.int64) if v is not None else None) for k, v in steps.items()}


def seg(st, s):
    a, b = st["offsets"][s], st["offsets"][s + 1]
    return st["height"][a:b], st["value"][a:b]


def run_gpu(images, dirs, construction, elem_bytes=8, share=False):
    cx = eu.build_complex(np.ascontiguousarray(images), construction)
    cr = eu.critical_points(cx)
    r = eu.transforms(cr, dirs, elem_bytes=elem_bytes, share_heights=share)
    torch.cuda.synchronize()
    return cx, cr, {k: to_np(v) for k, v in r.items()}


def check_transforms(images, dirs, construction, res, pairs=None):
    D = len(dirs)
    ref = oracle.transforms_batch(images, dirs, construction, pairs=pairs)
    for (b, d), want in ref.items():
        s = b * D + d
        T, E = seg(res["ect"], s)
        np.testing.assert_array_equal(T, want["T"], err_msg=f"ECT T b={b} d={d}")
        np.testing.assert_array_equal(E, want["E"], err_msg=f"ECT E b={b} d={d}")
        To, Eo = seg(res["ordinary"], s)
        np.testing.assert_array_equal(To, want["To"], err_msg=f"Radon T_o b={b} d={d}")
        np.testing.assert_array_equal(Eo, want["Eo"], err_msg=f"Radon E' b={b} d={d}")
        Tc, Ec = seg(res["classical"], s)
        np.testing.assert_array_equal(Tc, want["Tc"], err_msg=f"Radon T_c b={b} d={d}")
        np.testing.assert_array_equal(Ec, want["Ec"], err_msg=f"Radon E_c b={b} d={d}")


def check_critical(images, construction, cr, imgs_to_check=None):
    n = images.ndim - 1
    for b in (imgs_to_check if imgs_to_check is not None else range(images.shape[0])):
        g = oracle.Grid(images[b], construction)
        for e in range(1 << n):
            v, dm, j = cr.export(b, e)
            odm, oep = g.critical(e)
            oj = odm - oep
            keep = np.nonzero((odm != 0) | (oep != 0))[0]
            np.testing.assert_array_equal(v, keep, err_msg=f"kept vertices b={b} e={e}")
            np.testing.assert_array_equal(dm, odm[keep], err_msg=f"Delta^- b={b} e={e}")
            np.testing.assert_array_equal(j, oj[keep], err_msg=f"J b={b} e={e}")


def check_ht(images, dirs, construction, cr, kernel, param, precision, pairs=None, algorithms=("auto", "direct")):
    """Both HT algorithms (per-term kbar and tabulated kbar, eucalc_hybrid_ex) vs the
    oracle's quadrature of the Radon transform."""
    ref = oracle.ht_batch(images, dirs, construction, kernel, param, pairs=pairs)
    tol = HT_TOL[precision]
    for alg in algorithms:
        out = eu.hybrid(cr, dirs, kernel, param, precision, algorithm=alg).cpu().numpy()
        for (b, d), want in ref.items():
            got = float(out[b, d])
            assert abs(got - want) <= tol * max(abs(want), 1.0), (alg, kernel, precision, b, d, got, want)


def check_fused_ht(images, dirs, construction, cr, kernel, param, precision, pairs=None, elem_bytes=8):
    """eucalc_transforms_ht (HT from K2's merged histogram, NEXT f2) vs the oracle's
    quadrature, and its representations vs eucalc_transforms."""
    r = eu.transforms(cr, dirs, elem_bytes=elem_bytes, share_heights=True, ht=(kernel, param, precision))
    out = r["ht"].cpu().numpy()
    ref = oracle.ht_batch(images, dirs, construction, kernel, param, pairs=pairs)
    tol = HT_TOL[precision]
    for (b, d), want in ref.items():
        got = float(out[b, d])
        assert abs(got - want) <= tol * max(abs(want), 1.0), ("fused", kernel, precision, b, d, got, want)
    plain = eu.transforms(cr, dirs, elem_bytes=elem_bytes, share_heights=True)
    for k in ("ect", "ordinary", "classical"):
        n = int(plain[k]["offsets"][-1])
        assert torch.equal(plain[k]["offsets"], r[k]["offsets"])
        assert torch.equal(plain[k]["value"][:n], r[k]["value"][:n])


# ----------------------------------------------------------------------------- golden

def test_ex4_golden_gpu():
    img = synth.EX4[None].astype(np.uint8)
    cx, cr, res = run_gpu(img, np.array([[2, 2]], np.int32), "vertex")
    T, E = seg(res["ect"], 0)
    assert E.tolist() == [1, 3, 2] and T.tolist() == [0, 4, 6]
    To, Eo = seg(res["ordinary"], 0)
    assert Eo.tolist() == [2, 1, 0] and To.tolist() == [4, 8, 10]
    Tc, Ec = seg(res["classical"], 0)
    assert Ec.tolist() == [1, 2, 1]
    ht = eu.hybrid(cr, np.array([[2, 2]], np.int32), "exp", 1.0, "f64").item()
    assert abs(ht - (math.exp(2 / 3) + math.exp(4 / 3) - 2 * math.exp(-2 / 3))) < 1e-12
    check_critical(img, "vertex", cr)
    assert cx.height_map([2, 2]) == (3, 4)


# ----------------------------------------------------------------------------- random small, both regimes

CASES = [
    # (shape, batch, construction, levels, dir range, ndirs)
    ((9, 13), 5, "vertex", 256, 8, 17),
    ((9, 13), 5, "top", 256, 8, 17),
    ((70, 100), 2, "vertex", 4, 6, 9),       # 4 K1 tiles, ragged last
    ((70, 100), 2, "top", 7, 6, 9),
    ((3, 2100), 1, "vertex", 256, 3, 5),     # x-split tiles
    ((6, 7, 5), 4, "vertex", 256, 5, 11),
    ((6, 7, 5), 4, "top", 3, 5, 11),
    ((10, 12, 50), 1, "vertex", 256, 4, 7),  # 10 planes -> 10 tiles
    ((1, 9), 3, "vertex", 5, 4, 6),          # degenerate axis
    ((1, 1), 2, "top", 5, 4, 3),
    ((1, 5, 1), 2, "top", 9, 3, 4),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}-{c[2]}")
def test_random_parity(case):
    shape, batch, construction, levels, k, nd = case
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    images = rng.integers(0, levels, size=(batch, *shape)).astype(np.uint8)
    dirs = synth.random_directions(nd, len(shape), k, 99)
    cx, cr, res = run_gpu(images, dirs, construction)
    check_critical(images, construction, cr)
    check_transforms(images, dirs, construction, res)
    check_ht(images, dirs, construction, cr, "gauss", 1.0, "f64")
    check_ht(images, dirs, construction, cr, "cos", 64.0, "f32")
    check_fused_ht(images, dirs, construction, cr, "sin", 1.0, "f64")
    check_fused_ht(images, dirs, construction, cr, "gauss", 1.0, "f32")


def test_block_regime_multiwindow():
    """Large height range -> one CTA per segment, several 26624-bin windows."""
    img = synth.grf_image(160, 5)[None]
    dirs = np.concatenate([synth.random_directions(6, 2, 90, 5), np.array([[90, -89], [-90, 90]], np.int32)])
    cx, cr, res = run_gpu(img, dirs, "vertex")
    check_transforms(img, dirs, "vertex", res)
    check_fused_ht(img, dirs, "vertex", cr, "cos", 7.5, "f64", pairs=[(0, 0), (0, 6), (0, 7)])


def test_block_regime_span_runs_and_tile_fallback():
    """Multi-window 2-D segments: the span fill streams maximal runs of consecutive hit
    tiles (a tall narrow image: runs cross tile rows; small windows forced by large
    directions), and images with more than 2048 K1 tiles take the per-tile culled path;
    8- and 4-byte outputs."""
    # 3073 x 97 vertices: L = 3072, xs = (xi_0, 32 xi_1), 4 x 49 tiles
    tall = np.ascontiguousarray(np.tile(synth.grf_image(256, 11), (13, 1))[:3073, :97])[None]
    dirs = np.array([[20, -3], [-33, 2], [18, 3], [-1, -1], [64, 1], [127, -3]], np.int32)
    for eb in (8, 4):
        _, _, res = run_gpu(tall, dirs, "vertex", elem_bytes=eb)
        check_transforms(tall, dirs, "vertex", res)
    big = np.ascontiguousarray(np.tile(synth.grf_image(528, 12), (4, 4)))[None]  # 2112 x 2112: 66 x 33 tiles
    d2 = np.array([[40, -37], [-3, 2]], np.int32)
    _, _, res = run_gpu(big, d2, "vertex", elem_bytes=4)
    check_transforms(big, d2, "vertex", res)


def test_block_regime_3d_culled_windows():
    """3-D, several K1 tiles (16x16x8 boxes) and height windows -> tile culling."""
    vol = synth.smooth_volume(40, 77)[None]
    dirs = np.concatenate([synth.random_directions(3, 3, 400, 12), np.array([[400, -399, 398]], np.int32)])
    cx, cr, res = run_gpu(vol, dirs, "vertex")
    check_transforms(vol, dirs, "vertex", res)


@pytest.mark.parametrize("env", [{}, {"EUCALC_K2_CHK_BITS": "1"}, {"EUCALC_K2_CHK_BITS": "6"},
                                 {"EUCALC_K2_NO_CHK": "1"}, {"EUCALC_K2_UNIT": "0"},
                                 {"EUCALC_K2_UNIT": "0", "EUCALC_K2_CHK_BITS": "1"},
                                 {"EUCALC_K2_UNIT": "0", "EUCALC_K2_SLOTS": "0"},
                                 {"EUCALC_K2_UNIT": "0", "EUCALC_K2_SLOTS": "0", "EUCALC_K2_CHK_BITS": "1"}],
                         ids=["checked", "restart", "partial", "split", "per-segment", "per-segment-restart",
                              "per-segment-lookback", "per-segment-lookback-restart"])
def test_block_regime_checked_packed_bins(env, monkeypatch):
    """Block regime with packed 16+16 bins whose exactness no bound proves: every
    add is checked and a flagged segment restarts with split bins. The test hooks
    narrow the checked range (bits 1: every segment restarts; bits 6: some do) or
    disable the packed path; all must give the oracle's exact representations. 3-D
    lists go through the unit path (several directions per pass over a list, a
    flagged unit redoes each of its directions with split bins) unless
    EUCALC_K2_UNIT=0 selects one CTA per segment."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    eu.k2_restarts(reset=True)
    vol = synth.smooth_volume(64, 78)[None]
    # small coordinates: many vertices per height level, so no bound proves the packed bins
    dirs = np.array([[1, 1, 1], [2, -1, 3], [-1, 2, 1], [3, -2, -1], [1, -1, 2], [-2, -3, -1]], np.int32)
    cx, cr, res = run_gpu(vol, dirs, "vertex")
    check_transforms(vol, dirs, "vertex", res)
    if env.get("EUCALC_K2_CHK_BITS") == "1":  # every unproven segment restarted
        assert eu.k2_restarts() == len(dirs)
    img = np.stack([synth.grf_image(160, 6), 255 - synth.grf_image(160, 7)])
    d2 = np.concatenate([synth.random_directions(4, 2, 90, 6), np.array([[90, -89]], np.int32)])
    cx, cr, res = run_gpu(img, d2, "top")
    check_transforms(img, d2, "top", res)


@pytest.mark.parametrize("restart", [False, True], ids=["packed", "restart-split"])
def test_block_regime_slot_mode(restart, monkeypatch):
    """Block regime with >= 2 x SMs segments: every segment staged in its own slot, offsets
    by k2_scan, entries moved by k2_unit_copy (no look-back); against the oracle on sampled
    segments and identical to the look-back path on all of them, also when every segment
    restarts with split bins (two windows)."""
    if restart:
        monkeypatch.setenv("EUCALC_K2_CHK_BITS", "1")
    img = np.stack([synth.grf_image(160, 21), 255 - synth.grf_image(160, 22)])
    dirs = synth.random_directions(200, 2, 90, 23)
    _, _, res = run_gpu(img, dirs, "vertex", elem_bytes=4)
    check_transforms(img, dirs, "vertex", res, pairs=[(b, d) for b in (0, 1) for d in (0, 57, 199)])
    monkeypatch.setenv("EUCALC_K2_SLOTS", "0")
    _, _, res0 = run_gpu(img, dirs, "vertex", elem_bytes=4)
    same_streams(res, res0)


def same_streams(x, y):
    for k in x:
        np.testing.assert_array_equal(x[k]["offsets"], y[k]["offsets"])
        n = x[k]["offsets"][-1]
        np.testing.assert_array_equal(x[k]["height"][:n], y[k]["height"][:n])
        np.testing.assert_array_equal(x[k]["value"][:n], y[k]["value"][:n])


def test_unit_path_image_order_and_balanced_units(monkeypatch):
    """3-D unit path: a batch whose images differ in list size (tickets run image-major,
    heaviest image first, the light image listed first here) and a single image with more
    units than SMs (units balanced over the SMs: 3 and 4 directions per unit), against the
    oracle; and the interleaved / unbalanced plans give identical outputs."""
    vol = synth.smooth_volume(64, 81)
    batch = np.stack([(vol > np.median(vol)).astype(np.uint8), vol])
    dirs, _ = synth.fibonacci_directions(40, 12.0)
    _, _, res = run_gpu(batch, dirs, "vertex", elem_bytes=4)
    check_transforms(batch, dirs, "vertex", res, pairs=[(b, d) for b in (0, 1) for d in (0, 7, 19, 39)])
    monkeypatch.setenv("EUCALC_K2_IMG_ORDER", "0")
    _, _, res0 = run_gpu(batch, dirs, "vertex", elem_bytes=4)
    same_streams(res, res0)
    many, _ = synth.fibonacci_directions(700, 12.0)  # 175 units of 4 > 148 SMs
    one = vol[None]
    _, _, resb = run_gpu(one, many, "vertex", elem_bytes=4)
    check_transforms(one, many, "vertex", resb, pairs=[(0, d) for d in (0, 1, 350, 698, 699)])
    monkeypatch.setenv("EUCALC_K2_UNIT_BALANCE", "0")
    _, _, resu = run_gpu(one, many, "vertex", elem_bytes=4)
    same_streams(resb, resu)


def test_negative_and_int32_weights():
    rng = np.random.default_rng(3)
    images = rng.integers(-40000, 40000, size=(2, 12, 11)).astype(np.int32)
    dirs = synth.random_directions(5, 2, 5, 8)
    for construction in ("vertex", "top"):
        cx, cr, res = run_gpu(images, dirs, construction)
        check_critical(images, construction, cr)
        check_transforms(images, dirs, construction, res)
        check_ht(images, dirs, construction, cr, "sin", 1.0, "f64")


@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("kernel,param", [("gauss", 1.0), ("cos", 64.0), ("sin", 1.0), ("exp", 1.0), ("cos", 7.5)])
def test_ht_kernels(kernel, param, precision):
    vols = np.stack([synth.smooth_volume(12, 1500 + j) for j in range(2)])
    dirs, _ = synth.fibonacci_directions(40, 8.0)
    cx = eu.build_complex(vols, "vertex")
    cr = eu.critical_points(cx)
    check_ht(vols, dirs, "vertex", cr, kernel, param, precision, algorithms=("direct", "table"))


# ----------------------------------------------------------------------------- ABI behaviour

def test_output_widths_and_shared_heights():
    images = synth.blob_images(6, 28, 1)
    dirs = synth.random_directions(20, 2, 16, 3)
    _, _, r8 = run_gpu(images, dirs, "vertex", elem_bytes=8)
    for eb in (4, 2):
        _, _, r4 = run_gpu(images, dirs, "vertex", elem_bytes=eb, share=True)
        for k in ("ect", "ordinary", "classical"):
            S = images.shape[0] * len(dirs)
            np.testing.assert_array_equal(r8[k]["offsets"], r4[k]["offsets"])
            n = r8[k]["offsets"][S]
            np.testing.assert_array_equal(r8[k]["height"][:n], r4[k]["height"][:n])
            np.testing.assert_array_equal(r8[k]["value"][:n], r4[k]["value"][:n])
    # int16 must be refused when values cannot fit
    big = (np.random.default_rng(1).integers(0, 30000, size=(2, 28, 28))).astype(np.int32)
    cx = eu.build_complex(big, "vertex")
    cr = eu.critical_points(cx)
    with pytest.raises(eu.EucalcError) as ei:
        eu.transforms(cr, dirs, elem_bytes=2)
    assert ei.value.status == eu.E_RANGE
    r = eu.transforms(cr, dirs, elem_bytes="auto")
    assert r["ect"]["value"].element_size() == 4


@pytest.mark.parametrize("chunks,dchunks", [("1", None), ("3", None), (None, None), ("8", "3"), (None, "16")],
                         ids=["plain", "3-chunks", "default-chunks", "image-and-3-direction-chunks",
                              "one-direction-per-chunk"])
def test_host_buffers_match_device(chunks, dchunks, monkeypatch):
    """Host outputs (copied back chunk by chunk of images, and of direction ranges of
    single-image chunks, while the next chunks compute, offsets shifted on the host;
    EUCALC_HOST_CHUNKS=1: one pass) equal the device outputs, with and without shared
    classical heights and the fused HT, in 2-D (warp regime) and 3-D (unit path), for a
    batch and for a single image."""
    if chunks:
        monkeypatch.setenv("EUCALC_HOST_CHUNKS", chunks)
    if dchunks:
        monkeypatch.setenv("EUCALC_HOST_DIR_CHUNKS", dchunks)
    vol = synth.smooth_volume(40, 93)
    cases = [(synth.blob_images(8, 28, 2), synth.random_directions(16, 2, 16, 4)),
             (np.stack([vol, (vol > np.median(vol)).astype(np.uint8), vol[::-1].copy()]),
              synth.random_directions(9, 3, 20, 6)),
             (vol[None], synth.random_directions(11, 3, 20, 7))]
    for images, dirs in cases:
        cx = eu.build_complex(images, "vertex")
        cr = eu.critical_points(cx)
        S = images.shape[0] * len(dirs)
        for share in (False, True):
            dev = eu.transforms(cr, dirs, device="cuda", share_heights=share, ht=("gauss", 1.0, "f64"))
            host = eu.transforms(cr, dirs, device="cpu", share_heights=share, ht=("gauss", 1.0, "f64"))
            np.testing.assert_array_equal(dev.pop("ht").cpu().numpy(), host.pop("ht").numpy())
            dev = {k: to_np(v) for k, v in dev.items()}
            host = {k: to_np(v) for k, v in host.items()}
            for k in dev:
                n = dev[k]["offsets"][S]
                np.testing.assert_array_equal(dev[k]["offsets"], host[k]["offsets"])
                np.testing.assert_array_equal(dev[k]["value"][:n], host[k]["value"][:n])
                np.testing.assert_array_equal(dev[k]["height"][:n], host[k]["height"][:n])
    images, dirs = cases[0]
    cx = eu.build_complex(images, "vertex")
    cr = eu.critical_points(cx)
    hd = eu.hybrid(cr, dirs, "gauss", 1.0, "f64", device="cuda").cpu().numpy()
    hh = eu.hybrid(cr, dirs, "gauss", 1.0, "f64", device="cpu").numpy()
    np.testing.assert_array_equal(hd, hh)


def test_determinism():
    vols = np.stack([synth.smooth_volume(20, 7 + j) for j in range(2)])
    dirs, _ = synth.fibonacci_directions(64, 8.0)
    outs = []
    for _ in range(2):
        cx = eu.build_complex(vols, "vertex")
        cr = eu.critical_points(cx)
        r = {k: to_np(v) for k, v in eu.transforms(cr, dirs).items()}
        h = eu.hybrid(cr, dirs, "cos", 64.0, "f32").cpu().numpy()
        outs.append((r, h))
    (r1, h1), (r2, h2) = outs
    for k in r1:
        for kk in ("offsets", "height", "value"):
            n = r1[k]["offsets"][-1]
            np.testing.assert_array_equal(r1[k][kk][:n] if kk != "offsets" else r1[k][kk],
                                          r2[k][kk][:n] if kk != "offsets" else r2[k][kk])
    assert h1.tobytes() == h2.tobytes()


def test_errors():
    images = synth.blob_images(2, 28, 3)
    cx = eu.build_complex(images, "vertex")
    cr = eu.critical_points(cx)
    bad = np.array([[1, 2], [3, 0], [0, 1]], np.int32)
    with pytest.raises(eu.EucalcError) as ei:
        eu.transforms(cr, bad)
    assert ei.value.status == eu.E_NONGENERIC and ei.value.bad_index == 1
    with pytest.raises(eu.EucalcError) as ei:
        eu.hybrid(cr, bad)
    assert ei.value.status == eu.E_NONGENERIC
    # capacity: hand the ABI a too-small buffer
    import ctypes
    dirs = np.array([[1, 2], [3, -1]], np.int32)
    off = torch.zeros(5, dtype=torch.int64, device="cuda")
    h = torch.zeros(4, dtype=torch.int64, device="cuda")
    v = torch.zeros(4, dtype=torch.int64, device="cuda")
    st = eu._Steps(off.data_ptr(), h.data_ptr(), v.data_ptr(), 4, 8, 0)
    req = ctypes.c_int64()
    rc = eu.lib().eucalc_ect(cr._h, dirs.ctypes.data_as(ctypes.c_void_p), 2, ctypes.byref(st), ctypes.byref(req),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == eu.E_CAPACITY and req.value == cr.output_bound(dirs)[0] > 4
    with pytest.raises(eu.EucalcError) as ei:
        eu.build_complex(np.zeros((1, 4, 4, 4, 4), np.uint8))
    assert ei.value.status == eu.E_ARG


def test_counts_match_oracle():
    images = synth.blob_images(4, 28, 9)
    cx = eu.build_complex(images, "vertex")
    cr = eu.critical_points(cx)
    cnt = cr.counts()
    for b in range(4):
        g = oracle.Grid(images[b], "vertex")
        for e in range(4):
            c, _, o, _ = g.critical_table(e)
            assert tuple(cnt[b, e]) == (len(c), len(o))


# ----------------------------------------------------------------------------- BASELINE configs

def test_config1_full():
    c = synth.config_inputs(1)
    _, cr, res = run_gpu(c["images"], c["dirs"], c["construction"])
    check_critical(c["images"], c["construction"], cr)
    check_transforms(c["images"], c["dirs"], c["construction"], res)


@pytest.mark.parametrize("variant", ["gray", "binary"])
@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_config2_small_full(variant, construction):
    c = synth.config_inputs(2, variant, small=True)
    imgs, dirs = c["images"][:16], c["dirs"]
    _, cr, res = run_gpu(imgs, dirs, construction)
    check_transforms(imgs, dirs, construction, res)
    check_critical(imgs, construction, cr, imgs_to_check=range(4))
    check_fused_ht(imgs, dirs, construction, cr, "sin", 1.0, "f64", pairs=[(0, 0), (3, 17), (15, 255)], elem_bytes=2)


def test_config2_full_size_sampled():
    """Full config 2 (1024 images x 256 directions) in the bench's launch
    configuration; a seeded sample of (image, direction) segments vs the oracle."""
    c = synth.config_inputs(2, "gray")
    imgs, dirs = c["images"], c["dirs"]
    _, cr, res = run_gpu(imgs, dirs, "vertex", elem_bytes=4, share=True)
    rng = np.random.default_rng(0)
    pairs = [(int(b), int(d)) for b, d in zip(rng.integers(0, 1024, 300), rng.integers(0, 256, 300))]
    pairs += [(0, 0), (1023, 255)]
    check_transforms(imgs, dirs, "vertex", res, pairs=pairs)
    check_fused_ht(imgs, dirs, "vertex", cr, "sin", 1.0, "f64", pairs=pairs[:40], elem_bytes=4)


def _squares_image(m, k, rng, value=255):
    img = np.zeros((m, m), np.uint8)
    for _ in range(k):
        y, x = rng.integers(1, m - 4, 2)
        img[y:y + 3, x:x + 3] = value
    return img


@pytest.mark.parametrize("with_gray", [False, True])
def test_sparse_lists_register_sort(with_gray):
    """K2's register sort path (lists of <= 32 records: 8-, 16- and 32-lane
    networks) next to histogram segments, with the packed 16+16 prefix sums
    (every list's sum |a|+|b| < 2^15) and without (a uniform gray image in the
    batch lifts the bound)."""
    rng = np.random.default_rng(77)
    imgs = [_squares_image(40, k, rng) for k in (0, 1, 2, 3, 5, 8, 12, 30)]
    if with_gray:
        imgs.append(rng.integers(0, 256, (40, 40)).astype(np.uint8))
    imgs = np.stack(imgs)
    dirs = synth.random_directions(48, 2, 16, 78)
    cx, cr, res = run_gpu(imgs, dirs, "vertex")
    L = cr.list_lengths()
    assert (L <= 8).any() and ((L > 8) & (L <= 16)).any() and ((L > 16) & (L <= 32)).any() and (L > 32).any(), L
    check_transforms(imgs, dirs, "vertex", res)
    check_fused_ht(imgs, dirs, "vertex", cr, "gauss", 1.0, "f64", elem_bytes=8)


def test_config2_binary_full_size_bench_launch():
    """Full config-2 binary batch in bench.py's launch (narrowest width, shared
    heights, fused HT): sampled segments vs the oracle."""
    c = synth.config_inputs(2, "binary")
    imgs, dirs = c["images"], c["dirs"]
    cx = eu.build_complex(imgs, "vertex")
    cr = eu.critical_points(cx)
    r = eu.transforms(cr, dirs, elem_bytes="auto", share_heights=True, ht=("sin", 1.0, "f64"))
    torch.cuda.synchronize()
    assert r["ect"]["value"].element_size() == 2
    ht = r.pop("ht").cpu().numpy()
    res = {k: to_np(v) for k, v in r.items()}
    rng = np.random.default_rng(5)
    pairs = [(int(b), int(d)) for b, d in zip(rng.integers(0, 1024, 300), rng.integers(0, 256, 300))]
    pairs += [(0, 0), (1023, 255)]
    check_transforms(imgs, dirs, "vertex", res, pairs=pairs)
    ref = oracle.ht_batch(imgs, dirs, "vertex", "sin", 1.0, pairs=pairs[:60])
    for (b, d), want in ref.items():
        assert abs(float(ht[b, d]) - want) <= 1e-9 * max(abs(want), 1.0), (b, d)


def test_capacity_upper_bound_matches_tight():
    """eucalc_output_bound_upper (no K1 result needed) bounds eucalc_output_bound,
    and outputs sized by either are identical."""
    c = synth.config_inputs(2, "gray", small=True)
    imgs, dirs = c["images"][:8], c["dirs"][:40]
    cx = eu.build_complex(imgs, "vertex")
    cr = eu.critical_points(cx)
    bu = ctypes_bound_upper(cx, dirs)
    bt = cr.output_bound(dirs)[0]
    assert bu >= bt > 0
    a = eu.transforms(cr, dirs, elem_bytes=2, share_heights=True, capacity="tight", ht=("sin", 1.0, "f64"))
    b = eu.transforms(cr, dirs, elem_bytes=2, share_heights=True, capacity="upper", ht=("sin", 1.0, "f64"))
    assert a["ect"]["value"].numel() == max(bt, 1) and b["ect"]["value"].numel() == max(bu, 1)
    assert torch.equal(a["ht"], b["ht"])
    for k in ("ect", "ordinary", "classical"):
        n = int(a[k]["offsets"][-1])
        assert torch.equal(a[k]["offsets"], b[k]["offsets"])
        assert torch.equal(a[k]["value"][:n], b[k]["value"][:n])
        assert torch.equal(a[k]["height"][:n], b[k]["height"][:n])


def ctypes_bound_upper(cx, dirs):
    import ctypes

    d = np.ascontiguousarray(dirs, dtype=np.int32)
    bu = ctypes.c_int64()
    assert eu.lib().eucalc_output_bound_upper(cx._h, ctypes.c_void_p(d.ctypes.data), len(d), ctypes.byref(bu),
                                              None) == 0
    return bu.value


def test_config3_sampled():
    c = synth.config_inputs(3)
    img, dirs = c["images"], c["dirs"][:64]
    _, cr, res = run_gpu(img, dirs, "vertex")
    check_transforms(img, dirs, "vertex", res, pairs=[(0, d) for d in (0, 17, 63)])
    check_critical(img, "vertex", cr)


def test_config4_sampled():
    c = synth.config_inputs(4)
    img, dirs = c["images"], c["dirs"][:48]
    _, cr, res = run_gpu(img, dirs, "vertex")
    check_transforms(img, dirs, "vertex", res, pairs=[(0, 0), (0, 31)])


@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_k1_3d_full_and_ragged_tiles(construction):
    """3-D K1 tables on a volume with full 16x16 xy tiles (VERTEX 8-bit: the z-column
    walk that carries shared planes) and ragged ones (per-vertex stencil), both
    binary and gray, against the oracle's star sums."""
    vol = synth.smooth_volume(48, 91)[:37, :40, :48]
    imgs = np.stack([vol, (vol > np.median(vol)).astype(np.uint8)])
    _, cr, _ = run_gpu(imgs, synth.random_directions(2, 3, 5, 4), construction)
    check_critical(imgs, construction, cr)


def test_config5_sampled():
    c = synth.config_inputs(5)
    vols, dirs = c["images"][:2], c["dirs"]
    cx = eu.build_complex(vols, "vertex")
    cr = eu.critical_points(cx)
    pairs = [(0, 0), (1, 4999), (0, 9999)]
    for kernel, param in (("gauss", 1.0), ("cos", 64.0)):
        for precision in ("f64", "f32"):
            check_ht(vols, dirs, "vertex", cr, kernel, param, precision, pairs=pairs, algorithms=("direct", "table"))


@pytest.mark.parametrize("construction", ["vertex", "top"])
def test_degenerate_images(construction):
    """All-zero images (no critical points: empty lists and empty segments), constant
    images (closed forms) and a 1x1 image, through K1-K4 and the fused HT."""
    imgs = np.stack([np.zeros((9, 7), np.uint8), np.full((9, 7), 5, np.uint8), np.eye(9, 7, dtype=np.uint8)])
    dirs = synth.random_directions(6, 2, 4, 17)
    cx, cr, res = run_gpu(imgs, dirs, construction)
    check_transforms(imgs, dirs, construction, res)
    assert cr.list_lengths()[0].tolist() == [0, 0]
    for s in range(len(dirs)):  # the zero image has empty segments in every stream
        for k in ("ect", "ordinary", "classical"):
            assert res[k]["offsets"][s + 1] == res[k]["offsets"][s]
    check_fused_ht(imgs, dirs, construction, cr, "gauss", 1.0, "f64")
    check_ht(imgs, dirs, construction, cr, "exp", 1.0, "f64")
    r = eu.transforms(cr, dirs)
    v = eu.vectorize(cx, dirs, -1.0, 1.0, 7, ect=r["ect"]).cpu().numpy()
    assert not v[: len(dirs)].any()  # zero image: ECT identically 0
    one = np.array([[[3]]], np.uint8)
    cx1, cr1, r1 = run_gpu(one, np.array([[1, 1]], np.int32), construction)
    check_transforms(one, np.array([[1, 1]], np.int32), construction, r1)


K1_GEOMETRY_CASES = [
    # 3-D: several 64-plane walk chunks, rows not a multiple of 8, x not a multiple of 32
    ((150, 20, 70), np.uint8, "vertex"), ((150, 20, 70), np.uint8, "top"),
    ((70, 9, 33), np.int16, "vertex"), ((66, 9, 31), np.int32, "top"),
    ((65, 17, 40), np.int32, "vertex"),
    # 3-D 8-bit VERTEX (two vertices per lane, 64-wide tiles): odd x extent (byte
    # loads), an odd number of planes (odd walk tail), x = 64 exactly, x < 32
    ((37, 29, 131), np.uint8, "vertex"), ((9, 5, 64), np.uint8, "vertex"), ((200, 3, 2), np.uint8, "vertex"),
    ((23, 8, 1), np.uint8, "vertex"),
    # 2-D: several 64-row tiles and 32-wide column blocks, ragged both ways
    ((130, 100), np.uint8, "vertex"), ((130, 100), np.uint8, "top"), ((129, 65), np.int16, "top"),
    ((200, 33), np.int32, "vertex"),
]


@pytest.mark.parametrize("case", K1_GEOMETRY_CASES, ids=lambda c: f"{c[0]}-{np.dtype(c[1]).name}-{c[2]}")
def test_k1_pencil_geometry(case):
    """K1's pencils (32 vertices per warp, walking the slowest axis in 64-plane
    chunks in 3-D / 64-row tiles in 2-D) on extents that are not multiples of the
    tile: critical tables vs the oracle's star sums, the per-orthant counts, and
    transforms (K2 culls by the K1 tile offsets) on a few directions."""
    shape, dt, construction = case
    rng = np.random.default_rng(sum(shape))
    lo, hi = (0, 256) if dt == np.uint8 else (-300, 300)
    images = rng.integers(lo, hi, size=(2, *shape)).astype(dt)
    dirs = np.concatenate([synth.random_directions(4, len(shape), 7, 3),
                           synth.random_directions(2, len(shape), 300, 5)])
    cx, cr, res = run_gpu(images, dirs, construction)
    check_critical(images, construction, cr, imgs_to_check=[1])
    check_transforms(images, dirs, construction, res, pairs=[(0, 0), (1, 3), (1, 4), (0, 5)])
    cnt = cr.counts()
    g = oracle.Grid(images[1], construction)
    for e in range(1 << len(shape)):
        c, _, o, _ = g.critical_table(e)
        assert tuple(cnt[1, e]) == (len(c), len(o))
