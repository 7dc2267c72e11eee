"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no cells, stars, heights or
transforms): it only draws images and integer directions with numpy PCG64
(``np.random.default_rng(seed)``), following the recipes of SURVEY.md §8(d)
for the five BASELINE.json configs (BJ:7-11) and the paper's own synthetic
workloads (periodic squares, P:175 / S:396-404; uniform images).

Every function is a pure function of its arguments (seed included).
"""
from __future__ import annotations

import math

import numpy as np

# Seeds of SURVEY.md §8(d): image seed 1000+k, direction seed 2000+k for config k;
# volume j of config 5 uses seed 1500+j.
IMAGE_SEED = {k: 1000 + k for k in range(1, 6)}
DIR_SEED = {k: 2000 + k for k in range(1, 6)}


# --------------------------------------------------------------------------- directions

def random_directions(count: int, n: int, k: int, seed: int) -> np.ndarray:
    """``count`` integer directions, each coordinate uniform on [-k, k] \\ {0}.

    Genericity needs every coordinate nonzero, hence the excluded 0
    (SURVEY.md §8(c) E13). Returns int32 [count, n].
    """
    rng = np.random.default_rng(seed)
    mag = rng.integers(1, k + 1, size=(count, n))
    sgn = rng.integers(0, 2, size=(count, n)) * 2 - 1
    return (mag * sgn).astype(np.int32)


def fibonacci_directions(count: int, scale: float) -> np.ndarray:
    """Integer-rounded, ``scale``-scaled Fibonacci-sphere points (BJ:10-11).

    z_i = 1-(2i+1)/N, r = sqrt(1-z^2), phi_i = i*pi*(3-sqrt5),
    v = (r cos phi, r sin phi, z) * scale, rounded half away from zero; a
    component that rounds to 0 becomes sign(unrounded) (+1 if exactly 0),
    because P:105 requires nonzero coordinates.
    Returns (int32 [count, 3], number of directions that had a zero fixed).
    """
    i = np.arange(count, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / count
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    v = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1) * scale
    rounded = np.sign(v) * np.floor(np.abs(v) + 0.5)
    zero = rounded == 0
    fix = np.where(v < 0, -1.0, 1.0)
    rounded = np.where(zero, fix, rounded)
    return rounded.astype(np.int32), int(zero.any(axis=1).sum())


def fibonacci_zero_fixed(count: int, scale: float) -> np.ndarray:
    """bool [count]: the directions of ``fibonacci_directions(count, scale)`` that
    had a component rounded to 0 and fixed to +-1 (E12)."""
    i = np.arange(count, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / count
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    v = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1) * scale
    return (np.floor(np.abs(v) + 0.5) == 0).any(axis=1)


# --------------------------------------------------------------------------- images

def uniform_image(shape, levels: int, seed: int, dtype=np.uint8) -> np.ndarray:
    """I.i.d. uniform values in {0..levels-1} (BJ:7; P:261 'uniform distribution')."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, levels, size=tuple(shape)).astype(dtype)


def blob_images(batch: int, m: int, seed: int) -> np.ndarray:
    """Config 2 (BJ:8): each image a sum of 3-6 isotropic Gaussian blobs.

    centre ~ U[0,m)^2, sigma ~ U[1.5,5], amplitude ~ U[60,255];
    f(p) = sum A exp(-|p-c|^2 / (2 sigma^2)) at integer pixels; I = clip(round(f), 0, 255).
    Returns uint8 [batch, m, m].
    """
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(m, dtype=np.float64), np.arange(m, dtype=np.float64), indexing="ij")
    out = np.empty((batch, m, m), dtype=np.uint8)
    for b in range(batch):
        k = int(rng.integers(3, 7))
        f = np.zeros((m, m))
        for _ in range(k):
            cy, cx = rng.uniform(0, m, size=2)
            s = rng.uniform(1.5, 5.0)
            a = rng.uniform(60.0, 255.0)
            f += a * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
        out[b] = np.clip(np.rint(f), 0, 255).astype(np.uint8)
    return out


def binarize(img: np.ndarray, threshold) -> np.ndarray:
    """1 where img >= threshold else 0 (config 2 binary variant, BJ:8)."""
    return (img >= threshold).astype(img.dtype)


def grf_image(m: int, seed: int, levels: int = 256) -> np.ndarray:
    """Config 3 (BJ:9): Gaussian random field with power spectrum ~ k^-3.

    white N(0,1) -> FFT -> * |k|^(-3/2) (k from fftfreq, k=0 -> 0) -> real IFFT
    -> q = min(floor(levels (f-min)/(max-min)), levels-1). Returns int16 [m, m].
    """
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((m, m))
    ky = np.fft.fftfreq(m)[:, None]
    kx = np.fft.fftfreq(m)[None, :]
    k = np.sqrt(ky * ky + kx * kx)
    amp = np.zeros_like(k)
    amp[k > 0] = k[k > 0] ** -1.5
    f = np.real(np.fft.ifft2(np.fft.fft2(w) * amp))
    q = np.floor(levels * (f - f.min()) / (f.max() - f.min()))
    return np.minimum(q, levels - 1).astype(np.int16)


def smooth_volume(m: int, seed: int, sigma: float = 3.0) -> np.ndarray:
    """Configs 4-5 (BJ:10-11): U[0,1) i.i.d. noise, separable Gaussian blur
    (sigma voxels, periodic boundary, truncate 4 sigma), min-max requantised to
    {0..255}. Returns uint8 [m, m, m]."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    v = rng.random((m, m, m), dtype=np.float64)
    f = gaussian_filter(v, sigma=sigma, mode="wrap", truncate=4.0)
    q = np.floor(256.0 * (f - f.min()) / (f.max() - f.min()))
    return np.minimum(q, 255).astype(np.uint8)


def median_binarize(v: np.ndarray) -> np.ndarray:
    """1 iff v > median(v) (config 4 binary variant)."""
    return (v > np.median(v)).astype(v.dtype)


def squares_image(m: int, k: int, s: int | None = None, dtype=np.uint8) -> np.ndarray:
    """Periodic pattern of k x k isolated s x s foreground squares.

    Top-left corners at (floor(i m/k), floor(j m/k)); requires k (s+1) <= m so the
    squares are separated by background.
    """
    if s is None:
        s = max(2, m // (2 * max(k, 1)))
    img = np.zeros((m, m), dtype=dtype)
    for i in range(k):
        for j in range(k):
            y, x = (i * m) // k, (j * m) // k
            img[y:y + s, x:x + s] = 1
    return img


# EX4: the 4x4 binary image of the paper's running example as reconstructed by
# SPEC from Appendix A ("9 vertices, 9 edges, and 2 squares" and Table 2).
EX4 = np.array([[1, 0, 0, 0], [0, 1, 1, 0], [1, 1, 1, 1], [1, 1, 0, 0]], dtype=np.uint8)


# --------------------------------------------------------------------------- configs

def config_inputs(k: int, variant: str = "gray", small: bool = False):
    """Inputs of BASELINE.json config k (1-based). Returns dict(images, dirs, ...).

    images: numpy array [batch, *shape]; dirs: int32 [D, n].
    ``small=True`` keeps the recipe but shrinks sizes for quick tests.
    """
    if k == 1:
        img = uniform_image((32, 32), 256, IMAGE_SEED[1])[None]
        dirs = random_directions(32, 2, 8, DIR_SEED[1])
        return dict(images=img, dirs=dirs, construction="top")
    if k == 2:
        batch = 64 if small else 1024
        imgs = blob_images(batch, 28, IMAGE_SEED[2])
        if variant == "binary":
            imgs = binarize(imgs, 128)
        dirs = random_directions(256, 2, 16, DIR_SEED[2])
        return dict(images=imgs, dirs=dirs, construction="vertex")
    if k == 3:
        m = 256 if small else 2048
        img = grf_image(m, IMAGE_SEED[3])[None]
        dirs = random_directions(4096, 2, 64, DIR_SEED[3])
        return dict(images=img, dirs=dirs, construction="vertex")
    if k == 4:
        m = 64 if small else 256
        v = smooth_volume(m, IMAGE_SEED[4])
        if variant == "binary":
            v = median_binarize(v)
        dirs, nfix = fibonacci_directions(1024, 32.0)
        return dict(images=v[None], dirs=dirs, construction="vertex", zero_fixed=nfix)
    if k == 5:
        m = 32 if small else 128
        nb = 2 if small else 16
        vols = np.stack([smooth_volume(m, 1500 + j) for j in range(nb)])
        dirs, nfix = fibonacci_directions(10000, 64.0)
        return dict(images=vols, dirs=dirs, construction="vertex", zero_fixed=nfix)
    raise ValueError(k)
