"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python face of the plain C oracle in ``oracle/eucalc_oracle.c`` (see its header
for the passages of arxiv 2405.02256 each function follows). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package. It shares no code with the product
package ``paper_2405_02256_b200`` and never imports it.

Conventions:
  * images are row-major, axis i of the array <-> direction coordinate xi_i;
  * heights are integer lattice heights H = sum_i xi_i * (L/(M_i-1)) * p_i,
    L = lcm of (M_i - 1) over axes with M_i > 1 (E10); the paper's normalised
    height is t = (2H - L*csum) / (2L), csum = sum of xi_i over those axes;
  * J (jump) = Delta^- - chi(upper star) = -(paper's Delta^ord) (E1).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from fractions import Fraction
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eucalc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

VERTEX, TOP = 0, 1
KERNELS = {"gauss": 0, "cos": 1, "sin": 2, "exp": 3, "one": 4}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no tuning)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64 = ctypes.c_int64
            lib.eo_doubled_grid.argtypes = [P, ctypes.c_int, P, ctypes.c_int, P]
            lib.eo_euler.argtypes = [P, ctypes.c_int, P]
            lib.eo_euler.restype = i64
            lib.eo_critical.argtypes = [P, ctypes.c_int, P, ctypes.c_int, P, P]
            lib.eo_ect_at.argtypes = [P, ctypes.c_int, P, P, i64]
            lib.eo_ect_at.restype = i64
            lib.eo_radon_at.argtypes = [P, ctypes.c_int, P, P, i64]
            lib.eo_radon_at.restype = i64
            lib.eo_transforms.argtypes = [P, ctypes.c_int, P, P, i64] + [P] * 9
            lib.eo_transforms_real.argtypes = [P, ctypes.c_int, P, P, i64] + [P] * 9
            lib.eo_ht_quad.argtypes = [P, ctypes.c_int, P, P, i64, i64, ctypes.c_int, ctypes.c_double, ctypes.c_int]
            lib.eo_ht_quad.restype = ctypes.c_double
            lib.eo_ht_cells.argtypes = [P, ctypes.c_int, P, P, i64, i64, ctypes.c_int, ctypes.c_double]
            lib.eo_ht_cells.restype = ctypes.c_double
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _construction(c) -> int:
    if isinstance(c, str):
        return {"vertex": VERTEX, "top": TOP}[c.lower()]
    return int(c)


# --------------------------------------------------------------------------- grid

class Grid:
    """A weighted cubical complex on the doubled grid (step 1 of SURVEY §8(c))."""

    def __init__(self, img: np.ndarray, construction):
        img = np.ascontiguousarray(img, dtype=np.int32)
        self.construction = _construction(construction)
        self.m = np.array(img.shape, dtype=np.int64)
        self.n = img.ndim
        if self.construction == VERTEX:
            self.d = 2 * self.m - 1
        else:
            self.d = 2 * self.m + 1
        self.M = (self.d + 1) // 2  # vertices per axis
        self.cells = np.empty(tuple(int(x) for x in self.d), dtype=np.int32)
        rc = _get().eo_doubled_grid(_p(img), self.n, _p(self.m), self.construction, _p(self.cells))
        if rc != 0:
            raise ValueError("bad image")
        Ms = [int(x) for x in self.M if x > 1]
        self.L = 1
        for v in Ms:
            self.L = self.L * (v - 1) // math.gcd(self.L, v - 1)
        self.scale = np.array([self.L // (int(x) - 1) if x > 1 else 0 for x in self.M], dtype=np.int64)

    # -- helpers
    def xs(self, xi) -> np.ndarray:
        """Axis-scaled integer direction xs_i = xi_i * L/(M_i - 1) (E10)."""
        xi = np.asarray(xi, dtype=np.int64)
        if xi.shape != (self.n,) or np.any(xi == 0):
            raise ValueError("direction must have n nonzero coordinates (P:105)")
        return np.ascontiguousarray(xi * self.scale)

    def csum(self, xi) -> int:
        return int(sum(int(x) for x, M in zip(xi, self.M) if M > 1))

    def t_of(self, H, xi):
        """Paper's normalised height t = H/L - csum/2 (E10) as float64."""
        return (2.0 * np.asarray(H, dtype=np.float64) - self.L * self.csum(xi)) / (2.0 * self.L)

    def euler(self) -> int:
        return int(_get().eo_euler(_p(self.cells), self.n, _p(self.d)))

    def critical(self, e: int):
        """(dminus, eplus) over the vertex lattice for orthant index e."""
        nv = int(np.prod(self.M))
        dm = np.empty(nv, dtype=np.int64)
        ep = np.empty(nv, dtype=np.int64)
        _get().eo_critical(_p(self.cells), self.n, _p(self.d), int(e), _p(dm), _p(ep))
        return dm, ep

    def critical_table(self, e: int):
        """Per-orthant tables: (classical vertex ids, Delta^-, ordinary ids, J).

        Vertex ids are row-major over the vertex lattice; J = dminus - eplus (E1)."""
        dm, ep = self.critical(e)
        j = dm - ep
        c = np.nonzero(dm)[0]
        o = np.nonzero(j)[0]
        return c, dm[c], o, j[o]

    def ect_at(self, xi, t2: int) -> int:
        return int(_get().eo_ect_at(_p(self.cells), self.n, _p(self.d), _p(self.xs(xi)), int(t2)))

    def radon_at(self, xi, t2: int) -> int:
        return int(_get().eo_radon_at(_p(self.cells), self.n, _p(self.d), _p(self.xs(xi)), int(t2)))

    def height_range(self, xi):
        xs = self.xs(xi)
        ext = xs * (self.M - 1)
        return int(ext[ext < 0].sum()), int(ext[ext > 0].sum())

    def transforms(self, xi):
        """Canonical exact ECT (T,E) and Radon (T_o,E', T_c,E_c), heights in lattice units."""
        xs = self.xs(xi)
        lo, hi = self.height_range(xi)
        cap = hi - lo + 1
        bufs = [np.empty(cap, dtype=np.int64) for _ in range(6)]
        cnt = [np.zeros(1, dtype=np.int64) for _ in range(3)]
        rc = _get().eo_transforms(_p(self.cells), self.n, _p(self.d), _p(xs), cap,
                                  _p(bufs[0]), _p(bufs[1]), _p(cnt[0]),
                                  _p(bufs[2]), _p(bufs[3]), _p(cnt[1]),
                                  _p(bufs[4]), _p(bufs[5]), _p(cnt[2]))
        if rc != 0:
            raise RuntimeError(f"eo_transforms rc={rc}")
        a, b, c = (int(x[0]) for x in cnt)
        return dict(T=bufs[0][:a].copy(), E=bufs[1][:a].copy(),
                    To=bufs[2][:b].copy(), Eo=bufs[3][:b].copy(),
                    Tc=bufs[4][:c].copy(), Ec=bufs[5][:c].copy())

    def transforms_real(self, xi):
        """Canonical ECT / Radon for a real-valued direction (NEXT f3, E22): heights
        are the doubles <xi, x> of the vertices (P:116 embedding, left-to-right,
        no FMA); returns T/To/Tc as float64 and E/Eo/Ec as int64."""
        xi = np.ascontiguousarray(np.asarray(xi, dtype=np.float64))
        if xi.shape != (self.n,) or np.any(xi == 0):
            raise ValueError("direction must have n nonzero coordinates (P:105)")
        cap = int(np.prod(self.M))
        hb = [np.empty(cap, dtype=np.float64) for _ in range(3)]
        vb = [np.empty(cap, dtype=np.int64) for _ in range(3)]
        cnt = [np.zeros(1, dtype=np.int64) for _ in range(3)]
        rc = _get().eo_transforms_real(_p(self.cells), self.n, _p(self.d), _p(xi), cap,
                                       _p(hb[0]), _p(vb[0]), _p(cnt[0]), _p(hb[1]), _p(vb[1]), _p(cnt[1]),
                                       _p(hb[2]), _p(vb[2]), _p(cnt[2]))
        if rc != 0:
            raise RuntimeError(f"eo_transforms_real rc={rc}")
        a, b, c = (int(x[0]) for x in cnt)
        return dict(T=hb[0][:a].copy(), E=vb[0][:a].copy(), To=hb[1][:b].copy(), Eo=vb[1][:b].copy(),
                    Tc=hb[2][:c].copy(), Ec=vb[2][:c].copy())

    # -- evaluation at real t straight from the definitions
    def _t2(self, xi, t):
        """The query t (a Python float = IEEE double, taken exactly) in doubled
        lattice units: t2 = 2H with t = H/L - csum/2 (E10), i.e. t2 = 2Lt + L*csum,
        an exact rational."""
        t2 = Fraction(t) * (2 * self.L) + self.L * self.csum(xi)
        # every cell height lies in [lo, hi]: thresholds beyond change nothing, and
        # clamping keeps the doubled threshold inside the C oracle's int64
        lo, hi = self.height_range(xi)
        return min(max(t2, Fraction(2 * lo - 3)), Fraction(2 * hi + 3))

    def ect_eval(self, xi, t) -> int:
        """ECT(xi, t) = chi[phi_{xi <= t}] at real t: every cell with
        2 max_P <= t2 counts, i.e. 2 max_P <= floor(t2) (max_P is a lattice height)."""
        if math.isinf(t):
            return 0 if t < 0 else self.euler()
        return self.ect_at(xi, math.floor(self._t2(xi, t)))

    def radon_eval(self, xi, t) -> int:
        """Radon(xi, t) = chi[phi_{xi = t}] at real t. An integer t2 is
        probed as is; a non-integer t2 lies strictly between two doubled lattice
        heights (even numbers) and is replaced by the odd integer of its unit
        interval, which satisfies the same strict comparisons against even values."""
        if math.isinf(t):
            return 0
        t2 = self._t2(xi, t)
        if t2.denominator == 1:
            return self.radon_at(xi, int(t2))
        k = math.floor(t2)
        return self.radon_at(xi, k if k % 2 else k + 1)

    @staticmethod
    def sample_points(a: float, b: float, N: int):
        """The vectorisation grid t_i = a + i(b-a)/(N-1), i = 0..N-1,
        evaluated in IEEE double in the order (i*(b-a))/(N-1) then a + . (E20)."""
        if N == 1:
            return [float(a)]
        return [float(a) + (i * (float(b) - float(a))) / (N - 1) for i in range(N)]

    def vectorize(self, xi, a: float, b: float, N: int, kind: str = "ect"):
        f = self.ect_eval if kind == "ect" else self.radon_eval
        return np.array([f(xi, t) for t in self.sample_points(a, b, N)], dtype=np.int64)

    def ht_quad(self, xi, kernel: str, param: float = 1.0, nsub: int = 1) -> float:
        return float(_get().eo_ht_quad(_p(self.cells), self.n, _p(self.d), _p(self.xs(xi)), self.L,
                                       self.csum(xi), KERNELS[kernel], float(param), int(nsub)))

    def ht_cells(self, xi, kernel: str, param: float = 1.0) -> float:
        return float(_get().eo_ht_cells(_p(self.cells), self.n, _p(self.d), _p(self.xs(xi)), self.L,
                                        self.csum(xi), KERNELS[kernel], float(param)))


# --------------------------------------------------------------------------- batches

def _threads(threads):
    return threads or os.cpu_count() or 1


def transforms_batch(images, dirs, construction, pairs=None, threads=None):
    """Oracle ECT/Radon for every (image, direction) pair (or the listed pairs).

    Returns dict[(b, d)] -> transforms dict. Threads run over (image, direction)
    (ctypes releases the GIL); each grid is materialised once per image.
    """
    images = np.asarray(images)
    dirs = np.asarray(dirs)
    if pairs is None:
        pairs = [(b, d) for b in range(images.shape[0]) for d in range(dirs.shape[0])]
    need = sorted({b for b, _ in pairs})
    with ThreadPoolExecutor(_threads(threads)) as ex:
        grids = dict(zip(need, ex.map(lambda b: Grid(images[b], construction), need)))
        res = ex.map(lambda bd: grids[bd[0]].transforms(dirs[bd[1]]), pairs)
        return dict(zip(pairs, res))


def transforms_real_batch(images, dirs, construction, pairs=None, threads=None):
    """Oracle ECT/Radon for real-valued directions (float64 [D, n]) per (image, direction)."""
    images = np.asarray(images)
    dirs = np.asarray(dirs, dtype=np.float64)
    if pairs is None:
        pairs = [(b, d) for b in range(images.shape[0]) for d in range(dirs.shape[0])]
    need = sorted({b for b, _ in pairs})
    with ThreadPoolExecutor(_threads(threads)) as ex:
        grids = dict(zip(need, ex.map(lambda b: Grid(images[b], construction), need)))
        res = ex.map(lambda bd: grids[bd[0]].transforms_real(dirs[bd[1]]), pairs)
        return dict(zip(pairs, res))


def ht_batch(images, dirs, construction, kernel, param, pairs=None, threads=None, form="quad"):
    images = np.asarray(images)
    dirs = np.asarray(dirs)
    if pairs is None:
        pairs = [(b, d) for b in range(images.shape[0]) for d in range(dirs.shape[0])]
    need = sorted({b for b, _ in pairs})
    with ThreadPoolExecutor(_threads(threads)) as ex:
        grids = dict(zip(need, ex.map(lambda b: Grid(images[b], construction), need)))
        if form == "quad":
            f = lambda bd: grids[bd[0]].ht_quad(dirs[bd[1]], kernel, param)
        else:
            f = lambda bd: grids[bd[0]].ht_cells(dirs[bd[1]], kernel, param)
        return dict(zip(pairs, ex.map(f, pairs)))
