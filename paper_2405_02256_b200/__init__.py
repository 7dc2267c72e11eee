"""eucalc-b200: exact ECT / Radon / hybrid transforms of weighted cubical complexes
(arxiv 2405.02256) on one B200, behind the C ABI of include/eucalc.h.

This module is a thin ctypes binding with the ABI's names: it marshals
arguments (torch tensors or numpy arrays -> pointers, the current CUDA stream)
and allocates outputs with torch. Every step of the path runs in the CUDA
kernels of libeucalc.so; there is no CPU fallback — if the library is missing
the import of the native layer raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# EUCALC_LIB=checked loads libeucalc_checked.so (device bounds checks compiled in;
# tests only): the same kernels, every EU_DCHECK traps on an out-of-range index
# EUCALC_LIB=dev loads libeucalc_dev.so (development builds: K2 instantiated for 8-byte
# records and 32-bit outputs only, anything else returns an error)
LIB_PATH = os.path.join(_HERE, {"checked": "libeucalc_checked.so", "dev": "libeucalc_dev.so"}.get(
    os.environ.get("EUCALC_LIB", ""), "libeucalc.so"))

OK, E_ARG, E_NOMEM, E_CUDA, E_NONGENERIC, E_CAPACITY, E_RANGE, E_STATE = range(8)
DTYPES = {np.dtype(np.uint8): 0, np.dtype(np.int16): 1, np.dtype(np.int32): 2}
CONSTRUCTIONS = {"vertex": 0, "top": 1}
KERNELS = {"gauss": 0, "cos": 1, "sin": 2, "exp": 3}
PRECISIONS = {"f32": 0, "f64": 1}


class EucalcError(RuntimeError):
    def __init__(self, status, msg, bad_index=-1, required=None):
        super().__init__(f"eucalc status {status}: {msg}")
        self.status = status
        self.bad_index = bad_index
        self.required = required


class _Steps(ctypes.Structure):
    _fields_ = [("offsets", ctypes.c_void_p), ("height", ctypes.c_void_p), ("value", ctypes.c_void_p),
                ("capacity", ctypes.c_int64), ("elem_bytes", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None


def lib():
    """Load libeucalc.so (in-tree). Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2405_02256_b200._build` "
                              "(the CUDA extension is required, there is no CPU path)")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32, St = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int
        L.eucalc_build_complex.argtypes = [P, I32, I32, P, I64, I32, P, ctypes.POINTER(P)]
        L.eucalc_destroy_complex.argtypes = [P]
        L.eucalc_critical_points.argtypes = [P, P, ctypes.POINTER(P)]
        L.eucalc_destroy_critical.argtypes = [P]
        L.eucalc_critical_counts.argtypes = [P, P, P]
        L.eucalc_critical_list_lengths.argtypes = [P, P, P]
        L.eucalc_critical_list_lengths.restype = St
        L.eucalc_critical_export.argtypes = [P, I64, I32, P, P, P, I64, ctypes.POINTER(I64), P]
        L.eucalc_output_bound.argtypes = [P, P, I64, ctypes.POINTER(I64), ctypes.POINTER(I64), P]
        L.eucalc_output_bound_upper.argtypes = [P, P, I64, ctypes.POINTER(I64), P]
        SP = ctypes.POINTER(_Steps)
        L.eucalc_transforms.argtypes = [P, P, I64, SP, SP, SP, ctypes.POINTER(I64), P]
        L.eucalc_transforms_ht.argtypes = [P, P, I64, SP, SP, SP, I32, ctypes.c_double, I32, P,
                                           ctypes.POINTER(I64), P]
        L.eucalc_transforms_real.argtypes = [P, P, I64, SP, SP, SP, ctypes.POINTER(I64), P]
        L.eucalc_ect.argtypes = [P, P, I64, SP, ctypes.POINTER(I64), P]
        L.eucalc_radon.argtypes = [P, P, I64, SP, SP, ctypes.POINTER(I64), P]
        L.eucalc_hybrid.argtypes = [P, P, I64, I32, ctypes.c_double, I32, P, P]
        L.eucalc_hybrid_ex.argtypes = [P, P, I64, I32, ctypes.c_double, I32, I32, P, P]
        L.eucalc_evaluate.argtypes = [P, P, I64, I32, SP, SP, P, I64, P, I32, P]
        L.eucalc_vectorize.argtypes = [P, P, I64, I32, SP, SP, ctypes.c_double, ctypes.c_double, I64, P, I32, P]
        L.eucalc_height_map.argtypes = [P, P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.eucalc_profile_enable.argtypes = [I32]
        L.eucalc_profile_enable.restype = None
        L.eucalc_profile_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]
        L.eucalc_profile_span.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]
        L.eucalc_launch_count.argtypes = [I32]
        L.eucalc_launch_count.restype = I64
        L.eucalc_k2_restarts.argtypes = [I32]
        L.eucalc_k2_restarts.restype = I64
        L.eucalc_status_string.restype = ctypes.c_char_p
        L.eucalc_last_error.restype = ctypes.c_char_p
        L.eucalc_last_bad_index.restype = I64
        for f in ("eucalc_build_complex", "eucalc_destroy_complex", "eucalc_critical_points",
                  "eucalc_destroy_critical", "eucalc_critical_counts", "eucalc_critical_export",
                  "eucalc_output_bound", "eucalc_output_bound_upper", "eucalc_transforms", "eucalc_ect", "eucalc_radon",
                  "eucalc_hybrid", "eucalc_hybrid_ex", "eucalc_height_map", "eucalc_evaluate", "eucalc_transforms_ht",
                  "eucalc_transforms_real",
                  "eucalc_vectorize"):
            getattr(L, f).restype = St
        _lib = L
    return _lib


def _check(st, required=None):
    if st != OK:
        L = lib()
        raise EucalcError(st, L.eucalc_last_error().decode(), L.eucalc_last_bad_index(), required)


def _stream(stream):
    import torch

    if stream is None:
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(0)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(x):
    """(pointer, keepalive) for a torch tensor or numpy array (host or device)."""
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x)
    return ctypes.c_void_p(a.ctypes.data), a


def _dirs_i32(dirs):
    if hasattr(dirs, "data_ptr"):
        import torch

        assert dirs.dtype == torch.int32 and dirs.is_contiguous() and dirs.dim() == 2
        return dirs
    return np.ascontiguousarray(np.asarray(dirs, dtype=np.int32).reshape(len(dirs), -1))


class Complex:
    """eucalc_build_complex handle: a batch of same-shape images (P:116 / P:140)."""

    def __init__(self, images, construction="vertex", stream=None):
        if hasattr(images, "data_ptr"):
            import torch

            tmap = {torch.uint8: 0, torch.int16: 1, torch.int32: 2}
            dt = tmap[images.dtype]
            images = images.contiguous()
            shape = tuple(images.shape)
        else:
            images = np.ascontiguousarray(images)
            dt = DTYPES[images.dtype]
            shape = images.shape
        self.batch = int(shape[0])
        self.shape = tuple(int(s) for s in shape[1:])
        self.ndim = len(self.shape)
        self.construction = construction
        self.stream = stream
        p, keep = _ptr(images)
        shp = (ctypes.c_int64 * self.ndim)(*self.shape)
        h = ctypes.c_void_p()
        _check(lib().eucalc_build_complex(p, dt, self.ndim, shp, self.batch, CONSTRUCTIONS[construction],
                                          _stream(stream), ctypes.byref(h)))
        self._h = h
        del keep

    def height_map(self, xi):
        """(L, csum) with t = (2H - L*csum) / (2L) (paper's normalised height, E10)."""
        d = (ctypes.c_int32 * self.ndim)(*[int(v) for v in xi])
        L, cs = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().eucalc_height_map(self._h, d, ctypes.byref(L), ctypes.byref(cs)))
        return L.value, cs.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.eucalc_destroy_complex(self._h)
            self._h = None


class Critical:
    """eucalc_critical_points handle (K1: per-pair critical lists)."""

    def __init__(self, cx: Complex, stream=None):
        self.cx = cx
        self.stream = stream
        h = ctypes.c_void_p()
        _check(lib().eucalc_critical_points(cx._h, _stream(stream), ctypes.byref(h)))
        self._h = h

    def counts(self):
        """int64 [batch, 2^n, 2] = (N^-, N^ord) per orthant (syncs)."""
        out = np.zeros((self.cx.batch, 1 << self.cx.ndim, 2), dtype=np.int64)
        _check(lib().eucalc_critical_counts(self._h, ctypes.c_void_p(out.ctypes.data), _stream(self.stream)))
        return out

    def list_lengths(self):
        """int64 [batch, 2^(n-1)] lengths of the antipodal-pair lists (syncs)."""
        out = np.zeros((self.cx.batch, 1 << (self.cx.ndim - 1)), dtype=np.int64)
        _check(lib().eucalc_critical_list_lengths(self._h, ctypes.c_void_p(out.ctypes.data), _stream(self.stream)))
        return out

    def export(self, image: int, orthant: int):
        """(vertex ids, Delta^-, J) of (image, orthant), ascending vertex id (syncs)."""
        n = ctypes.c_int64()
        st = lib().eucalc_critical_export(self._h, image, orthant, None, None, None, 0, ctypes.byref(n),
                                          _stream(self.stream))
        if st not in (OK, E_CAPACITY):
            _check(st)
        k = n.value
        v = np.empty(k, dtype=np.int64)
        dm = np.empty(k, dtype=np.int32)
        j = np.empty(k, dtype=np.int32)
        _check(lib().eucalc_critical_export(self._h, image, orthant, ctypes.c_void_p(v.ctypes.data),
                                            ctypes.c_void_p(dm.ctypes.data), ctypes.c_void_p(j.ctypes.data),
                                            k, ctypes.byref(n), _stream(self.stream)))
        return v, dm, j

    def output_bound(self, dirs):
        d = _dirs_i32(dirs)
        p, keep = _ptr(d)
        be, bo = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().eucalc_output_bound(self._h, p, int(d.shape[0]), ctypes.byref(be), ctypes.byref(bo),
                                         _stream(self.stream)))
        return be.value, bo.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.eucalc_destroy_critical(self._h)
            self._h = None


def build_complex(images, construction="vertex", stream=None) -> Complex:
    return Complex(images, construction, stream)


def critical_points(cx: Complex, stream=None) -> Critical:
    return Critical(cx, stream)


def _alloc_steps(torch, S, cap, elem_bytes, device, with_height=True):
    dt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[elem_bytes]
    pin = device == "cpu" and torch.cuda.is_available()
    mk = lambda n, t: torch.empty(n, dtype=t, device=device, pin_memory=pin)
    off = mk(S + 1, torch.int64)
    h = mk(max(cap, 1), dt) if with_height else None
    v = mk(max(cap, 1), dt)
    st = _Steps(off.data_ptr(), h.data_ptr() if h is not None else 0, v.data_ptr(), cap, elem_bytes, 0)
    return dict(offsets=off, height=h, value=v), st


class _CsrBlock:
    """All requested CSR streams (and optionally one extra tensor, the fused HT
    output) carved out of ONE allocation: one allocator call instead of up to
    nine. Offsets first (8-byte aligned), then heights/values. The C structs
    (`sts`) are built from raw addresses, so the library call can be issued
    before any tensor view is created (views(): after the launch, off the
    device's critical path)."""

    def __init__(self, torch, S, cap, elem_bytes, device, names, share, extra=None):
        self.torch, self.S, self.cap, self.eb = torch, S, max(cap, 1), elem_bytes
        self.dt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[elem_bytes]
        pin = device == "cpu" and torch.cuda.is_available()
        arr = (self.cap * elem_bytes + 255) // 256 * 256
        offb = ((S + 1) * 8 + 255) // 256 * 256
        self.plan = []
        total = 0
        for name in names:
            has_h = not (name == "classical" and share)
            h = total + offb if has_h else None
            v = total + offb + (arr if has_h else 0)
            self.plan.append((name, total, h, v))
            total = v + arr
        self.extra = extra
        self.xoff = total
        if extra is not None:
            xshape, xdt = extra
            self.xn = int(np.prod(xshape)) * (4 if xdt == torch.float32 else 8)
            total += (self.xn + 255) // 256 * 256
        self.buf = torch.empty(total, dtype=torch.uint8, device=device, pin_memory=pin)
        base = self.buf.data_ptr()
        self.sts = {}
        for name, o, h, v in self.plan:
            self.sts[name] = _Steps(base + o, base + h if h is not None else 0, base + v, cap, elem_bytes, 0)
        self.extra_ptr = base + self.xoff

    def views(self):
        torch, buf, n = self.torch, self.buf, self.cap * self.eb
        res = {}
        for name, o, h, v in self.plan:
            res[name] = dict(offsets=buf[o:o + (self.S + 1) * 8].view(torch.int64),
                             height=buf[h:h + n].view(self.dt) if h is not None else None,
                             value=buf[v:v + n].view(self.dt))
        if self.extra is not None:
            xshape, xdt = self.extra
            res["_extra"] = buf[self.xoff:self.xoff + self.xn].view(xdt).view(xshape)
        return res


def _alloc_all(torch, S, cap, elem_bytes, device, names, share, extra=None):
    """(views dict, C structs) of a _CsrBlock (callers that need the views first)."""
    blk = _CsrBlock(torch, S, cap, elem_bytes, device, names, share, extra)
    return blk.views(), blk.sts


_UPPER_MAX_BYTES = 8 << 30  # capacity="auto": the no-sync bound when its outputs fit this


def transforms(cr: Critical, dirs, ect=True, ordinary=True, classical=True, elem_bytes=8, device="cuda",
               share_heights=False, stream=None, ht=None, capacity="auto"):
    """eucalc_transforms: canonical ECT (T,E) and Radon (T_o,E'), (T_c,E_c) for every
    (image, direction), as CSR torch tensors on `device` ("cuda" or "cpu").

    elem_bytes: 2, 4 or 8 (int16/int32/int64 heights and values), or "auto" for
    the narrowest width the library accepts (E_RANGE -> next width).
    share_heights=True lets the classical stream reuse the ECT heights (T_c = T,
    Lemma 6) instead of writing them twice; its "height" is then the ECT tensor.
    ht=(kernel, param, precision) also returns res["ht"] [batch, D], the hybrid
    transform from the same merged histogram (eucalc_transforms_ht, NEXT f2).
    capacity: "tight" sizes the outputs by eucalc_output_bound (waits for K1's
    list lengths); "upper" by eucalc_output_bound_upper (no wait: the allocation
    overlaps K1, the library then waits inside the launch call); "auto" = upper
    for device outputs of at most 8 GiB, else tight."""
    if elem_bytes == "auto":
        for eb in (2, 4):
            try:
                return transforms(cr, dirs, ect, ordinary, classical, eb, device, share_heights, stream, ht,
                                  capacity)
            except EucalcError as e:
                if e.status != E_RANGE:
                    raise
        elem_bytes = 8
    import torch

    d = _dirs_i32(dirs)
    D = int(d.shape[0])
    S = cr.cx.batch * D
    st = _stream(stream if stream is not None else cr.stream)
    p, keep = _ptr(d)
    names = [n for n, want in (("ect", ect), ("ordinary", ordinary), ("classical", classical)) if want]
    bound = None
    if capacity in ("auto", "upper") and device != "cpu":
        bu = ctypes.c_int64()
        _check(lib().eucalc_output_bound_upper(cr.cx._h, p, D, ctypes.byref(bu), st))
        if capacity == "upper" or bu.value * elem_bytes * 2 * len(names) <= _UPPER_MAX_BYTES:
            bound = bu.value
    if bound is None:
        be, bo = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().eucalc_output_bound(cr._h, p, D, ctypes.byref(be), ctypes.byref(bo), st))
        bound = be.value
    share = share_heights and ect and classical
    extra = None
    if ht is not None:  # the HT output shares the CSR allocation
        extra = ((cr.cx.batch, D), torch.float32 if ht[2] == "f32" else torch.float64)
    blk = _CsrBlock(torch, S, bound, elem_bytes, device, names, share, extra)
    sts = blk.sts
    if share:
        sts["classical"].height = sts["ect"].height
    req = ctypes.c_int64()
    refs = [ctypes.byref(sts[n]) if n in sts else None for n in ("ect", "ordinary", "classical")]
    if ht is None:
        _check(lib().eucalc_transforms(cr._h, p, D, refs[0], refs[1], refs[2], ctypes.byref(req), st), req.value)
    else:
        kern, param, prec = ht
        _check(lib().eucalc_transforms_ht(cr._h, p, D, refs[0], refs[1], refs[2], KERNELS[kern], float(param),
                                          PRECISIONS[prec], ctypes.c_void_p(blk.extra_ptr), ctypes.byref(req), st),
               req.value)
    res = blk.views()  # tensor views after the launch (the kernels already run)
    if share:
        res["classical"]["height"] = res["ect"]["height"]
    if ht is not None:
        res["ht"] = res.pop("_extra")
    return res


def transforms_real(cr: Critical, dirs, ect=True, ordinary=True, classical=True, device="cuda", share_heights=False,
                    stream=None):
    """eucalc_transforms_real: canonical ECT / Radon for real-valued directions
    (float64 [D, n]); heights are float64 paper heights <xi, x>, values int64."""
    import torch

    d = dirs if hasattr(dirs, "data_ptr") else np.ascontiguousarray(np.asarray(dirs, dtype=np.float64).reshape(len(dirs), -1))
    D = int(d.shape[0])
    S = cr.cx.batch * D
    st = _stream(stream if stream is not None else cr.stream)
    p, keep = _ptr(d)
    names = [n for n, want in (("ect", ect), ("ordinary", ordinary), ("classical", classical)) if want]
    share = share_heights and ect and classical
    req = ctypes.c_int64()
    # first call with no outputs: the library reports the capacity it needs
    _check(lib().eucalc_transforms_real(cr._h, p, D, None, None, None, ctypes.byref(req), st))
    res, sts = _alloc_all(torch, S, req.value, 8, device, names, share)
    for name in names:
        res[name]["height"] = res[name]["height"].view(torch.float64) if res[name]["height"] is not None else None
    if share:
        res["classical"]["height"] = res["ect"]["height"]
        sts["classical"].height = sts["ect"].height
    refs = [ctypes.byref(sts[n]) if n in sts else None for n in ("ect", "ordinary", "classical")]
    _check(lib().eucalc_transforms_real(cr._h, p, D, refs[0], refs[1], refs[2], ctypes.byref(req), st), req.value)
    return res


def shard_directions(dirs, rank: int, world: int):
    """Multi-GPU split of ONE image's directions: the directions,
    stably grouped by antipodal orthant pair (directions of one pair read the
    same critical list, Lemma 3), cut into `world` contiguous chunks of
    near-equal size. Returns (indices into dirs, dirs[indices]) for `rank`. Each
    rank runs K1 on the whole image and K2/K3 on its chunk; outputs stay sharded
    (no data-path collective). Host logic only."""
    d = np.ascontiguousarray(np.asarray(dirs).reshape(len(dirs), -1))
    n = d.shape[1]
    full = (1 << n) - 1
    e = ((d > 0).astype(np.int64) << np.arange(n)).sum(1)
    pair = np.where((e >> (n - 1)) & 1, e ^ full, e)
    order = np.argsort(pair, kind="stable")
    per = (len(order) + world - 1) // world
    idx = order[min(len(order), rank * per):min(len(order), (rank + 1) * per)]
    return idx, d[idx]


def ect(cr: Critical, dirs, **kw):
    return transforms(cr, dirs, ect=True, ordinary=False, classical=False, **kw)["ect"]


def radon(cr: Critical, dirs, **kw):
    r = transforms(cr, dirs, ect=False, ordinary=True, classical=True, **kw)
    return r["ordinary"], r["classical"]


HT_ALGORITHMS = {"auto": 0, "direct": 1, "table": 2}


def hybrid(cr: Critical, dirs, kernel="gauss", param=1.0, precision="f64", device="cuda", stream=None,
           algorithm="auto"):
    """eucalc_hybrid_ex: HT(xi) = int kappa(t) Radon(xi,t) dt for every (image, direction).
    algorithm: "auto", "direct" (kbar per term) or "table" (kbar tabulated per lattice u)."""
    import torch

    d = _dirs_i32(dirs)
    D = int(d.shape[0])
    dt = torch.float32 if precision == "f32" else torch.float64
    pin = device == "cpu" and torch.cuda.is_available()
    out = torch.empty((cr.cx.batch, D), dtype=dt, device=device, pin_memory=pin)
    p, keep = _ptr(d)
    _check(lib().eucalc_hybrid_ex(cr._h, p, D, KERNELS[kernel], float(param), PRECISIONS[precision],
                                  HT_ALGORITHMS[algorithm], ctypes.c_void_p(out.data_ptr()),
                               _stream(stream if stream is not None else cr.stream)))
    return out


def _steps_struct(st):
    """ctypes eucalc_steps of a CSR dict returned by transforms()."""
    h, v = st["height"], st["value"]
    return _Steps(st["offsets"].data_ptr(), h.data_ptr(), v.data_ptr(), int(v.numel()), int(v.element_size()), 0)


def evaluate(cx: Complex, dirs, t, ect=None, ordinary=None, classical=None, out_elem_bytes=8, device="cuda",
             stream=None):
    """eucalc_evaluate: ECT(xi,t) (pass ect=) or Radon(xi,t) (pass ordinary= and
    classical=) at the queries t (paper units) for every (image, direction)
    segment; returns [batch*D, len(t)]."""
    return _eval(cx, dirs, ect, ordinary, classical, out_elem_bytes, device, stream, t=t)


def vectorize(cx: Complex, dirs, a, b, N, ect=None, ordinary=None, classical=None, out_elem_bytes=8,
              device="cuda", stream=None):
    """eucalc_vectorize: values at t_i = a + (i*(b-a))/(N-1), i < N."""
    return _eval(cx, dirs, ect, ordinary, classical, out_elem_bytes, device, stream, ab=(a, b, N))


def _eval(cx, dirs, ect, ordinary, classical, out_elem_bytes, device, stream, t=None, ab=None):
    import torch

    d = _dirs_i32(dirs)
    D = int(d.shape[0])
    if ect is not None:
        kind, rep, cls = 0, _steps_struct(ect), None
    else:
        kind, rep, cls = 1, _steps_struct(ordinary), _steps_struct(classical)
    nq = len(t) if t is not None else int(ab[2])
    pin = device == "cpu" and torch.cuda.is_available()
    out = torch.empty((cx.batch * D, nq), dtype=torch.int32 if out_elem_bytes == 4 else torch.int64,
                      device=device, pin_memory=pin)
    p, keep = _ptr(d)
    st = _stream(stream if stream is not None else cx.stream)
    if t is not None:
        tq = t if hasattr(t, "data_ptr") else np.ascontiguousarray(np.asarray(t, dtype=np.float64))
        tp, keep_t = _ptr(tq)
        _check(lib().eucalc_evaluate(cx._h, p, D, kind, ctypes.byref(rep), ctypes.byref(cls) if cls else None,
                                     tp, nq, ctypes.c_void_p(out.data_ptr()), out_elem_bytes, st))
    else:
        _check(lib().eucalc_vectorize(cx._h, p, D, kind, ctypes.byref(rep), ctypes.byref(cls) if cls else None,
                                      float(ab[0]), float(ab[1]), nq, ctypes.c_void_p(out.data_ptr()),
                                      out_elem_bytes, st))
    return out


def profile_enable(on=True):
    """Record per-stage CUDA-event times on the launching stream (clears previous records)."""
    lib().eucalc_profile_enable(1 if on else 0)


def profile_read(stage=None):
    """(milliseconds, launches) summed over recorded `stage` launches (None = all)."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    lib().eucalc_profile_read(stage.encode() if stage else None, ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


def profile_span(stage=None):
    """Milliseconds from the first start to the last end of the recorded `stage` launches."""
    ms = ctypes.c_double()
    lib().eucalc_profile_span(stage.encode() if stage else None, ctypes.byref(ms))
    return ms.value


def k2_restarts(reset=False) -> int:
    """eucalc_k2_restarts: block-regime segments recomputed with split bins (counted
    only under the EUCALC_K2_CHK_BITS test hook)."""
    return int(lib().eucalc_k2_restarts(1 if reset else 0))


def launch_count(reset=False) -> int:
    return int(lib().eucalc_launch_count(1 if reset else 0))


def segment(steps, s):
    """(heights, values) of CSR segment s as numpy (moves to host)."""
    off = steps["offsets"]
    a, b = int(off[s]), int(off[s + 1])
    h = steps["height"][a:b].cpu().numpy().astype(np.int64)
    v = steps["value"][a:b].cpu().numpy().astype(np.int64)
    return h, v
