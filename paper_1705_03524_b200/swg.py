"""ctypes binding of the C-ABI in include/swg.h (libswg.so).

This is the Python harness view of the B200 hot path: tests and bench.py
call the SAME extern "C" entry points a C/C++/cgo/ctypes user of the
reference-facing API would bind.  There is no fallback:
if libswg.so is missing or no sm_100 device is present, every entry point
raises.

Error classes mirror the reference exception taxonomy
(/root/reference/proj/include/swih/errors.hpp:10-79).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import build as _build

# SWG_LIB selects an A/B variant build of the same library (tuning only)
LIB_PATH = os.environ.get("SWG_LIB", _build.LIB)

# enums (include/swg.h)
FMT_GRAY8, FMT_GRAY16, FMT_RGB8, FMT_BINS16 = 0, 1, 2, 3
PLANES_PLAIN, PLANES_AFFINE, PLANES_QUADRATIC, PLANES_DECAY = 1, 3, 5, 4
TABLE_PLAIN, TABLE_XRAMP, TABLE_YRAMP = 0, 1, 2
UNIFORM, MANHATTAN, CHEBYSHEV, GAUSS_CHEB = 0, 1, 2, 3
EUCLID_QUAD, EXP_L1 = 4, 5  # declared extensions
SWIH, BRUTE, CAKE, PLAIN = 0, 1, 2, 3
BHATTACHARYYA, INTERSECTION = 0, 1
STRICT, CLIPPED = 0, 1
RING_MEAN, RING_LEVEL = 0, 1
MAX_BINS = 1024


class Error(RuntimeError):
    code = 1

    def __init__(self, msg: str = "", code: Optional[int] = None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class IoError(Error): code = 2
class ZeroMassError(Error): code = 3
class InvalidKernelError(Error): code = 4
class OutOfRangeError(Error): code = 5
class UnsupportedKernelError(Error): code = 6
class WindowOutOfBoundsError(Error): code = 7


class CapacityError(Error):
    code = 8

    def __init__(self, msg="", required_bytes=0):
        super().__init__(msg)
        self.required_bytes = required_bytes


class ConfigError(Error): code = 9
class ModelError(Error): code = 10
class SizeError(Error): code = 11
class CudaError(Error): code = 64
class NoDeviceError(Error): code = 65
class ArgumentError(Error): code = 66


_BY_CODE = {c.code: c for c in (Error, IoError, ZeroMassError, InvalidKernelError, OutOfRangeError,
                                UnsupportedKernelError, WindowOutOfBoundsError, CapacityError,
                                ConfigError, ModelError, SizeError, CudaError, NoDeviceError,
                                ArgumentError)}


class Kernel(C.Structure):
    _fields_ = [("kind", C.c_int), ("kw", C.c_int), ("kh", C.c_int), ("sigma", C.c_double)]

    def __init__(self, kind=UNIFORM, kw=1, kh=None, sigma=0.5):
        super().__init__(kind, kw, kw if kh is None else kh, sigma)

    @property
    def hx(self):
        return (self.kw - 1) // 2

    @property
    def hy(self):
        return (self.kh - 1) // 2

    def __repr__(self):
        return f"Kernel(kind={self.kind}, {self.kw}x{self.kh}, sigma={self.sigma})"


class Peak(C.Structure):
    _fields_ = [("map_x", C.c_int), ("map_y", C.c_int), ("center_x", C.c_int),
                ("center_y", C.c_int), ("score", C.c_double)]

    def astuple(self):
        return (self.map_x, self.map_y, self.center_x, self.center_y, self.score)


class _PlanInfo(C.Structure):
    _fields_ = [("kernel", C.c_char * 32), ("planes", C.c_int), ("entry_bytes", C.c_int),
                ("bins_read", C.c_int), ("ctas", C.c_int)]


class _Req(C.Structure):
    _fields_ = [("kernel", Kernel), ("method", C.c_int), ("sim", C.c_int), ("rings", C.c_int),
                ("ring_rule", C.c_int), ("row_begin", C.c_int), ("row_end", C.c_int),
                ("model", C.POINTER(C.c_double)), ("partial_in", C.c_void_p),
                ("partial_out", C.c_void_p)]


class Term(C.Structure):
    _fields_ = [("valid", C.c_int), ("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int),
                ("y1", C.c_int), ("sx", C.c_int64), ("sy", C.c_int64), ("beta", C.c_int64)]


@dataclass
class MapRequest:
    """likelihood_map arguments (matching.hpp:72-75) + MatchOptions."""
    kernel: Kernel
    model: np.ndarray
    method: int = SWIH
    sim: int = BHATTACHARYYA
    rings: int = 4
    ring_rule: int = RING_MEAN
    rows: Optional[tuple] = None
    partial_in: object = None   # device (rows, mw, 2) float64 tensor / address
    partial_out: object = None


_lib = None


def lib():
    """Load libswg.so (build it first if this checkout has no binary)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        _build.build()
    L = C.CDLL(LIB_PATH)
    vp, st = C.c_void_p, C.c_int
    L.swg_abi_version.restype = C.c_int
    L.swg_last_error.restype = C.c_char_p
    L.swg_last_required_bytes.restype = C.c_size_t
    for name, args in {
        "swg_device_count": [C.POINTER(C.c_int)],
        "swg_ctx_create": [C.c_int, C.POINTER(vp)],
        "swg_ctx_destroy": [vp],
        "swg_ctx_synchronize": [vp],
        "swg_ctx_set_stream": [vp, vp],
        "swg_ctx_launch_count": [vp, C.POINTER(C.c_uint64)],
        "swg_ctx_map_copy_count": [vp, C.POINTER(C.c_uint64)],
        "swg_tables_build": [vp, vp, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int,
                             C.c_int, C.c_size_t, C.POINTER(vp)],
        "swg_tables_build_decay": [vp, vp, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_double, C.c_size_t, C.POINTER(vp)],
        "swg_tables_build_bins": [vp, vp, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_size_t,
                                  C.POINTER(vp)],
        "swg_tables_bin_range": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "swg_tables_rebuild": [vp, vp, C.c_int, C.c_size_t],
        "swg_tables_rebuild_bins": [vp, vp, C.c_int, C.c_size_t, C.c_int],
        "swg_tables_rebuild_for": [vp, vp, C.c_int, C.c_size_t, C.c_int, vp],
        "swg_tables_built_bytes": [vp, C.POINTER(C.c_size_t)],
        "swg_tables_upload_i64": [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, C.POINTER(vp)],
        "swg_tables_destroy": [vp],
        "swg_tables_info": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                            C.POINTER(C.c_int), C.POINTER(C.c_size_t)],
        "swg_tables_export_i64": [vp, C.c_int, C.c_int, C.c_int, vp],
        "swg_tables_export_u32": [vp, C.c_int, C.c_int, C.c_int, vp],
        "swg_tables_export_f64": [vp, C.c_int, C.c_int, C.c_int, vp],
        "swg_tables_feature_image": [vp, vp],
        "swg_tables_device_layout": [vp, C.POINTER(vp), C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_size_t), C.POINTER(C.c_int)],
        "swg_query_terms": [vp, C.c_int, C.c_int, vp, vp],
        "swg_query_windows": [vp, C.c_int, vp, vp, C.POINTER(Kernel), C.c_int, C.c_int, vp],
        "swg_decay_windows": [vp, C.c_int, vp, vp, C.POINTER(Kernel), vp],
        "swg_tables_last_row": [vp, vp],
        "swg_tables_add_carry": [vp, C.c_int, vp],
        "swg_cake_windows": [vp, C.c_int, vp, vp, C.POINTER(Kernel), C.c_int, C.c_int, C.c_int,
                             vp],
        "swg_cake_plan": [C.POINTER(Kernel), C.c_int, C.c_int, vp, vp, vp],
        "swg_likelihood_maps": [vp, C.c_int, vp, vp, vp, vp, vp],
        "swg_likelihood_maps_async": [vp, C.c_int, vp, vp, vp, vp, vp],
        "swg_request_plan": [vp, vp, vp],
        "swg_request_groups": [vp, st, vp, vp],
        "swg_likelihood_batch": [vp, C.c_int, vp, C.c_int, C.c_size_t, C.c_int, vp, vp, vp],
        "swg_brute_windows": [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                              C.POINTER(Kernel), C.c_int, vp, vp],
        "swg_host_alloc": [C.c_size_t, C.POINTER(vp)],
        "swg_device_alloc": [C.c_size_t, C.POINTER(vp)],
        "swg_device_free": [vp],
        "swg_ipc_export": [vp, vp],
        "swg_ipc_import": [vp, C.POINTER(vp)],
        "swg_ipc_close": [vp],
        "swg_host_free": [vp],
    }.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/swg.h (for the load test)."""
    import re
    hdr = os.path.join(_build.ROOT, "include", "swg.h")
    return sorted(set(re.findall(r"\b(swg_[a-z0-9_]+)\s*\(", open(hdr).read())))


def _check(status):
    if status == 0:
        return
    L = lib()
    msg = L.swg_last_error().decode(errors="replace")
    cls = _BY_CODE.get(status, Error)
    if cls is CapacityError:
        raise CapacityError(msg, int(L.swg_last_required_bytes()))
    raise cls(msg, status) if cls is Error else cls(msg)


def _ptr(a):
    """Host numpy array -> (address, is_device=0); torch tensor -> device ptr."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(type(a))


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().swg_device_count(C.byref(n)))
    return n.value


class Context:
    """One device + one CUDA stream (swg_ctx)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().swg_ctx_create(device, C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            lib().swg_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().swg_ctx_synchronize(self._h))

    def set_stream(self, stream_ptr: Optional[int]):
        _check(lib().swg_ctx_set_stream(self._h, stream_ptr))

    @property
    def launches(self) -> int:
        n = C.c_uint64()
        _check(lib().swg_ctx_launch_count(self._h, C.byref(n)))
        return n.value

    @property
    def map_copies(self) -> int:
        """Device->host map copies issued so far (zero-copy maps issue none)."""
        n = C.c_uint64()
        _check(lib().swg_ctx_map_copy_count(self._h, C.byref(n)))
        return n.value

    def build(self, pixels, fmt=FMT_GRAY8, bins=16, planes=PLANES_AFFINE, budget=0,
              width=None, height=None, pitch=0) -> "Tables":
        return Tables(self, pixels, fmt, bins, planes, budget, width, height, pitch)

    def build_decay(self, pixels, decay, fmt=FMT_GRAY8, bins=16, budget=0, width=None,
                    height=None, pitch=0) -> "Tables":
        """Decayed directional tables for EXP_L1 maps with sigma == decay."""
        t = Tables.__new__(Tables)
        t.ctx = self
        t._h = C.c_void_p()
        is_dev, ptr, w, h = Tables._src(pixels, fmt, width, height)
        t._keep = pixels
        _check(lib().swg_tables_build_decay(self._h, ptr, is_dev, pitch, w, h, fmt, bins,
                                            float(decay), budget, C.byref(t._h)))
        t._info()
        t.decay = float(decay)
        return t

    def brute_windows(self, fi, bins, cx, cy, kernel, border=STRICT, integer=None):
        """swg_brute_windows: brute-force weighted histograms of explicit
        windows of a host feature image (BruteForcePlan, baselines.cpp:24-69).
        integer=True -> int64 counts (integer kernels), else fp64 sums."""
        fi = np.ascontiguousarray(fi, np.uint16)
        h, w = fi.shape
        cx = np.ascontiguousarray(cx, np.int32)
        cy = np.ascontiguousarray(cy, np.int32)
        if integer is None:
            integer = kernel.kind not in (GAUSS_CHEB, EXP_L1)
        out = np.empty((len(cx), bins), np.int64 if integer else np.float64)
        _check(lib().swg_brute_windows(self._h, _ptr(fi), w, h, bins, len(cx), _ptr(cx),
                                       _ptr(cy), C.byref(kernel), border,
                                       _ptr(out) if integer else None,
                                       None if integer else _ptr(out)))
        return out

    def build_bins(self, pixels, bin_begin, bin_end, fmt=FMT_GRAY8, bins=16,
                   planes=PLANES_AFFINE, decay=0.0, budget=0, width=None, height=None,
                   pitch=0) -> "Tables":
        """Tables for the quantiser's bins [bin_begin, bin_end) (bin-range
        sharding); maps chain through MapRequest.partial_in / partial_out."""
        t = Tables.__new__(Tables)
        t.ctx = self
        t._h = C.c_void_p()
        is_dev, ptr, w, h = Tables._src(pixels, fmt, width, height)
        t._keep = pixels
        _check(lib().swg_tables_build_bins(self._h, ptr, is_dev, pitch, w, h, fmt, bins, planes,
                                           float(decay), bin_begin, bin_end, budget,
                                           C.byref(t._h)))
        t._info()
        if planes == PLANES_DECAY:
            t.decay = float(decay)
        return t

    def upload_i64(self, plain, xramp, yramp) -> "Tables":
        plain, xramp, yramp = (np.ascontiguousarray(a, np.int64) for a in (plain, xramp, yramp))
        b, h1, w1 = plain.shape
        t = Tables.__new__(Tables)
        t.ctx = self
        t._h = C.c_void_p()
        _check(lib().swg_tables_upload_i64(self._h, w1 - 1, h1 - 1, b, _ptr(plain), _ptr(xramp),
                                           _ptr(yramp), C.byref(t._h)))
        t._info()
        return t


class Tables:
    """Device-resident integral tables (swg_tables)."""

    def __init__(self, ctx: Context, pixels, fmt, bins, planes, budget, width, height, pitch):
        self.ctx = ctx
        self._h = C.c_void_p()
        is_dev, ptr, w, h = self._src(pixels, fmt, width, height)
        self._keep = pixels
        _check(lib().swg_tables_build(ctx._h, ptr, is_dev, pitch, w, h, fmt, bins, planes, budget,
                                      C.byref(self._h)))
        self._info()

    @staticmethod
    def _src(pixels, fmt, width, height):
        if isinstance(pixels, np.ndarray):
            want = {FMT_GRAY8: np.uint8, FMT_RGB8: np.uint8}.get(fmt, np.uint16)
            if pixels.dtype != want or not pixels.flags.c_contiguous:
                raise TypeError(f"pixels must be C-contiguous {np.dtype(want).name}")
            h, w = pixels.shape[:2]
            return 0, pixels.ctypes.data, width or w, height or h
        # torch CUDA tensor (device-resident input)
        h, w = pixels.shape[:2]
        return (1 if pixels.is_cuda else 0), pixels.data_ptr(), width or w, height or h

    def _info(self):
        w, h, b, p = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nbytes = C.c_size_t()
        _check(lib().swg_tables_info(self._h, C.byref(w), C.byref(h), C.byref(b), C.byref(p),
                                     C.byref(nbytes)))
        self.width, self.height, self.bins, self.planes = w.value, h.value, b.value, p.value
        self.device_bytes = nbytes.value
        b0, b1, tot = C.c_int(), C.c_int(), C.c_int()
        _check(lib().swg_tables_bin_range(self._h, C.byref(b0), C.byref(b1), C.byref(tot)))
        self.bin_begin, self.bin_end, self.total_bins = b0.value, b1.value, tot.value

    def close(self):
        if getattr(self, "_h", None):
            lib().swg_tables_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rebuild(self, pixels, pitch=0):
        fmt = FMT_GRAY8
        is_dev = 0 if isinstance(pixels, np.ndarray) else int(pixels.is_cuda)
        self._keep = pixels
        _check(lib().swg_tables_rebuild(self._h, _ptr(pixels), is_dev, pitch))

    def rebuild_for(self, pixels, reqs, pitch=0):
        """swg_tables_rebuild_for: a new frame, building only the table units
        (octets / bin pairs) the requests' sweeps read; the rest are built on
        first use.  Returns nothing; built_bytes() reports the plane bytes."""
        is_dev = 0 if isinstance(pixels, np.ndarray) else int(pixels.is_cuda)
        self._keep = pixels
        creqs, _keep = self._creqs(reqs, self.total_bins)
        _check(lib().swg_tables_rebuild_for(self._h, _ptr(pixels), is_dev, pitch, len(reqs),
                                            C.addressof(creqs) if len(reqs) else None))

    def built_bytes(self) -> int:
        v = C.c_size_t(0)
        _check(lib().swg_tables_built_bytes(self._h, C.byref(v)))
        return int(v.value)

    def rebuild_bins(self, bin_begin, pixels=None, pitch=0):
        """Rebuild for bins [bin_begin, bin_begin + bins): from `pixels` (a
        new frame) or, by default, from the resident feature image."""
        is_dev = 0 if pixels is None or isinstance(pixels, np.ndarray) else int(pixels.is_cuda)
        if pixels is not None:
            self._keep = pixels
        _check(lib().swg_tables_rebuild_bins(self._h, _ptr(pixels) if pixels is not None
                                             else None, is_dev, pitch, bin_begin))
        self.bin_begin, self.bin_end = bin_begin, bin_begin + self.bins

    def export_i64(self, kind=TABLE_PLAIN, b0=0, b1=None):
        b1 = self.bins if b1 is None else b1
        out = np.empty((b1 - b0, self.height + 1, self.width + 1), np.int64)
        _check(lib().swg_tables_export_i64(self._h, kind, b0, b1, _ptr(out)))
        return out

    def export_f64(self, kind=0, b0=0, b1=None):
        """Decay tables: fp64 planes of orientation `kind` (0 SE .. 3 hv-flip)."""
        b1 = self.bins if b1 is None else b1
        out = np.empty((b1 - b0, self.height + 1, self.width + 1), np.float64)
        _check(lib().swg_tables_export_f64(self._h, kind, b0, b1, _ptr(out)))
        return out

    def export_u32(self, kind=TABLE_PLAIN, b0=0, b1=None):
        b1 = self.bins if b1 is None else b1
        out = np.empty((b1 - b0, self.height + 1, self.width + 1), np.uint32)
        _check(lib().swg_tables_export_u32(self._h, kind, b0, b1, _ptr(out)))
        return out

    def feature_image(self):
        out = np.empty((self.height, self.width), np.uint16)
        _check(lib().swg_tables_feature_image(self._h, _ptr(out)))
        return out

    def query_terms(self, terms: Sequence[Sequence[tuple]]):
        """terms[w] = list of (valid, x0, y0, x1, y1, sx, sy, beta)."""
        n = len(terms)
        tpw = max(1, max((len(t) for t in terms), default=1))
        arr = (Term * (n * tpw))()
        for i, ts in enumerate(terms):
            for k, t in enumerate(ts):
                arr[i * tpw + k] = Term(*t)
        out = np.empty((n, self.bins), np.int64)
        _check(lib().swg_query_terms(self._h, n, tpw, C.addressof(arr), _ptr(out)))
        return out

    def query_windows(self, cx, cy, kernel: Kernel, method=SWIH, border=STRICT):
        cx = np.ascontiguousarray(np.atleast_1d(cx), np.int32)
        cy = np.ascontiguousarray(np.atleast_1d(cy), np.int32)
        out = np.empty((len(cx), self.bins), np.int64)
        _check(lib().swg_query_windows(self._h, len(cx), _ptr(cx), _ptr(cy), C.byref(kernel),
                                       method, border, _ptr(out)))
        return out

    def last_row(self, out=None):
        """Device uint32 tensor (octets, planes, width+1, 8): this band's last
        record row (swg_tables_last_row)."""
        import torch
        if out is None:
            out = torch.empty((-(-self.bins // 8), self.planes, self.width + 1, 8),
                              dtype=torch.int32, device="cuda")
        _check(lib().swg_tables_last_row(self._h, C.c_void_p(out.data_ptr())))
        return out

    def add_carry(self, y0, carry):
        """Local band tables -> global rows y0.. (swg_tables_add_carry)."""
        _check(lib().swg_tables_add_carry(self._h, int(y0), C.c_void_p(carry.data_ptr())))

    def decay_windows(self, cx, cy, kernel: Kernel):
        """Exponential-kernel window histograms (strict) from decayed tables."""
        cx = np.ascontiguousarray(np.atleast_1d(cx), np.int32)
        cy = np.ascontiguousarray(np.atleast_1d(cy), np.int32)
        out = np.empty((len(cx), self.bins), np.float64)
        _check(lib().swg_decay_windows(self._h, len(cx), _ptr(cx), _ptr(cy), C.byref(kernel),
                                       _ptr(out)))
        return out

    def cake_windows(self, cx, cy, kernel: Kernel, rings, rule=RING_MEAN, border=STRICT):
        cx = np.ascontiguousarray(np.atleast_1d(cx), np.int32)
        cy = np.ascontiguousarray(np.atleast_1d(cy), np.int32)
        out = np.empty((len(cx), self.bins), np.float64)
        _check(lib().swg_cake_windows(self._h, len(cx), _ptr(cx), _ptr(cy), C.byref(kernel),
                                      rings, rule, border, _ptr(out)))
        return out

    def map_shape(self, kernel: Kernel, rows=None):
        mw, mh = self.width - kernel.kw + 1, self.height - kernel.kh + 1
        r0, r1 = rows if rows else (0, mh)
        return (r1 - r0, mw)

    def likelihood_maps(self, reqs: Sequence[MapRequest], scores: str = "host",
                        scores_dev=None, peaks_dev=None):
        """Run len(reqs) map requests.  scores="host" returns numpy maps
        (pageable memory: the library copies them), "pinned" the same in
        page-locked memory (the sweeps write them directly), "none" skips them
        (peaks only); device outputs may be given as torch tensors (then the
        call is asynchronous).  Returns (maps, peaks)."""
        n = len(reqs)
        creqs, _keep = self._creqs(reqs, self.total_bins)
        maps = [None] * n
        host_ptrs = None
        pinned = []
        if any(min(self.map_shape(r.kernel, r.rows)) <= 0 for r in reqs):
            scores = "none"  # invalid geometry: let the library raise SizeError
        if scores in ("host", "pinned"):
            host_ptrs = (C.c_void_p * n)()
            for i, r in enumerate(reqs):
                if r.partial_out is None:
                    shape = self.map_shape(r.kernel, r.rows)
                    if scores == "pinned":
                        pinned.append(PinnedBuffer(shape, np.float64))
                        maps[i] = pinned[-1].array
                    else:
                        maps[i] = np.empty(shape, np.float64)
                    host_ptrs[i] = maps[i].ctypes.data
        dev_ptrs = None
        if scores_dev is not None:
            dev_ptrs = (C.c_void_p * n)(*[_ptr(x) for x in scores_dev])
        peaks = (Peak * n)() if peaks_dev is None else None
        _check(lib().swg_likelihood_maps(
            self._h, n, C.addressof(creqs),
            C.addressof(host_ptrs) if host_ptrs is not None else None,
            C.addressof(dev_ptrs) if dev_ptrs is not None else None,
            C.addressof(peaks) if peaks is not None else None,
            _ptr(peaks_dev) if peaks_dev is not None else None))
        if pinned:  # own copies: the page-locked buffers are freed with `pinned`
            maps = [None if m is None else m.copy() for m in maps]
        if peaks is None:
            return maps, None
        return maps, [None if r.partial_out is not None else p.astuple()
                      for p, r in zip(peaks, reqs)]

    def request_plan(self, req: "MapRequest") -> dict:
        """What likelihood_maps runs for `req` (swg_request_plan): sweep
        kernel, planes read, bytes per entry, bins whose records are read,
        CTAs."""
        creqs, _keep = self._creqs([req], self.total_bins)
        out = _PlanInfo()
        _check(lib().swg_request_plan(self._h, C.addressof(creqs), C.byref(out)))
        return {"kernel": out.kernel.decode(), "planes": out.planes,
                "entry_bytes": out.entry_bytes, "bins_read": out.bins_read, "ctas": out.ctas}

    def request_groups(self, reqs: Sequence["MapRequest"]) -> list:
        """swg_request_groups: per request, the multi-scale cake launch it
        joins in one likelihood_maps call (-1: its own launch)."""
        creqs, _keep = self._creqs(reqs, self.total_bins)
        out = (C.c_int * len(reqs))()
        _check(lib().swg_request_groups(self._h, len(reqs), C.addressof(creqs), out))
        return list(out)

    @staticmethod
    def _creqs(reqs, bins):
        creqs = (_Req * len(reqs))()
        models = []
        for i, r in enumerate(reqs):
            m = np.ascontiguousarray(r.model, np.float64)
            if m.shape != (bins,):
                raise ModelError(f"likelihood map: model must be normalized with {bins} bins")
            models.append(m)
            r0, r1 = r.rows if r.rows else (0, 0)
            creqs[i] = _Req(r.kernel, r.method, r.sim, r.rings, r.ring_rule, r0, r1,
                            m.ctypes.data_as(C.POINTER(C.c_double)),
                            _ptr(r.partial_in) if r.partial_in is not None else None,
                            _ptr(r.partial_out) if r.partial_out is not None else None)
        return creqs, models

    def likelihood_batch(self, frames, reqs: Sequence[MapRequest], pitch=0, is_device=None,
                         peaks_dev=None):
        """swg_likelihood_batch: rebuild from each frame (numpy arrays / torch
        tensors, or raw addresses with is_device given) and run `reqs`, peaks
        only.  Returns peaks[f][i] (host) unless peaks_dev is given."""
        addrs = []
        for f in frames:
            if isinstance(f, int):
                addrs.append(f)
            else:
                addrs.append(_ptr(f))
                if is_device is None:
                    is_device = 0 if isinstance(f, np.ndarray) else int(f.is_cuda)
        nf, n = len(frames), len(reqs)
        fr = (C.c_void_p * max(nf, 1))(*addrs)
        creqs, _keep = self._creqs(reqs, self.total_bins)
        peaks = (Peak * (nf * n))() if peaks_dev is None else None
        _check(lib().swg_likelihood_batch(
            self._h, nf, C.addressof(fr), int(is_device or 0), pitch, n, C.addressof(creqs),
            C.addressof(peaks) if peaks is not None else None,
            _ptr(peaks_dev) if peaks_dev is not None else None))
        if peaks is None:
            return None
        return [[peaks[f * n + i].astuple() for i in range(n)] for f in range(nf)]

    def likelihood_map(self, kernel, model, method=SWIH, sim=BHATTACHARYYA, rings=4,
                       ring_rule=RING_MEAN, rows=None):
        maps, peaks = self.likelihood_maps([MapRequest(kernel, model, method, sim, rings,
                                                       ring_rule, rows)])
        return maps[0], peaks[0]


class PinnedBuffer:
    """Page-locked host memory from libswg's own CUDA runtime
    (swg_host_alloc); exposed as a numpy array."""

    def __init__(self, shape, dtype):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self._p = C.c_void_p()
        _check(lib().swg_host_alloc(max(self.nbytes, 1), C.byref(self._p)))
        buf = (C.c_char * max(self.nbytes, 1)).from_address(self._p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            if self._p:
                lib().swg_host_free(self._p)
        except Exception:
            pass


def cake_plan(kernel: Kernel, rings: int, rule=RING_MEAN):
    sx = np.zeros(max(rings, 1), np.int32)
    sy = np.zeros(max(rings, 1), np.int32)
    rw = np.zeros(max(rings, 1), np.float64)
    _check(lib().swg_cake_plan(C.byref(kernel), rings, rule, _ptr(sx), _ptr(sy), _ptr(rw)))
    return sx, sy, rw


def device_alloc(nbytes: int) -> int:
    """Raw device allocation (its own base address, so its IPC handle maps
    exactly this buffer); free with device_free."""
    p = C.c_void_p()
    _check(lib().swg_device_alloc(nbytes, C.byref(p)))
    return p.value


def device_free(address: int) -> None:
    _check(lib().swg_device_free(address))


def ipc_export(tensor) -> bytes:
    """Handle of a device allocation for another process (swg_ipc_export)."""
    buf = (C.c_ubyte * 64)()
    _check(lib().swg_ipc_export(_ptr(tensor), buf))
    return bytes(buf)


def ipc_import(handle: bytes) -> int:
    """Map another process's device allocation; returns its device address
    (pass it anywhere a device pointer is taken, e.g. MapRequest.partial_out)."""
    buf = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().swg_ipc_import(buf, C.byref(p)))
    return p.value


def ipc_close(address: int) -> None:
    _check(lib().swg_ipc_close(address))
