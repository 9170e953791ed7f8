"""ctypes bindings for the parity checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle`` — our C restatement (``oracle/liboracle.so``, swih_oracle.c).
* ``Ref``    — the unmodified reference library compiled from
  /root/reference/proj/src (``oracle/_ref/libswihref.so``, see Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libswihref.so")

UNIFORM, MANHATTAN, CHEBYSHEV, GAUSS_CHEB = 0, 1, 2, 3
EUCLID_QUAD, EXP_L1 = 4, 5  # declared extensions (parity unpinned)
SWIH, BRUTE, CAKE, PLAIN = 0, 1, 2, 3
BHATTACHARYYA, INTERSECTION = 0, 1
STRICT, CLIPPED = 0, 1
RING_MEAN, RING_LEVEL = 0, 1

_p = np.ctypeslib.ndpointer
_u8 = _p(np.uint8, flags="C_CONTIGUOUS")
_u16 = _p(np.uint16, flags="C_CONTIGUOUS")
_i64 = _p(np.int64, flags="C_CONTIGUOUS")
_f64 = _p(np.float64, flags="C_CONTIGUOUS")
_i32 = _p(np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


class _Kernel(C.Structure):
    _fields_ = [("kind", C.c_int), ("kw", C.c_int), ("kh", C.c_int), ("sigma", C.c_double)]


class _Peak(C.Structure):
    _fields_ = [("map_x", C.c_int), ("map_y", C.c_int), ("center_x", C.c_int),
                ("center_y", C.c_int), ("score", C.c_double)]


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle).  The reference part only when
    /root/reference is present (this container; the GPU box uses the
    prebuilt .so that gpurun ships)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
        # the reference's own unit tests against libswih_b200.so (built first)
        if os.path.exists(os.path.join(HERE, "..", "paper_1705_03524_b200", "lib",
                                       "libswih_b200.so")):
            targets.append("reftests")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def kernel(kind, kw, kh=None, sigma=0.5):
    return _Kernel(kind, kw, kw if kh is None else kh, sigma)


class Oracle:
    """Restated reference algorithm (swih_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        K = C.POINTER(_Kernel)
        L.orc_random_gray.argtypes = [C.c_int, C.c_int, C.c_uint64, _u8]
        L.orc_quantize_gray8.argtypes = [_u8, C.c_size_t, C.c_int, _u16]
        L.orc_quantize_gray16.argtypes = [_u16, C.c_size_t, C.c_int, _u16]
        L.orc_quantize_rgb8.argtypes = [_u8, C.c_size_t, C.c_int, _u16]
        L.orc_weight_at.argtypes = [K, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.orc_kernel_weight_sum.argtypes = [K, C.POINTER(C.c_double)]
        L.orc_build_tables.argtypes = [_u16, C.c_int, C.c_int, C.c_int, _i64, _i64, _i64]
        L.orc_swih_query.argtypes = [_i64, _i64, _i64, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, K, C.c_int, _i64]
        L.orc_plain_query.argtypes = [_i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      K, C.c_int, _i64]
        L.orc_brute_counts.argtypes = [_u16, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       K, C.c_int, _i64]
        L.orc_brute_weights.argtypes = [_u16, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        K, C.c_int, _f64]
        L.orc_cake_plan.argtypes = [K, C.c_int, C.c_int, _i32, _i32, _f64]
        L.orc_cake_histogram.argtypes = [_i64, C.c_int, C.c_int, C.c_int, K, C.c_int,
                                         _i32, _i32, _f64, C.c_int, C.c_int, C.c_int, _f64]
        L.orc_score_counts.argtypes = [C.c_int, _f64, _i64, C.c_int, C.POINTER(C.c_double)]
        L.orc_score_weights.argtypes = [C.c_int, _f64, _f64, C.c_int, C.POINTER(C.c_double)]
        L.orc_similarity.argtypes = [C.c_int, _f64, _f64, C.c_int, C.POINTER(C.c_double)]
        L.orc_normalize.argtypes = [_f64, C.c_int, _f64]
        L.orc_target_model.argtypes = [_u16, C.c_int, C.c_int, C.c_int, K, C.c_int,
                                       C.c_int, C.c_int, _f64]
        L.orc_likelihood_map.argtypes = [_u16, C.c_int, C.c_int, C.c_int, _f64, C.c_int, K,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, _f64]
        L.orc_likelihood_map_mt.argtypes = [_u16, C.c_int, C.c_int, C.c_int, _f64, K,
                                            C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_int, _f64]
        L.orc_peak.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_Peak)]
        L.orc_fast_map.argtypes = [_u16, C.c_int, C.c_int, C.c_int, _f64, K, C.c_int,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _f64,
                                   C.POINTER(_Peak), C.POINTER(C.c_longlong)]

    @staticmethod
    def _check(st):
        if st:
            raise OracleError(st)

    def random_gray(self, w, h, seed):
        out = np.empty((h, w), np.uint8)
        self.lib.orc_random_gray(w, h, seed, out)
        return out

    def quantize_gray8(self, img, bins):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.empty(img.shape, np.uint16)
        self._check(self.lib.orc_quantize_gray8(img, img.size, bins, out))
        return out

    def quantize_gray16(self, img, bins):
        img = np.ascontiguousarray(img, np.uint16)
        out = np.empty(img.shape, np.uint16)
        self._check(self.lib.orc_quantize_gray16(img, img.size, bins, out))
        return out

    def quantize_rgb8(self, img, levels):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.empty(img.shape[:2], np.uint16)
        self._check(self.lib.orc_quantize_rgb8(img, img.shape[0] * img.shape[1], levels, out))
        return out

    def weight_at(self, k, dx, dy):
        w = C.c_double()
        self._check(self.lib.orc_weight_at(C.byref(k), dx, dy, C.byref(w)))
        return w.value

    def kernel_weight_sum(self, k):
        w = C.c_double()
        self._check(self.lib.orc_kernel_weight_sum(C.byref(k), C.byref(w)))
        return w.value

    def build_tables(self, fi, bins):
        fi = np.ascontiguousarray(fi, np.uint16)
        h, w = fi.shape
        shape = (bins, h + 1, w + 1)
        p, x, y = (np.empty(shape, np.int64) for _ in range(3))
        self.lib.orc_build_tables(fi, w, h, bins, p, x, y)
        return p, x, y

    def swih_query(self, tables, cx, cy, k, border=STRICT):
        p, x, y = tables
        b, h1, w1 = p.shape
        out = np.empty(b, np.int64)
        self._check(self.lib.orc_swih_query(p, x, y, w1 - 1, h1 - 1, b, cx, cy,
                                            C.byref(k), border, out))
        return out

    def plain_query(self, tables, cx, cy, k, border=STRICT):
        p = tables[0]
        b, h1, w1 = p.shape
        out = np.empty(b, np.int64)
        self._check(self.lib.orc_plain_query(p, w1 - 1, h1 - 1, b, cx, cy, C.byref(k),
                                             border, out))
        return out

    def brute_counts(self, fi, bins, cx, cy, k, border=STRICT):
        fi = np.ascontiguousarray(fi, np.uint16)
        out = np.empty(bins, np.int64)
        self._check(self.lib.orc_brute_counts(fi, fi.shape[1], fi.shape[0], bins, cx, cy,
                                              C.byref(k), border, out))
        return out

    def brute_weights(self, fi, bins, cx, cy, k, border=STRICT):
        fi = np.ascontiguousarray(fi, np.uint16)
        out = np.empty(bins, np.float64)
        self._check(self.lib.orc_brute_weights(fi, fi.shape[1], fi.shape[0], bins, cx, cy,
                                               C.byref(k), border, out))
        return out

    def cake_plan(self, k, rings, rule=RING_MEAN):
        sx = np.zeros(max(rings, 1), np.int32)
        sy = np.zeros(max(rings, 1), np.int32)
        rw = np.zeros(max(rings, 1), np.float64)
        self._check(self.lib.orc_cake_plan(C.byref(k), rings, rule, sx, sy, rw))
        return sx, sy, rw

    def cake_histogram(self, tables, k, rings, rule, cx, cy, border=STRICT):
        p = tables[0]
        b, h1, w1 = p.shape
        sx, sy, rw = self.cake_plan(k, rings, rule)
        out = np.empty(b, np.float64)
        self._check(self.lib.orc_cake_histogram(p, w1 - 1, h1 - 1, b, C.byref(k), rings,
                                                sx, sy, rw, cx, cy, border, out))
        return out

    def score_counts(self, sim, model, raw):
        s = C.c_double()
        self._check(self.lib.orc_score_counts(sim, np.ascontiguousarray(model, np.float64),
                                              np.ascontiguousarray(raw, np.int64),
                                              len(raw), C.byref(s)))
        return s.value

    def score_weights(self, sim, model, raw):
        s = C.c_double()
        self._check(self.lib.orc_score_weights(sim, np.ascontiguousarray(model, np.float64),
                                               np.ascontiguousarray(raw, np.float64),
                                               len(raw), C.byref(s)))
        return s.value

    def similarity(self, sim, p, q):
        s = C.c_double()
        self._check(self.lib.orc_similarity(sim, np.ascontiguousarray(p, np.float64),
                                            np.ascontiguousarray(q, np.float64), len(p),
                                            C.byref(s)))
        return s.value

    def normalize(self, h):
        h = np.ascontiguousarray(h, np.float64)
        out = np.empty_like(h)
        self._check(self.lib.orc_normalize(h, len(h), out))
        return out

    def target_model(self, templ_fi, bins, k, method=SWIH, rings=1, rule=RING_MEAN):
        t = np.ascontiguousarray(templ_fi, np.uint16)
        out = np.empty(bins, np.float64)
        self._check(self.lib.orc_target_model(t, t.shape[1], t.shape[0], bins, C.byref(k),
                                              method, rings, rule, out))
        return out

    def likelihood_map(self, fi, bins, model, k, method=SWIH, sim=BHATTACHARYYA,
                       rings=1, rule=RING_MEAN, rows=None, threads=1, normalized=True):
        fi = np.ascontiguousarray(fi, np.uint16)
        h, w = fi.shape
        mw, mh = w - k.kw + 1, h - k.kh + 1
        v0, v1 = rows if rows else (0, mh)
        out = np.empty((max(v1 - v0, 0), max(mw, 0)), np.float64)
        model = np.ascontiguousarray(model, np.float64)
        if threads > 1:
            st = self.lib.orc_likelihood_map_mt(fi, w, h, bins, model, C.byref(k), method,
                                                sim, rings, rule, v0, v1, threads, out)
        else:
            st = self.lib.orc_likelihood_map(fi, w, h, bins, model, int(normalized),
                                             C.byref(k), method, sim, rings, rule, v0,
                                             v1, out)
        self._check(st)
        return out

    def fast_map(self, fi, bins, model, k, method=SWIH, sim=BHATTACHARYYA, rings=1,
                 rule=RING_MEAN, threads=None, eps=1e-8):
        """Full strict map computed bin-outer (swih_fastmap.c): bit-identical
        to likelihood_map for the exact methods; for the exponential brute
        force a tolerance map with every window within `eps` of its maximum
        re-scored exactly.  Returns (map, peak tuple, re-scored count)."""
        fi = np.ascontiguousarray(fi, np.uint16)
        h, w = fi.shape
        out = np.empty((h - k.kh + 1, w - k.kw + 1), np.float64)
        p, n = _Peak(), C.c_longlong(0)
        self._check(self.lib.orc_fast_map(fi, w, h, bins, np.ascontiguousarray(model, np.float64),
                                          C.byref(k), method, sim, rings, rule,
                                          threads or os.cpu_count(), eps, out, C.byref(p),
                                          C.byref(n)))
        return out, (p.map_x, p.map_y, p.center_x, p.center_y, p.score), n.value

    def peak(self, scores, hx, hy):
        scores = np.ascontiguousarray(scores, np.float64)
        p = _Peak()
        self._check(self.lib.orc_peak(scores, scores.shape[1], scores.shape[0], hx, hy,
                                      C.byref(p)))
        return (p.map_x, p.map_y, p.center_x, p.center_y, p.score)


class Ref:
    """The reference library itself (oracle/_ref/libswihref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_required_bytes.restype = C.c_size_t
        L.ref_random_gray.argtypes = [C.c_int, C.c_int, C.c_uint64, _u8]
        L.ref_quantize.argtypes = [_u8, C.c_int, C.c_int, C.c_int, _u16]
        L.ref_weight_at.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.POINTER(C.c_double)]
        L.ref_kernel_weight_sum.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.POINTER(C.c_double)]
        L.ref_tables_new.argtypes = [_u16, C.c_int, C.c_int, C.c_int, C.c_size_t,
                                     C.POINTER(vp)]
        L.ref_tables_free.argtypes = [vp]
        L.ref_tables_export.argtypes = [vp, C.c_int, _i64]
        L.ref_tables_cell.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_int64)]
        L.ref_rect_sum.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_int64)]
        L.ref_directional.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_int64)]
        L.ref_tables_save.argtypes = [vp, C.c_char_p]
        L.ref_tables_load.argtypes = [C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_write_map_files.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                          C.c_char_p]
        L.ref_write_bench_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_double, C.c_double, C.c_double,
                                          C.c_char_p]
        L.ref_swih_query.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, _i64]
        L.ref_plain_query.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i64]
        L.ref_quadrant_histogram.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_int64, C.c_int64, C.c_int64, _f64]
        L.ref_cake_histogram.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_int, _f64]
        L.ref_cake_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                    _i32, _i32, _f64]
        L.ref_brute_counts.argtypes = [_u16, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _i64]
        L.ref_brute_weights.argtypes = [_u16, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _f64]
        L.ref_similarity.argtypes = [C.c_int, _f64, _f64, C.c_int, C.POINTER(C.c_double)]
        L.ref_normalize.argtypes = [_f64, C.c_int, _f64]
        L.ref_target_model.argtypes = [_u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _f64]
        L.ref_likelihood_map.argtypes = [_u8, C.c_int, C.c_int, C.c_int, _f64, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t,
                                         vp, _i32, C.POINTER(C.c_double)]
        L.ref_peak.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_int, _i32,
                               C.POINTER(C.c_double)]
        L.ref_sweep_rows.argtypes = [vp, _f64, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_int, _f64]

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def random_gray(self, w, h, seed):
        out = np.empty((h, w), np.uint8)
        self.lib.ref_random_gray(w, h, seed, out)
        return out

    def quantize(self, img, bins):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.empty(img.shape, np.uint16)
        self._check(self.lib.ref_quantize(img, img.shape[1], img.shape[0], bins, out))
        return out

    def weight_at(self, k, dx, dy):
        w = C.c_double()
        self._check(self.lib.ref_weight_at(k.kind, k.kw, k.kh, k.sigma, dx, dy, C.byref(w)))
        return w.value

    def kernel_weight_sum(self, k):
        w = C.c_double()
        self._check(self.lib.ref_kernel_weight_sum(k.kind, k.kw, k.kh, k.sigma, C.byref(w)))
        return w.value

    def tables(self, fi, bins, budget=0):
        return RefTables(self, fi, bins, budget)

    def brute_counts(self, fi, bins, cx, cy, k, border=STRICT):
        fi = np.ascontiguousarray(fi, np.uint16)
        out = np.empty(bins, np.int64)
        self._check(self.lib.ref_brute_counts(fi, fi.shape[1], fi.shape[0], bins, cx, cy,
                                              k.kind, k.kw, k.kh, k.sigma, border, out))
        return out

    def brute_weights(self, fi, bins, cx, cy, k, border=STRICT):
        fi = np.ascontiguousarray(fi, np.uint16)
        out = np.empty(bins, np.float64)
        self._check(self.lib.ref_brute_weights(fi, fi.shape[1], fi.shape[0], bins, cx, cy,
                                               k.kind, k.kw, k.kh, k.sigma, border, out))
        return out

    def cake_plan(self, k, rings, rule=RING_MEAN):
        sx = np.zeros(max(rings, 1), np.int32)
        sy = np.zeros(max(rings, 1), np.int32)
        rw = np.zeros(max(rings, 1), np.float64)
        self._check(self.lib.ref_cake_plan(k.kind, k.kw, k.kh, k.sigma, rings, rule,
                                           sx, sy, rw))
        return sx, sy, rw

    def similarity(self, sim, p, q):
        s = C.c_double()
        self._check(self.lib.ref_similarity(sim, np.ascontiguousarray(p, np.float64),
                                            np.ascontiguousarray(q, np.float64), len(p),
                                            C.byref(s)))
        return s.value

    def normalize(self, h):
        h = np.ascontiguousarray(h, np.float64)
        out = np.empty_like(h)
        self._check(self.lib.ref_normalize(h, len(h), out))
        return out

    def target_model(self, templ, bins, k, method=SWIH, rings=1, rule=RING_MEAN):
        t = np.ascontiguousarray(templ, np.uint8)
        out = np.empty(bins, np.float64)
        self._check(self.lib.ref_target_model(t, t.shape[1], t.shape[0], bins, k.kind, k.kw,
                                              k.kh, k.sigma, method, rings, rule, out))
        return out

    def likelihood_map(self, img, bins, model, k, method=SWIH, sim=BHATTACHARYYA,
                       rings=1, rule=RING_MEAN, threads=1, budget=0, normalized=True,
                       want_scores=True):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        mw, mh = w - k.kw + 1, h - k.kh + 1
        out = np.empty((max(mh, 0), max(mw, 0)), np.float64) if want_scores else None
        pk = np.zeros(4, np.int32)
        ps = C.c_double()
        self._check(self.lib.ref_likelihood_map(
            img, w, h, bins, np.ascontiguousarray(model, np.float64), int(normalized),
            k.kind, k.kw, k.kh, k.sigma, method, sim, rings, rule, threads, budget,
            out.ctypes.data_as(C.c_void_p) if out is not None else None, pk, C.byref(ps)))
        return out, (int(pk[0]), int(pk[1]), int(pk[2]), int(pk[3]), ps.value)

    def load_tables(self, path):
        """IntegralTableSet::load_file -> (w, h, bins, plain, xramp, yramp) int64."""
        h_, w, hh, b = C.c_void_p(), C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.ref_tables_load(path.encode(), C.byref(h_), C.byref(w),
                                             C.byref(hh), C.byref(b)))
        try:
            out = []
            for kind in range(3):
                a = np.empty((b.value, hh.value + 1, w.value + 1), np.int64)
                self._check(self.lib.ref_tables_export(h_, kind, a))
                out.append(a)
        finally:
            self.lib.ref_tables_free(h_)
        return (w.value, hh.value, b.value, *out)

    def write_map_files(self, scores, hx, hy, csv_path=None, pgm_path=None):
        """write_map_csv_file / write_pgm_file(map_to_gray) of a map."""
        scores = np.ascontiguousarray(scores, np.float64)
        self._check(self.lib.ref_write_map_files(
            scores, scores.shape[1], scores.shape[0], hx, hy,
            csv_path.encode() if csv_path else None, pgm_path.encode() if pgm_path else None))

    def write_bench_csv(self, rec, path):
        """write_bench_csv_header + write_bench_csv_row of one record."""
        self._check(self.lib.ref_write_bench_csv(
            rec["method"].encode(), rec["width"], rec["height"], rec["kw"], rec["kh"],
            rec["bins"], rec["build_ms"], rec["query_total_ms"], rec["query_mean_us"],
            path.encode()))

    def peak(self, scores, hx, hy):
        scores = np.ascontiguousarray(scores, np.float64)
        pk = np.zeros(4, np.int32)
        ps = C.c_double()
        self._check(self.lib.ref_peak(scores, scores.shape[1], scores.shape[0], hx, hy, pk,
                                      C.byref(ps)))
        return (int(pk[0]), int(pk[1]), int(pk[2]), int(pk[3]), ps.value)


class RefTables:
    def __init__(self, ref: Ref, fi, bins, budget=0):
        self.ref = ref
        fi = np.ascontiguousarray(fi, np.uint16)
        self.h, self.w = fi.shape
        self.bins = bins
        self.h_ = C.c_void_p()
        ref._check(ref.lib.ref_tables_new(fi, self.w, self.h, bins, budget, C.byref(self.h_)))

    def __del__(self):
        if getattr(self, "h_", None) and self.h_.value:
            self.ref.lib.ref_tables_free(self.h_)
            self.h_ = None

    def export(self, kind):
        out = np.empty((self.bins, self.h + 1, self.w + 1), np.int64)
        self.ref._check(self.ref.lib.ref_tables_export(self.h_, kind, out))
        return out

    def cell(self, kind, x, y, b):
        v = C.c_int64()
        self.ref._check(self.ref.lib.ref_tables_cell(self.h_, kind, x, y, b, C.byref(v)))
        return v.value

    def rect_sum(self, kind, x0, y0, x1, y1, b):
        v = C.c_int64()
        self.ref._check(self.ref.lib.ref_rect_sum(self.h_, kind, x0, y0, x1, y1, b,
                                                  C.byref(v)))
        return v.value

    def directional(self, d, x, y, b):
        v = C.c_int64()
        self.ref._check(self.ref.lib.ref_directional(self.h_, d, x, y, b, C.byref(v)))
        return v.value

    def save(self, path):
        self.ref._check(self.ref.lib.ref_tables_save(self.h_, path.encode()))

    def swih_query(self, cx, cy, k, border=STRICT):
        out = np.empty(self.bins, np.int64)
        self.ref._check(self.ref.lib.ref_swih_query(self.h_, cx, cy, k.kind, k.kw, k.kh,
                                                    k.sigma, border, out))
        return out

    def plain_query(self, cx, cy, kw, kh, border=STRICT):
        out = np.empty(self.bins, np.int64)
        self.ref._check(self.ref.lib.ref_plain_query(self.h_, cx, cy, kw, kh, border, out))
        return out

    def quadrant_histogram(self, rect, sx, sy, beta):
        out = np.empty(self.bins, np.float64)
        valid = rect is not None
        x0, y0, x1, y1 = rect if valid else (0, 0, 0, 0)
        self.ref._check(self.ref.lib.ref_quadrant_histogram(self.h_, int(valid), x0, y0, x1,
                                                            y1, sx, sy, beta, out))
        return out

    def cake_histogram(self, k, rings, rule, cx, cy, border=STRICT):
        out = np.empty(self.bins, np.float64)
        self.ref._check(self.ref.lib.ref_cake_histogram(self.h_, k.kind, k.kw, k.kh, k.sigma,
                                                        rings, rule, cx, cy, border, out))
        return out

    def sweep_rows(self, model, k, method, sim, rings, rule, threads, v0, v1):
        mw = self.w - k.kw + 1
        out = np.empty((v1 - v0, mw), np.float64)
        self.ref._check(self.ref.lib.ref_sweep_rows(
            self.h_, np.ascontiguousarray(model, np.float64), k.kind, k.kw, k.kh, k.sigma,
            method, sim, rings, rule, threads, v0, v1, out))
        return out
