"""GPU tests of the build kernels' shape-dependent paths.

The band column sums (K1a `k_colsum`, K1a' `k_colsum_decay`) keep a thread's
per-bin sums in shared memory and walk the bins in chunks of as many octets /
pairs as the shared memory holds; the decayed build (`k_build_decay_warp`)
gives a CTA fewer warps when the bands are tall (one carry per band row and
warp in shared memory).  The BASELINE configs never leave one chunk or eight
warps, so these shapes are forced here and compared with a numpy
restatement of the tables (`integral_tables.cpp:72-115` for the integer
planes; the decayed prefix sums of DESIGN.md for the declared exponential
kernel).
"""
import numpy as np
import pytest

from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu


def _u16_image(w, h, seed):
    return np.random.default_rng(seed).integers(0, 65536, size=(h, w), dtype=np.uint16)


def _integer_plane(fi, b, kind):
    """(H+1) x (W+1) inclusive 2-D prefix sums of bin b's weight plane (exact)."""
    h, w = fi.shape
    one = (fi == b).astype(np.int64)
    x = np.arange(w, dtype=np.int64)[None, :]
    y = np.arange(h, dtype=np.int64)[:, None]
    wgt = (one, one * x, one * y, one * x * x, one * y * y)[kind]
    out = np.zeros((h + 1, w + 1), np.int64)
    out[1:, 1:] = wgt.cumsum(0).cumsum(1)
    return out


def _check_plane(t, fi, b, kind):
    """The 32-bit planes the sweeps read (kinds 0-2: mod 2^32) and the exact
    int64 export (every kind) against numpy."""
    want = _integer_plane(fi, b, kind)
    if kind < 3:
        got = t.export_u32(kind, b, b + 1)[0]
        assert (got == (want & 0xFFFFFFFF).astype(np.uint32)).all(), (b, kind)
    else:
        assert (t.export_i64(kind, b, b + 1)[0] == want).all(), (b, kind)


def _decayed_plane(f, b, d):
    """E(X, Y) = sum_{x < X, y < Y} [f == b] d^(X-1-x) d^(Y-1-y)."""
    h, w = f.shape
    one = (f == b).astype(np.float64)
    r = np.zeros((h, w + 1))
    for x in range(w):
        r[:, x + 1] = d * r[:, x] + one[:, x]
    out = np.zeros((h + 1, w + 1))
    for y in range(h):
        out[y + 1] = d * out[y] + r[y]
    return out


@pytest.mark.parametrize("planes,kinds", [(swg.PLANES_PLAIN, 1), (swg.PLANES_AFFINE, 3),
                                          (swg.PLANES_QUADRATIC, 5)])
def test_integer_column_sums_in_chunks(ctx, planes, kinds):
    """200 bins = 25 octets: more than one shared-memory chunk of column sums
    for every carry layout (24 / 12 / 8 octets per chunk), many bands."""
    bins, w, h = 200, 150, 700
    img = _u16_image(w, h, 5)
    t = ctx.build(img, swg.FMT_GRAY16, bins, planes)
    fi = t.feature_image()
    assert fi.shape == (h, w) and fi.max() < bins
    for b in (0, 7, 8, 95, 96, 103, 191, 192, 199):  # first / last bins of several chunks
        for kind in range(kinds):
            _check_plane(t, fi, b, kind)


def test_integer_column_sums_selected_octets(ctx):
    """A selective rebuild sums only the octets it builds; an export then
    builds the rest (their own column sums) and everything equals numpy."""
    bins, w, h = 72, 130, 500
    img0, img1 = _u16_image(w, h, 6), _u16_image(w, h, 7)
    t = ctx.build(img0, swg.FMT_GRAY16, bins, swg.PLANES_QUADRATIC)
    model = np.zeros(bins)
    model[[2, 40, 41, 70]] = 0.25  # octets 0, 5, 8
    t.rebuild_for(img1, [swg.MapRequest(swg.Kernel(swg.EUCLID_QUAD, 15, 15), model)])
    fi = t.feature_image()
    for b in (2, 41, 70, 9, 63):  # built octets, then stale ones
        for kind in range(5):
            _check_plane(t, fi, b, kind)


def test_decayed_column_sums_in_chunks(ctx):
    """100 bins = 50 pairs: two shared-memory chunks of decayed column sums;
    all four orientations (the h-flipped ones read their partner's carries
    mirrored), a width that is no multiple of the strip or of 8."""
    bins, w, h, d = 100, 301, 420, 0.9
    img = _u16_image(w, h, 8)
    t = ctx.build_decay(img, d, swg.FMT_GRAY16, bins)
    fi = t.feature_image()
    flips = (fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])
    for b in (0, 1, 74, 75, 76, 99):
        for k, f in enumerate(flips):
            got = t.export_f64(k, b, b + 1)[0]
            np.testing.assert_allclose(got, _decayed_plane(np.ascontiguousarray(f), b, d),
                                       rtol=1e-12, atol=1e-13, err_msg=f"bin {b} orientation {k}")


def test_decayed_build_tall_bands(ctx):
    """512 bins (64 octets) leave 5 bands: 540-row bands, whose per-row
    carries leave room for 4 warps per CTA instead of 8, and 8 chunks of
    column sums."""
    bins, w, h, d = 512, 24, 2700, 0.9375
    img = _u16_image(w, h, 9)
    t = ctx.build_decay(img, d, swg.FMT_GRAY16, bins)
    fi = t.feature_image()
    flips = (fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])
    for b in (0, 77, 300, 511):
        for k, f in enumerate(flips):
            got = t.export_f64(k, b, b + 1)[0]
            np.testing.assert_allclose(got, _decayed_plane(np.ascontiguousarray(f), b, d),
                                       rtol=1e-12, atol=1e-13, err_msg=f"bin {b} orientation {k}")


def test_decayed_selective_equals_full(ctx):
    """A model-driven decayed rebuild (its pairs' column sums only, the four
    orientations in one launch) writes the same planes as a full rebuild."""
    bins, w, h, d = 64, 260, 330, 0.9375
    img0, img1 = _u16_image(w, h, 10), _u16_image(w, h, 11)
    ts = ctx.build_decay(img0, d, swg.FMT_GRAY16, bins)
    tf = ctx.build_decay(img0, d, swg.FMT_GRAY16, bins)
    tf.rebuild(img1)
    model = np.zeros(bins)
    model[[5, 6, 33, 60]] = 0.25
    ts.rebuild_for(img1, [swg.MapRequest(swg.Kernel(swg.EXP_L1, 21, 21, d), model)])
    assert 0 < ts.built_bytes() < tf.built_bytes()
    for b in (5, 6, 33, 60, 0, 47):  # built pairs, then stale ones
        for k in range(4):
            assert (ts.export_f64(k, b, b + 1) == tf.export_f64(k, b, b + 1)).all(), (b, k)


def test_random_shapes_against_numpy(ctx):
    """Seeded random table shapes (ragged widths and heights from 1 pixel up,
    1 to 130 bins, every plane set, 8- and 16-bit pixels): a few bins of every
    kind against numpy."""
    rng = np.random.default_rng(2024)
    shapes = [(1, 1, 1), (2, 700, 3), (513, 9, 17), (257, 257, 64)]
    shapes += [(int(rng.integers(1, 700)), int(rng.integers(1, 900)), int(rng.integers(1, 131)))
               for _ in range(8)]
    for n, (w, h, bins) in enumerate(shapes):
        planes = (swg.PLANES_PLAIN, swg.PLANES_AFFINE, swg.PLANES_QUADRATIC)[n % 3]
        if n % 2:
            img, fmt = _u16_image(w, h, 100 + n), swg.FMT_GRAY16
        else:
            img = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
            fmt = swg.FMT_GRAY8
        t = ctx.build(img, fmt, bins, planes)
        fi = t.feature_image()
        for b in sorted({0, bins - 1, int(rng.integers(0, bins))}):
            for kind in range((1, 3, 5)[n % 3]):
                _check_plane(t, fi, b, kind)
        if n % 4 == 0:  # and the decayed planes of the same image
            d = float(rng.choice([0.5, 0.9, 0.9375]))
            td = ctx.build_decay(img, d, fmt, bins)
            fd = td.feature_image()
            flips = (fd, fd[:, ::-1], fd[::-1, :], fd[::-1, ::-1])
            for b in sorted({0, bins - 1}):
                for k, f in enumerate(flips):
                    np.testing.assert_allclose(td.export_f64(k, b, b + 1)[0],
                                               _decayed_plane(np.ascontiguousarray(f), b, d),
                                               rtol=1e-12, atol=1e-13,
                                               err_msg=f"{w}x{h} bins {bins} bin {b} orientation {k}")
