"""GPU parity: the sm_100a path through the C-ABI against the reference's
golden vectors (tests/golden) and the oracle restatement on seeded inputs.

Bar (BASELINE.json north_star): integral tables bit-exact (uint32 words ==
reference int64 mod 2^32; int64 export == reference), every likelihood-map
value bit-exact (the GPU repeats the reference's fp64 operation sequence),
peak locations and tie resolution identical.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu

K = swg.Kernel


def build(ctx, img, bins, planes=swg.PLANES_AFFINE, fmt=swg.FMT_GRAY8):
    return ctx.build(np.ascontiguousarray(img), fmt, bins, planes)


# ------------------------------------------------------------------ tables
@pytest.mark.parametrize("name,bins", [("cross3", 2), ("tables_32x32_s99_b8", 8)])
def test_tables_golden(ctx, name, bins):
    g = golden(name)
    t = build(ctx, g["image"], bins)
    for kind, key in ((0, "plain"), (1, "xramp"), (2, "yramp")):
        assert (t.export_i64(kind) == g[key]).all()
        assert (t.export_u32(kind) == (g[key] & 0xFFFFFFFF).astype(np.uint32)).all()


@pytest.mark.parametrize("w,h,bins", [(1, 1, 4), (3, 2, 2), (17, 13, 8), (64, 64, 16),
                                      (255, 37, 5), (1000, 23, 3), (1025, 40, 4), (4096, 9, 2),
                                      (1031, 61, 2), (33, 700, 3)])
def test_tables_vs_oracle_shapes(ctx, oracle, w, h, bins):
    """Widths around the CPT / thread-count / band boundaries, tall images
    (many look-back bands), degenerate 1x1."""
    img = oracle.random_gray(w, h, w * 1000 + h)
    fi = oracle.quantize_gray8(img, bins)
    p, x, y = oracle.build_tables(fi, bins)
    t = build(ctx, img, bins)
    assert (t.feature_image() == fi).all()
    for kind, ref in ((0, p), (1, x), (2, y)):
        assert (t.export_u32(kind) == (ref & 0xFFFFFFFF).astype(np.uint32)).all(), kind
        assert (t.export_i64(kind) == ref).all(), kind
    tp = build(ctx, img, bins, swg.PLANES_PLAIN)
    assert (tp.export_u32(0) == p.astype(np.uint32)).all()


def test_tables_wrap_exact_large(ctx, oracle):
    """Ramp values beyond 2^32: the uint32 words are the low
    32 bits and the int64 export is exact."""
    w, h, bins = 2048, 2100, 1
    img = np.zeros((h, w), np.uint8)
    fi = oracle.quantize_gray8(img, bins)
    t = build(ctx, img, bins)
    xr = t.export_i64(1)
    yy, xx = np.meshgrid(np.arange(h + 1, dtype=np.int64), np.arange(w + 1, dtype=np.int64),
                         indexing="ij")
    expect = yy * (xx * (xx - 1) // 2)
    assert expect.max() > 2**32
    assert (xr[0] == expect).all()
    assert (t.export_u32(1)[0] == (expect & 0xFFFFFFFF).astype(np.uint32)).all()


@pytest.mark.parametrize("fmt", [swg.FMT_GRAY16, swg.FMT_RGB8, swg.FMT_BINS16])
def test_tables_other_formats(ctx, oracle, fmt):
    rng = np.random.default_rng(fmt)
    h, w = 45, 77
    if fmt == swg.FMT_GRAY16:
        img = rng.integers(0, 65536, (h, w), dtype=np.uint16)
        bins = 64
        fi = oracle.quantize_gray16(img, bins)
    elif fmt == swg.FMT_RGB8:
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        bins = 4
        fi = oracle.quantize_rgb8(img, bins)
    else:
        bins = 11
        img = rng.integers(0, bins, (h, w), dtype=np.uint16)
        fi = img
    nb = bins ** 3 if fmt == swg.FMT_RGB8 else bins
    p, x, y = oracle.build_tables(fi, nb)
    t = ctx.build(img, fmt, bins, swg.PLANES_AFFINE)
    assert t.bins == nb
    assert (t.feature_image() == fi).all()
    assert (t.export_i64(0) == p).all() and (t.export_i64(1) == x).all()
    assert (t.export_i64(2) == y).all()


def test_rebuild_same_buffers(ctx, oracle):
    a, b = oracle.random_gray(300, 200, 1), oracle.random_gray(300, 200, 2)
    t = build(ctx, a, 8)
    t.rebuild(b)
    assert (t.export_i64(1) == oracle.build_tables(oracle.quantize_gray8(b, 8), 8)[1]).all()


def test_upload_i64_round_trip(ctx):
    g = golden("tables_32x32_s99_b8")
    t = ctx.upload_i64(g["plain"], g["xramp"], g["yramp"])
    for kind, key in ((0, "plain"), (1, "xramp"), (2, "yramp")):
        assert (t.export_i64(kind) == g[key]).all()
    k = K(swg.MANHATTAN, 9, 9)
    b = build(ctx, g["image"], 8)
    assert (t.query_windows([10, 20], [10, 15], k) == b.query_windows([10, 20], [10, 15], k)).all()


# ------------------------------------------------------------------ queries
def test_cross3_queries(ctx):
    g = golden("cross3")
    t = build(ctx, g["image"], 2)
    assert t.query_windows(1, 1, K(swg.MANHATTAN, 3))[0].tolist() == [7, 8]
    assert t.query_windows(1, 1, K(swg.UNIFORM, 3))[0].tolist() == [5, 4]
    assert t.query_windows(1, 1, K(swg.UNIFORM, 3), swg.PLAIN)[0].tolist() == [5, 4]
    assert t.query_terms([[(1, 0, 0, 1, 1, 1, 1, 1)]])[0].tolist() == [4, 4]
    assert t.query_terms([[(0, 0, 0, 0, 0, 1, 1, 0)]])[0].tolist() == [0, 0]
    assert (t.cake_windows(1, 1, K(swg.CHEBYSHEV, 3), 2)[0] == g["cake_cheb3_r2"]).all()
    assert (t.cake_windows(1, 1, K(swg.MANHATTAN, 3), 2)[0] == g["cake_man3_r2"]).all()
    assert (t.cake_windows(1, 1, K(swg.MANHATTAN, 3), 2, swg.RING_LEVEL)[0]
            == g["cake_man3_level"]).all()


def test_clipped_queries_golden(ctx):
    g = golden("clipped_15x11_s8_b4")
    t = build(ctx, g["image"], 4)
    cy, cx = np.mgrid[0:11, 0:15]
    got = t.query_windows(cx.ravel(), cy.ravel(), K(swg.MANHATTAN, 7, 5), swg.SWIH, swg.CLIPPED)
    assert (got.reshape(11, 15, 4) == g["counts"]).all()


@pytest.mark.parametrize("seed", [4242, 55])
def test_exactness_gate(ctx, oracle, seed):
    """acceptance_main.cpp:44-85: swih == brute force at every strict centre,
    b in {2, 8, 16}, Manhattan kernels 1x1 .. 31x31."""
    rng = np.random.default_rng(seed)
    for i in range(6):
        w, h = int(rng.integers(33, 65)), int(rng.integers(33, 65))
        img = oracle.random_gray(w, h, int(rng.integers(1 << 30)))
        for bins in (2, 8, 16):
            fi = oracle.quantize_gray8(img, bins)
            t = build(ctx, img, bins)
            for kw, kh in ((1, 1), (3, 3), (5, 9), (7, 7), (11, 11), (31, 31)):
                k = K(swg.MANHATTAN, kw, kh)
                cy, cx = np.mgrid[k.hy:h - k.hy, k.hx:w - k.hx]
                got = t.query_windows(cx.ravel(), cy.ravel(), k)
                ok = O.kernel(O.MANHATTAN, kw, kh)
                want = np.array([oracle.brute_counts(fi, bins, int(a), int(b), ok)
                                 for a, b in zip(cx.ravel(), cy.ravel())])
                assert (got == want).all(), (w, h, bins, kw, kh)


def test_cake_windows_vs_oracle(ctx, oracle):
    img = oracle.random_gray(40, 40, 60)
    fi = oracle.quantize_gray8(img, 8)
    tabs = oracle.build_tables(fi, 8)
    t = build(ctx, img, 8, swg.PLANES_PLAIN)
    for kind, k, sig in ((swg.GAUSS_CHEB, 9, .6), (swg.CHEBYSHEV, 5, .5), (swg.MANHATTAN, 11, .5)):
        h = k // 2
        for rings, rule in ((h + 1, swg.RING_MEAN), (2, swg.RING_LEVEL)):
            for border, pts in ((swg.STRICT, [(h, h), (20, 20), (39 - h, 39 - h)]),
                                (swg.CLIPPED, [(0, 0), (3, 39), (39, 5)])):
                cxs, cys = [p[0] for p in pts], [p[1] for p in pts]
                got = t.cake_windows(cxs, cys, K(kind, k, k, sig), rings, rule, border)
                for i, (cx, cy) in enumerate(pts):
                    want = oracle.cake_histogram(tabs, O.kernel(kind, k, k, sig), rings,
                                                 rule, cx, cy, border)
                    assert (got[i] == want).all(), (kind, rings, rule, border, cx, cy)


def test_query_errors(ctx):
    t = build(ctx, np.zeros((9, 9), np.uint8), 2)
    with pytest.raises(swg.WindowOutOfBoundsError):
        t.query_windows(1, 4, K(swg.MANHATTAN, 5))
    with pytest.raises(swg.WindowOutOfBoundsError):
        t.query_windows(4, 9, K(swg.MANHATTAN, 3), swg.SWIH, swg.CLIPPED)
    with pytest.raises(swg.InvalidKernelError):
        t.query_windows(4, 4, K(swg.MANHATTAN, 4, 3))
    with pytest.raises(swg.UnsupportedKernelError):
        t.query_windows(4, 4, K(swg.GAUSS_CHEB, 3))
    with pytest.raises(swg.ConfigError):
        t.cake_windows(4, 4, K(swg.CHEBYSHEV, 3), 3)
    with pytest.raises(swg.OutOfRangeError):
        t.query_terms([[(1, 0, 0, 9, 3, 0, 0, 1)]])
    with pytest.raises(swg.OutOfRangeError):
        t.export_i64(0, 0, 3)
    with pytest.raises(swg.CapacityError) as e:
        ctx.build(np.zeros((8, 8), np.uint8), swg.FMT_GRAY8, 4, swg.PLANES_AFFINE, budget=64)
    assert e.value.required_bytes > 64


# ------------------------------------------------------------------ maps
@pytest.mark.parametrize("key,method,sim", [("map_bhatt", swg.SWIH, swg.BHATTACHARYYA),
                                            ("map_inter", swg.SWIH, swg.INTERSECTION),
                                            ("map_brute", swg.BRUTE, swg.BHATTACHARYYA)])
def test_map_golden(ctx, key, method, sim):
    g = golden("map_40x33_s2024_b8_man9x7")
    t = build(ctx, g["image"], 8)
    m, pk = t.likelihood_map(K(swg.MANHATTAN, 9, 7), g["model"], method, sim)
    assert (m == g[key]).all()
    if key != "map_brute":
        assert pk == tuple(g["peak_" + key[4:]].tolist())
        assert (pk[2], pk[3]) == (16, 12)


def test_map_plain_golden(ctx):
    g = golden("map_40x33_s2024_b8_man9x7")
    t = build(ctx, g["image"], 8, swg.PLANES_PLAIN)
    templ = np.ascontiguousarray(g["image"][9:16, 12:21])
    from paper_1705_03524_b200 import api
    mdl = api.target_model(ctx, templ, K(swg.MANHATTAN, 9, 7), bins=8, method=swg.PLAIN)
    m, pk = t.likelihood_map(K(swg.MANHATTAN, 9, 7), mdl, swg.PLAIN)
    assert (m == g["map_plain"]).all() and pk == tuple(g["peak_plain"].tolist())


def test_tiled_golden_all_methods(ctx):
    g = golden("tiled_9x6")
    t = build(ctx, g["image"], 2)
    for name, meth in (("swih", swg.SWIH), ("brute", swg.BRUTE), ("cake", swg.CAKE),
                       ("plain", swg.PLAIN)):
        m, pk = t.likelihood_map(K(swg.MANHATTAN, 3), g["model_" + name], meth, rings=2)
        assert (m == g["map_" + name]).all(), name


def test_gaussian_golden(ctx):
    g = golden("gauss_48x40_s60_b8_k9")
    t = build(ctx, g["image"], 8, swg.PLANES_PLAIN)
    kg = K(swg.GAUSS_CHEB, 9, 9, 0.6)
    assert (t.likelihood_map(kg, g["model_cake"], swg.CAKE, rings=5)[0] == g["map_cake"]).all()
    assert (t.likelihood_map(kg, g["model_cake"], swg.CAKE, swg.INTERSECTION, rings=5)[0]
            == g["map_cake_inter"]).all()
    assert (t.likelihood_map(kg, g["model_brute"], swg.BRUTE)[0] == g["map_brute"]).all()
    assert (t.likelihood_map(kg, g["model_brute"], swg.BRUTE, swg.INTERSECTION)[0]
            == g["map_brute_inter"]).all()


def test_chebyshev_golden(ctx):
    g = golden("cheb_40x36_s5_b8_k7x5")
    t = build(ctx, g["image"], 8, swg.PLANES_PLAIN)
    kc = K(swg.CHEBYSHEV, 7, 5)
    assert (t.likelihood_map(kc, g["model"], swg.BRUTE)[0] == g["map_brute"]).all()
    assert (t.likelihood_map(kc, g["model"], swg.CAKE, rings=2, ring_rule=swg.RING_LEVEL)[0]
            == g["map_cake_level"]).all()


@pytest.mark.parametrize("name,k", [("scene_96x80_man21_b16", 21), ("config1_s3", 33)])
def test_scene_golden(ctx, name, k):
    g = golden(name)
    t = build(ctx, g["image"], 16)
    m, pk = t.likelihood_map(K(swg.MANHATTAN, k), g["model"])
    assert (m == g["map"]).all()
    assert pk == tuple(g["peak"].tolist())


def test_peak_tie_rule(ctx):
    """A constant image: every window scores the same; the first cell wins
    (matching.cpp:211-223).  Ties across CTA boundaries and rows."""
    img = np.full((40, 300), 77, np.uint8)
    t = build(ctx, img, 4)
    mdl = np.array([0.25, 0.25, 0.25, 0.25])
    for k in (K(swg.MANHATTAN, 5), K(swg.UNIFORM, 3, 7)):
        m, pk = t.likelihood_map(k, mdl)
        assert (m == m[0, 0]).all()
        assert pk[:2] == (0, 0)
    # equal maxima placed late in row-major order: first one must win
    img = np.zeros((50, 400), np.uint8)
    img[30:33, 350:353] = 255
    img[40:43, 10:13] = 255
    img[30:33, 200:203] = 255
    t = build(ctx, img, 2)
    mdl = np.array([0.0, 1.0])
    m, pk = t.likelihood_map(K(swg.UNIFORM, 3), mdl)
    assert pk[:2] == (200, 30) and pk[4] == 1.0


@pytest.mark.parametrize("seed", [1, 2])
def test_maps_vs_oracle_random(ctx, oracle, seed):
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(60, 200)), int(rng.integers(40, 120))
    img = oracle.random_gray(w, h, seed)
    for bins in (2, 16, 32):
        fi = oracle.quantize_gray8(img, bins)
        t = build(ctx, img, bins)
        for kind, kw, kh, sig in ((swg.MANHATTAN, 1, 1, .5), (swg.MANHATTAN, 13, 7, .5),
                                  (swg.UNIFORM, 9, 15, .5), (swg.MANHATTAN, 31, 31, .5),
                                  (swg.GAUSS_CHEB, 11, 11, .5), (swg.CHEBYSHEV, 7, 9, .5)):
            ok = O.kernel(kind, kw, kh, sig)
            methods = [swg.SWIH, swg.PLAIN] if kind in (swg.MANHATTAN, swg.UNIFORM) else []
            methods += [swg.CAKE, swg.BRUTE]
            for method in methods:
                rings = min(kw, kh) // 2 + 1 if method == swg.CAKE else 1
                mdl = oracle.target_model(fi[:kh, :kw].copy(), bins, ok, method, rings)
                for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
                    want = oracle.likelihood_map(fi, bins, mdl, ok, method, sim, rings=rings)
                    got, pk = t.likelihood_map(K(kind, kw, kh, sig), mdl, method, sim, rings)
                    assert (got == want).all(), (bins, kind, kw, kh, method, sim)
                    assert pk == oracle.peak(want, kw // 2, kh // 2)


def test_map_row_ranges_and_device_outputs(ctx, oracle):
    torch = pytest.importorskip("torch")
    img = oracle.random_gray(128, 96, 9)
    fi = oracle.quantize_gray8(img, 16)
    t = build(ctx, img, 16)
    k = K(swg.MANHATTAN, 17, 17)
    ok = O.kernel(O.MANHATTAN, 17, 17)
    mdl = oracle.target_model(fi[:17, :17].copy(), 16, ok)
    full = oracle.likelihood_map(fi, 16, mdl, ok)
    got, pk = t.likelihood_map(k, mdl, rows=(10, 33))
    assert (got == full[10:33]).all()
    mx, my, _, _, sc = oracle.peak(full[10:33], 8, 8)
    assert pk == (mx, my + 10, mx + 8, my + 18, sc)
    dev = torch.empty(full.shape, dtype=torch.float64, device="cuda")
    peaks = torch.zeros(1, 3, dtype=torch.float64, device="cuda")  # 24 B >= sizeof(swg_peak)
    t.likelihood_maps([swg.MapRequest(k, mdl)], scores="none", scores_dev=[dev], peaks_dev=peaks)
    ctx.synchronize()
    assert (dev.cpu().numpy() == full).all()


def test_map_errors(ctx):
    t = build(ctx, np.full((5, 5), 10, np.uint8), 4)
    mdl = np.full(4, .25)
    with pytest.raises(swg.SizeError):
        t.likelihood_map(K(swg.MANHATTAN, 7), mdl)
    with pytest.raises(swg.UnsupportedKernelError):
        t.likelihood_map(K(swg.GAUSS_CHEB, 3), mdl, swg.SWIH)
    with pytest.raises(swg.InvalidKernelError):
        t.likelihood_map(K(swg.MANHATTAN, 2, 3), mdl)
    with pytest.raises(swg.ModelError):
        t.likelihood_map(K(swg.MANHATTAN, 3), np.full(3, 1 / 3))
    with pytest.raises(swg.ConfigError):
        t.likelihood_map(K(swg.MANHATTAN, 3), mdl, swg.CAKE, rings=3)


# ------------------------------------------------------------------ full-size properties
def test_config2_full_size_properties(ctx):
    """BASELINE config 2 geometry (1024^2, b=32): plain-table checksums
    (T(W,H) per bin = bin population; all bins sum to W*H) and the Gaussian
    maps' peaks on the planted targets."""
    from paper_1705_03524_b200 import api, synth
    sc = synth.config2(1)
    t = ctx.build(sc.image, swg.FMT_GRAY8, 32, swg.PLANES_PLAIN)
    corner = t.export_u32(0)[:, -1, -1].astype(np.int64)
    fi = (sc.image.astype(np.int64) * 32) >> 8
    assert (corner == np.bincount(fi.ravel(), minlength=32)).all()
    assert corner.sum() == 1024 * 1024
    for (cx, cy, tw, th), s in zip(sc.targets[:3], (32, 64, 96)):
        kw = synth.odd_window(s)
        k = K(swg.GAUSS_CHEB, kw, kw, 0.5)
        mdl = api.target_model(ctx, synth.crop(sc.image, cx, cy, kw, kw), k, bins=32,
                               method=swg.CAKE, rings=kw // 2 + 1)
        m, pk = t.likelihood_map(k, mdl, swg.CAKE, rings=kw // 2 + 1)
        assert m.min() >= 0.0 and m.max() <= 1.0
        assert abs(pk[2] - cx) <= 1 and abs(pk[3] - cy) <= 1 and pk[4] > 0.999


def test_width_limit_is_a_size_error(ctx):
    with pytest.raises(swg.SizeError):
        ctx.build(np.zeros((4, 4097), np.uint8), swg.FMT_GRAY8, 2, swg.PLANES_PLAIN)


def test_row_band_tables_and_maps_on_gpu(ctx, oracle):
    """Row-band split on the device: per-band GPU tables +
    boundary prefix rows rebuild the global tables exactly; per-band GPU maps
    are the full map's rows; the band peaks reduce to the full-map peak."""
    from paper_1705_03524_b200 import dist as D
    img = oracle.random_gray(301, 203, 77)
    bins, world = 16, 4
    full = build(ctx, img, bins)
    glob_ref = [full.export_i64(k) for k in range(3)]
    locs, rows = [], []
    for y0, y1 in D.table_bands(203, world):
        t = build(ctx, np.ascontiguousarray(img[y0:y1]), bins)
        loc = tuple(t.export_i64(k) for k in range(3))
        locs.append((y0, y1, loc))
        rows.append(D.last_rows(loc, y0))
    for r, (y0, y1, loc) in enumerate(locs):
        g = D.globalize_band_tables(loc, y0, D.band_carry(rows, r))
        for k in range(3):
            assert (g[k] == glob_ref[k][:, y0:y1 + 1]).all()
    k = K(swg.MANHATTAN, 25, 17)
    fi = oracle.quantize_gray8(img, bins)
    mdl = oracle.target_model(fi[40:57, 100:125].copy(), bins, O.kernel(O.MANHATTAN, 25, 17))
    fmap, fpk = full.likelihood_map(k, mdl)
    cands = []
    for bd in D.row_bands(203, 17, world):
        (v0, v1), (p0, p1) = bd.map_rows, bd.pixel_rows
        tb = build(ctx, np.ascontiguousarray(img[p0:p1]), bins)
        m, pk = tb.likelihood_map(k, mdl)
        assert (m == fmap[v0:v1]).all()
        cands.append((pk[4], (pk[1] + v0) * fmap.shape[1] + pk[0]))
    s, i = D.reduce_peaks(cands)
    assert (i % fmap.shape[1], i // fmap.shape[1], s) == (fpk[0], fpk[1], fpk[4])


def test_narrow_and_wide_plain_paths(ctx, oracle):
    """Plain-only tables sweep with 16-bit planes while every box has area
    < 2^16 and switch to 32-bit planes beyond (257x257 = 66049 px)."""
    img = oracle.random_gray(300, 280, 31)
    bins = 4
    fi = oracle.quantize_gray8(img, bins)
    t = build(ctx, img, bins, swg.PLANES_PLAIN)
    for kw, kh in ((255, 255), (257, 257), (255, 259)):
        for kind, method, rings in ((swg.UNIFORM, swg.PLAIN, 1), (swg.GAUSS_CHEB, swg.CAKE, 3)):
            ok = O.kernel(kind, kw, kh, 0.5)
            mdl = oracle.target_model(fi[:kh, :kw].copy(), bins, ok, method, rings)
            want = oracle.likelihood_map(fi, bins, mdl, ok, method, O.BHATTACHARYYA, rings=rings)
            got, pk = t.likelihood_map(K(kind, kw, kh, 0.5), mdl, method, rings=rings)
            assert (got == want).all(), (kw, kh, kind)
            assert pk == oracle.peak(want, kw // 2, kh // 2)


# ------------------------------------------------------------------ declared extensions
def test_quadratic_planes_exact(ctx, oracle):
    """x^2 / y^2 planes of the quadratic table set, exact int64."""
    img = oracle.random_gray(77, 61, 3)
    bins = 5
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC)
    p, x, y = oracle.build_tables(fi, bins)
    assert (t.export_i64(0) == p).all() and (t.export_i64(1) == x).all()
    assert (t.export_i64(2) == y).all()
    yy, xx = np.mgrid[0:61, 0:77].astype(np.int64)
    for kind, wgt in ((3, xx * xx), (4, yy * yy)):
        got = t.export_i64(kind)
        for b in range(bins):
            want = np.zeros((62, 78), np.int64)
            want[1:, 1:] = np.cumsum(np.cumsum((fi == b) * wgt, 0), 1)
            assert (got[b] == want).all(), (kind, b)


@pytest.mark.parametrize("bins", [8, 16])
def test_euclid_quadratic_maps_exact(ctx, oracle, bins):
    """Declared Euclidean kernel on quadratic planes (O(1)) == the oracle's
    brute-force map bit for bit; the GPU brute force agrees too."""
    img = oracle.random_gray(150, 120, bins)
    fi = oracle.quantize_gray8(img, bins)
    tq = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC)
    tp = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    for kw, kh in ((1, 1), (5, 5), (9, 7), (31, 31), (45, 59)):
        ok = O.kernel(O.EUCLID_QUAD, kw, kh)
        mdl = oracle.target_model(fi[10:10 + kh, 20:20 + kw].copy(), bins, ok, O.BRUTE)
        for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
            want = oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE, sim)
            got, pk = tq.likelihood_map(K(swg.EUCLID_QUAD, kw, kh), mdl, swg.SWIH, sim)
            assert (got == want).all(), (kw, kh, sim)
            assert pk == oracle.peak(want, kw // 2, kh // 2)
        got_b, _ = tp.likelihood_map(K(swg.EUCLID_QUAD, kw, kh), mdl, swg.BRUTE)
        assert (got_b == oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE)).all()
    with pytest.raises(swg.ConfigError):
        tp.likelihood_map(K(swg.EUCLID_QUAD, 5, 5), np.full(bins, 1 / bins), swg.SWIH)


def test_exponential_brute_and_cake(ctx, oracle):
    """Declared exponential kernel: GPU brute force == oracle brute force
    (same fp64 pixel order); exact ring telescope is not applicable (not
    ring-constant), the cake path is checked as an approximation route."""
    img = oracle.random_gray(96, 80, 5)
    bins = 8
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    for kw, lam in ((9, 0.75), (21, 0.9375)):
        ok = O.kernel(O.EXP_L1, kw, kw, lam)
        mdl = oracle.target_model(fi[:kw, :kw].copy(), bins, ok, O.BRUTE)
        want = oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE)
        got, pk = t.likelihood_map(K(swg.EXP_L1, kw, kw, lam), mdl, swg.BRUTE)
        assert (got == want).all()
        assert pk == oracle.peak(want, kw // 2, kw // 2)
        r = kw // 2 + 1
        mc = oracle.target_model(fi[:kw, :kw].copy(), bins, ok, O.CAKE, r)
        want_c = oracle.likelihood_map(fi, bins, mc, ok, O.CAKE, rings=r)
        got_c, _ = t.likelihood_map(K(swg.EXP_L1, kw, kw, lam), mc, swg.CAKE, rings=r)
        assert (got_c == want_c).all()


def _decayed_se(fi, bins, d):
    """numpy restatement of the decayed SE table: E(X,Y) = sum over x<X, y<Y
    of [fi==b] d^(X-1-x) d^(Y-1-y), zero row/column 0."""
    h, w = fi.shape
    out = np.zeros((bins, h + 1, w + 1))
    for b in range(bins):
        one = (fi == b).astype(np.float64)
        r = np.zeros((h, w + 1))
        for x in range(w):
            r[:, x + 1] = d * r[:, x] + one[:, x]
        for y in range(h):
            out[b, y + 1] = d * out[b, y] + r[y]
    return out


@pytest.mark.parametrize("w,h,bins,d", [(70, 53, 12, 0.9375), (33, 61, 5, 0.5), (1, 1, 3, 0.75)])
def test_decay_tables_vs_numpy(ctx, oracle, w, h, bins, d):
    img = oracle.random_gray(w, h, 11)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
    assert t.planes == swg.PLANES_DECAY
    flips = (fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])
    for k, f in enumerate(flips):
        want = _decayed_se(np.ascontiguousarray(f), bins, d)
        got = t.export_f64(k)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    with pytest.raises(swg.ConfigError):
        t.export_u32(0)


def test_exponential_swih_maps(ctx, oracle):
    """O(1) exponential maps on decay tables: map values within 1e-4 of the
    fp64 brute force; the peak (index AND score) is exact through the
    candidate re-score."""
    img = oracle.random_gray(120, 90, 21)
    bins = 8
    fi = oracle.quantize_gray8(img, bins)
    for d in (0.75, 0.9375):
        t = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
        for kw, kh in ((1, 1), (9, 9), (21, 15), (41, 41)):
            ok = O.kernel(O.EXP_L1, kw, kh, d)
            mdl = oracle.target_model(fi[30:30 + kh, 40:40 + kw].copy(), bins, ok, O.BRUTE)
            for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
                want = oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE, sim)
                got, pk = t.likelihood_map(K(swg.EXP_L1, kw, kh, d), mdl, swg.SWIH, sim)
                np.testing.assert_allclose(got, want, rtol=0, atol=1e-4)
                assert pk == oracle.peak(want, kw // 2, kh // 2), (d, kw, kh, sim)
        with pytest.raises(swg.ConfigError):  # sigma must match the tables' decay
            t.likelihood_map(K(swg.EXP_L1, 9, 9, 0.5), np.full(bins, 1 / bins), swg.SWIH)
        with pytest.raises(swg.ConfigError):  # decay tables serve EXP_L1 / brute only
            t.likelihood_map(K(swg.UNIFORM, 9, 9), np.full(bins, 1 / bins), swg.SWIH)
        # brute force from the decay tables' feature image
        ok = O.kernel(O.EXP_L1, 9, 9, d)
        mdl = oracle.target_model(fi[:9, :9].copy(), bins, ok, O.BRUTE)
        got_b, _ = t.likelihood_map(K(swg.EXP_L1, 9, 9, d), mdl, swg.BRUTE)
        assert (got_b == oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE)).all()


def test_exponential_swih_flat_image(ctx, oracle):
    """Every window ties: more candidates than the re-score capacity, the
    full-map fallback must still return the reference's first maximum."""
    img = np.full((96, 128), 77, np.uint8)
    bins = 4
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build_decay(img, 0.9375, swg.FMT_GRAY8, bins)
    ok = O.kernel(O.EXP_L1, 9, 9, 0.9375)
    mdl = oracle.target_model(fi[:9, :9].copy(), bins, ok, O.BRUTE)
    want = oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE)
    got, pk = t.likelihood_map(K(swg.EXP_L1, 9, 9, 0.9375), mdl, swg.SWIH)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-4)
    assert pk == oracle.peak(want, 4, 4)


def test_likelihood_batch_matches_per_frame(ctx, oracle):
    """swg_likelihood_batch over search-region crops (pointer + full-frame
    pitch) == one build + map per frame == the oracle's brute force."""
    from paper_1705_03524_b200 import api, synth
    seq = synth.config3(5, n_frames=4, h=200, w=320, search=96)
    F, H, W = seq.frames.shape[:3]
    S = seq.search
    scales = [K(swg.EUCLID_QUAD, 21, 27), K(swg.EUCLID_QUAD, 25, 31)]
    cx, cy = seq.track[0]
    models = [api.target_model(ctx, synth.crop(seq.frames[0], cx, cy, k.kw, k.kh), k,
                               fmt=swg.FMT_RGB8, bins=4) for k in scales]
    reqs = [swg.MapRequest(k, m) for k, m in zip(scales, models)]
    crops = []
    for f in range(F):
        x0, y0 = synth.search_origin(seq, f)
        crops.append(seq.frames[f, y0:y0 + S, x0:x0 + S])
    t = ctx.build(np.ascontiguousarray(crops[0]), swg.FMT_RGB8, 4, swg.PLANES_QUADRATIC)
    got = t.likelihood_batch(crops, reqs, pitch=W * 3)
    for f in range(F):
        fi = oracle.quantize_rgb8(np.ascontiguousarray(crops[f]), 4)
        t1 = ctx.build(np.ascontiguousarray(crops[f]), swg.FMT_RGB8, 4, swg.PLANES_QUADRATIC)
        _, pk1 = t1.likelihood_maps(reqs, scores="none")
        for i, k in enumerate(scales):
            ok = O.kernel(O.EUCLID_QUAD, k.kw, k.kh)
            want = oracle.likelihood_map(fi, 64, models[i], ok, O.BRUTE)
            assert got[f][i] == pk1[i] == oracle.peak(want, k.hx, k.hy), (f, i)
    # device crops with the same pitch
    import torch
    fd = torch.from_numpy(seq.frames).cuda()
    dev = [fd[f, y0:y0 + S, x0:x0 + S] for f, (x0, y0) in
           ((f, synth.search_origin(seq, f)) for f in range(F))]
    assert t.likelihood_batch(dev, reqs, pitch=W * 3) == got


def test_decay_row_bands_match_full_frame(ctx, oracle):
    """Row bands (config 4 on N GPUs): decay tables built on a band's pixel
    rows give the full frame's map rows (the band's carry cancels in the
    rectangle formula) within 1e-9, and the band peaks combine (max score,
    then smallest global index) to the full frame's exact peak."""
    import bench
    img = oracle.random_gray(97, 150, 8)
    bins, d = 6, 0.9375
    fi = oracle.quantize_gray8(img, bins)
    scales = [(K(swg.EXP_L1, 9, 9, d), swg.SWIH, 1, None), (K(swg.EXP_L1, 15, 13, d), swg.SWIH, 1, None)]
    full = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
    BH, plan = bench.band_plan(150, scales, 3)
    for si, (k, _, _, _) in enumerate(scales):
        ok = O.kernel(O.EXP_L1, k.kw, k.kh, d)
        mdl = oracle.target_model(fi[40:40 + k.kh, 30:30 + k.kw].copy(), bins, ok, O.BRUTE)
        want = oracle.likelihood_map(fi, bins, mdl, ok, O.BRUTE)
        fmap, fpk = full.likelihood_map(k, mdl, swg.SWIH)
        mw = fmap.shape[1]
        best = None
        for p0, rows in plan:
            v0, v1 = rows[si]
            if v1 <= v0:
                continue
            tb = ctx.build_decay(np.ascontiguousarray(img[p0:p0 + BH]), d, swg.FMT_GRAY8, bins)
            bmap, bpk = tb.likelihood_map(k, mdl, swg.SWIH, rows=(v0 - p0, v1 - p0))
            np.testing.assert_allclose(bmap, fmap[v0:v1], rtol=0, atol=1e-9)
            gidx = (bpk[1] + p0) * mw + bpk[0]
            if best is None or bpk[4] > best[0] or (bpk[4] == best[0] and gidx < best[1]):
                best = (bpk[4], gidx)
        pk = oracle.peak(want, k.hx, k.hy)
        assert fpk == pk
        assert best == (pk[4], pk[1] * mw + pk[0])


# ---------------------------------------------------------------- full-size spot checks
def _region_check(oracle, fi, bins, model, k, method, rings, got_map, regions, tol):
    """Map values of window regions of a full-size GPU map against the
    oracle on the pixel crop holding exactly those windows (window
    histograms do not depend on the crop: test_row_band_crop_identity)."""
    ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
    for (u0, v0, nu, nv) in regions:
        crop = np.ascontiguousarray(fi[v0:v0 + nv + k.kh - 1, u0:u0 + nu + k.kw - 1])
        want = oracle.likelihood_map(crop, bins, model, ok, method, rings=rings)
        sub = got_map[v0:v0 + nv, u0:u0 + nu]
        if tol == 0:
            assert (sub == want).all(), (k.kind, k.kw, u0, v0)
        else:
            np.testing.assert_allclose(sub, want, rtol=0, atol=tol)


def _peak_check(oracle, fi, bins, model, k, method, rings, pk, got_map):
    """The reported peak is the map's first maximum and its score is the
    oracle's score of that window."""
    assert pk[4] == got_map.max()
    assert (pk[0], pk[1]) == tuple(np.unravel_index(np.argmax(got_map), got_map.shape)[::-1])
    u, v = pk[0], pk[1]
    crop = np.ascontiguousarray(fi[v:v + k.kh, u:u + k.kw])
    ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
    assert oracle.likelihood_map(crop, bins, model, ok, method, rings=rings)[0, 0] == pk[4]


def test_config5_full_size_spot_checks(ctx, oracle):
    """BASELINE config 5 at full size (2048x2048 u16, 64 bins): all four
    kernels at the smallest, a middle and the largest scale."""
    from paper_1705_03524_b200 import api, synth
    sc = synth.config5(1)
    img, bins = sc.image, 64
    fi = oracle.quantize_gray16(img, bins)
    d = 15.0 / 16.0
    tabs = {swg.PLANES_AFFINE: ctx.build(img, swg.FMT_GRAY16, bins, swg.PLANES_AFFINE),
            swg.PLANES_PLAIN: ctx.build(img, swg.FMT_GRAY16, bins, swg.PLANES_PLAIN),
            swg.PLANES_QUADRATIC: ctx.build(img, swg.FMT_GRAY16, bins, swg.PLANES_QUADRATIC),
            swg.PLANES_DECAY: ctx.build_decay(img, d, swg.FMT_GRAY16, bins)}
    rng = np.random.default_rng(5)
    for kw in (17, 117, 257):
        cases = [(K(swg.MANHATTAN, kw, kw), swg.SWIH, 1, swg.PLANES_AFFINE, O.SWIH, 0),
                 (K(swg.GAUSS_CHEB, kw, kw, 0.5), swg.CAKE, kw // 2 + 1, swg.PLANES_PLAIN,
                  O.CAKE, 0),
                 (K(swg.EUCLID_QUAD, kw, kw), swg.SWIH, 1, swg.PLANES_QUADRATIC, O.BRUTE, 0),
                 (K(swg.EXP_L1, kw, kw, d), swg.SWIH, 1, swg.PLANES_DECAY, O.BRUTE, 1e-4)]
        mw = mh = 2048 - kw + 1
        regions = [(int(rng.integers(0, mw - 8)), int(rng.integers(0, mh - 4)), 8, 4),
                   (0, 0, 6, 3), (mw - 6, mh - 3, 6, 3)]
        for k, method, rings, planes, omethod, tol in cases:
            templ = synth.crop(img, 700, 1300, kw, kw)
            model = api.target_model(ctx, templ, k, fmt=swg.FMT_GRAY16, bins=bins,
                                     method=method, rings=rings)
            got, pk = tabs[planes].likelihood_map(k, model, method, rings=rings)
            _region_check(oracle, fi, bins, model, k, omethod, rings, got, regions, tol)
            _peak_check(oracle, fi, bins, model, k, omethod, rings, pk, got)


def test_config4_band_full_size_spot_checks(ctx, oracle):
    """BASELINE config 4 at full width (3840 RGB, 512 bins, exponential):
    the first row band's decay tables, every scale."""
    import bench
    from paper_1705_03524_b200 import api, synth
    sc = synth.config4(1)
    img = sc.image
    fi = oracle.quantize_rgb8(img, 8)
    d = 15.0 / 16.0
    wl = bench.workload("c4")
    scales = wl["groups"][0]["scales"]
    BH, plan = bench.band_plan(img.shape[0], scales, 4)
    p0, rows = plan[0]
    band = np.ascontiguousarray(img[p0:p0 + BH])
    t = ctx.build_decay(band, d, swg.FMT_RGB8, 8)
    bfi = fi[p0:p0 + BH]
    rng = np.random.default_rng(4)
    for si, (k, method, rings, _) in enumerate(scales):
        v0, v1 = rows[si]
        cx, cy = sc.targets[si][:2]
        model = api.target_model(ctx, synth.crop(img, cx, cy, k.kw, k.kh), k, fmt=swg.FMT_RGB8,
                                 bins=8)
        got, pk = t.likelihood_map(k, model, swg.SWIH, rows=(v0 - p0, v1 - p0))
        mw = got.shape[1]
        regions = [(int(rng.integers(0, mw - 4)), int(rng.integers(0, v1 - v0 - 2)), 4, 2),
                   (mw - 3, v1 - v0 - 2, 3, 2)]
        _region_check(oracle, bfi, 512, model, k, O.BRUTE, 1, got, regions, 1e-4)
        _peak_check(oracle, bfi, 512, model, k, O.BRUTE, 1, pk, got)


def test_config3_full_size_frames(ctx, oracle):
    """BASELINE config 3 frames at full size: search-region maps of all
    three Euclidean scales == the oracle's brute force, bit for bit."""
    from paper_1705_03524_b200 import api, synth
    seq = synth.config3(1, n_frames=3)
    W = seq.frames.shape[2]
    S = seq.search
    scales = [K(swg.EUCLID_QUAD, kw, kh) for kw, kh in ((45, 59), (49, 65), (53, 71))]
    cx, cy = seq.track[0]
    models = [api.target_model(ctx, synth.crop(seq.frames[0], cx, cy, k.kw, k.kh), k,
                               fmt=swg.FMT_RGB8, bins=4) for k in scales]
    for f in (1, 2):
        x0, y0 = synth.search_origin(seq, f)
        crop = np.ascontiguousarray(seq.frames[f, y0:y0 + S, x0:x0 + S])
        t = ctx.build(crop, swg.FMT_RGB8, 4, swg.PLANES_QUADRATIC)
        fi = oracle.quantize_rgb8(crop, 4)
        maps, pks = t.likelihood_maps([swg.MapRequest(k, m) for k, m in zip(scales, models)])
        for k, m, got, pk in zip(scales, models, maps, pks):
            want = oracle.likelihood_map(fi, 64, m, O.kernel(O.EUCLID_QUAD, k.kw, k.kh), O.BRUTE)
            assert (got == want).all()
            assert pk == oracle.peak(want, k.hx, k.hy)
            # the planted target is found within 2 px at the middle scale
        gx, gy = seq.track[f]
        assert abs(pks[1][2] + x0 - gx) <= 2 and abs(pks[1][3] + y0 - gy) <= 2


# ---------------------------------------------------------------- bin-range chains
def _chain_maps(ctx, img, bins, planes, ranges, req_kw, decay=0.0, rows=None):
    """Run a bin-range chain on one GPU (the ranks in sequence): returns the
    last range's (map, peak)."""
    import torch
    pin = None
    for g, (b0, b1) in enumerate(ranges):
        t = ctx.build_bins(img, b0, b1, swg.FMT_GRAY8, bins, planes, decay=decay)
        assert (t.bin_begin, t.bin_end, t.total_bins) == (b0, b1, bins)
        shape = t.map_shape(req_kw["kernel"], rows)
        last = g == len(ranges) - 1
        # fully written by the sweep; torch.empty issues no work on torch's
        # stream that could race the library's own stream
        pout = None if last else torch.empty(shape + (2,), dtype=torch.float64, device="cuda")
        r = swg.MapRequest(rows=rows, partial_in=pin, partial_out=pout, **req_kw)
        maps, pks = t.likelihood_maps([r], scores="host" if last else "none")
        if last:
            return maps[0], pks[0]
        assert pks[0] is None
        pin = pout


@pytest.mark.parametrize("ranges", [[(0, 8), (8, 16), (16, 20)], [(0, 3), (3, 11), (11, 20)],
                                    [(0, 20)]])
def test_bin_range_chain_bit_exact(ctx, oracle, ranges):
    """Config 4's bin-range sharding: tables holding only bins [b0, b1)
    continue each window's running sums; the chain's last map and peak are
    bit-identical to the single-table ones, for every table sweep."""
    img = oracle.random_gray(96, 70, 13)
    bins = 20
    fi = oracle.quantize_gray8(img, bins)
    d = 0.9375
    cases = [(K(swg.MANHATTAN, 9, 7), swg.SWIH, 1, swg.PLANES_AFFINE, swg.BHATTACHARYYA),
             (K(swg.MANHATTAN, 9, 7), swg.SWIH, 1, swg.PLANES_AFFINE, swg.INTERSECTION),
             (K(swg.GAUSS_CHEB, 11, 11, 0.5), swg.CAKE, 6, swg.PLANES_PLAIN, swg.BHATTACHARYYA),
             (K(swg.UNIFORM, 13, 9), swg.SWIH, 1, swg.PLANES_PLAIN, swg.BHATTACHARYYA),
             (K(swg.EUCLID_QUAD, 15, 11), swg.SWIH, 1, swg.PLANES_QUADRATIC, swg.INTERSECTION),
             (K(swg.EUCLID_QUAD, 15, 11), swg.SWIH, 1, swg.PLANES_QUADRATIC, swg.BHATTACHARYYA),
             (K(swg.EXP_L1, 13, 13, d), swg.SWIH, 1, swg.PLANES_DECAY, swg.BHATTACHARYYA)]
    for k, method, rings, planes, sim in cases:
        ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
        om = O.CAKE if method == swg.CAKE else (O.BRUTE if k.kind in (swg.EUCLID_QUAD, swg.EXP_L1)
                                                else O.SWIH)
        model = oracle.target_model(fi[20:20 + k.kh, 30:30 + k.kw].copy(), bins, ok, om, rings)
        if planes == swg.PLANES_DECAY:
            full = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
        else:
            full = ctx.build(img, swg.FMT_GRAY8, bins, planes)
        req = dict(kernel=k, model=model, method=method, sim=sim, rings=rings)
        want, wpk = full.likelihood_map(k, model, method, sim, rings=rings)
        got, gpk = _chain_maps(ctx, img, bins, planes, ranges, req, decay=d)
        assert (got == want).all(), (k.kind, sim, ranges)
        assert gpk == wpk
        # and the chain over a row range (vs the single table over the same
        # rows: the exponential peak re-score depends on the rows searched)
        want_r, wpk_r = full.likelihood_map(k, model, method, sim, rings=rings, rows=(5, 17))
        got_r, gpk_r = _chain_maps(ctx, img, bins, planes, ranges, req, decay=d, rows=(5, 17))
        assert (got_r == want_r).all() and gpk_r == wpk_r, ("rows", k.kind, sim, ranges)
        if k.kind != swg.EXP_L1:
            assert (want_r == want[5:17]).all()


def test_bin_range_errors(ctx, oracle):
    import torch
    img = oracle.random_gray(40, 30, 2)
    bins = 16
    t = ctx.build_bins(img, 0, 8, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    m = np.full(bins, 1.0 / bins)
    k = K(swg.GAUSS_CHEB, 9, 9, 0.5)
    with pytest.raises(swg.ConfigError):  # a range without a chain
        t.likelihood_map(k, m, swg.CAKE, rings=5)
    buf = torch.zeros(t.map_shape(k) + (2,), dtype=torch.float64, device="cuda")
    with pytest.raises(swg.ConfigError):  # intersection needs the full mass first
        t.likelihood_maps([swg.MapRequest(k, m, swg.CAKE, swg.INTERSECTION, 5, partial_out=buf)],
                          scores="none")
    with pytest.raises(swg.ConfigError):  # brute force does not chain
        t.likelihood_maps([swg.MapRequest(k, m, swg.BRUTE, partial_out=buf)], scores="none")
    with pytest.raises(swg.OutOfRangeError):
        ctx.build_bins(img, 8, 20, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    with pytest.raises(swg.OutOfRangeError):
        ctx.build_bins(img, 5, 5, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)


def test_decay_tables_max_width(ctx, oracle):
    """Decay build at the width limit (8 columns per thread, staged stores)."""
    img = oracle.random_gray(4096, 5, 3)
    bins = 3
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build_decay(img, 0.5, swg.FMT_GRAY8, bins)
    for k, f in enumerate((fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])):
        np.testing.assert_allclose(t.export_f64(k), _decayed_se(np.ascontiguousarray(f), bins, 0.5),
                                   rtol=1e-12, atol=1e-12)


def test_decay_tables_strips_and_blocks(ctx, oracle):
    """Decay build across column strips (600 wide: three 256-column strips
    with the strip-to-strip carry) and row blocks (64 bins: bands of 17 rows,
    one full 16-row block plus a partial one), slow decay so every carry
    matters."""
    img = oracle.random_gray(600, 600, 5)
    bins, d = 64, 0.9375
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
    for k, f in ((0, fi), (3, fi[::-1, ::-1])):
        np.testing.assert_allclose(t.export_f64(k), _decayed_se(np.ascontiguousarray(f), bins, d),
                                   rtol=1e-12, atol=1e-10)


def test_pinned_host_maps_zero_copy(ctx, oracle):
    """Host maps in page-locked memory are written by the sweeps directly
    (zero-copy): identical to the copied maps for every engine, one request
    or several fanned out (the exponential sweep keeps its copy path)."""
    img = oracle.random_gray(150, 120, 31)
    bins, d = 16, 0.9375
    fi = oracle.quantize_gray8(img, bins)
    tabs = {swg.PLANES_PLAIN: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN),
            swg.PLANES_AFFINE: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_AFFINE),
            swg.PLANES_QUADRATIC: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC),
            swg.PLANES_DECAY: ctx.build_decay(img, d, swg.FMT_GRAY8, bins)}
    cases = [(swg.PLANES_PLAIN, K(swg.GAUSS_CHEB, 21, 21, 0.5), swg.CAKE, 11),
             (swg.PLANES_PLAIN, K(swg.UNIFORM, 15, 9), swg.PLAIN, 1),
             (swg.PLANES_AFFINE, K(swg.MANHATTAN, 17, 13), swg.SWIH, 1),
             (swg.PLANES_QUADRATIC, K(swg.EUCLID_QUAD, 19, 15), swg.SWIH, 1),
             (swg.PLANES_DECAY, K(swg.EXP_L1, 13, 13, d), swg.SWIH, 1)]
    by_tab = {}
    for planes, k, method, rings in cases:
        mdl = oracle.target_model(fi[20:20 + k.kh, 30:30 + k.kw].copy(), bins,
                                  O.kernel(k.kind, k.kw, k.kh, k.sigma),
                                  O.BRUTE if k.kind == swg.EXP_L1 else method, rings)
        by_tab.setdefault(planes, []).append(swg.MapRequest(k, mdl, method, swg.BHATTACHARYYA,
                                                            rings))
    for planes, reqs in by_tab.items():
        for group in ([r] for r in reqs) if len(reqs) == 1 else (reqs[:1], reqs):
            c0 = ctx.map_copies
            want, wpk = tabs[planes].likelihood_maps(group, scores="host")
            c1 = ctx.map_copies
            got, gpk = tabs[planes].likelihood_maps(group, scores="pinned")
            c2 = ctx.map_copies
            assert c1 - c0 >= len(group)  # pageable maps are copied
            # page-locked maps: the sweeps write them, no copy (the exponential
            # sweep's exact-peak re-score keeps its device map and a copy)
            assert c2 - c1 == (len(group) if planes == swg.PLANES_DECAY else 0)
            assert gpk == wpk
            for g_, w_ in zip(got, want):
                assert (g_ == w_).all()


def test_fanout_reorders_costliest_first_outputs_stay_put(ctx, oracle):
    """Device-output requests given in ASCENDING cost order (the fan-out
    issues the costliest first): every map and peak still lands at its own
    index and equals the single-request result; host, device and no-map
    outputs mixed."""
    import torch
    img = oracle.random_gray(180, 150, 41)
    bins = 16
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    ks = [(K(swg.UNIFORM, 5, 5), swg.PLAIN, 1), (K(swg.GAUSS_CHEB, 11, 11, 0.5), swg.CAKE, 6),
          (K(swg.GAUSS_CHEB, 21, 21, 0.5), swg.CAKE, 11),
          (K(swg.GAUSS_CHEB, 31, 31, 0.5), swg.CAKE, 16),
          (K(swg.GAUSS_CHEB, 41, 41, 0.5), swg.BRUTE, 1)]
    reqs = []
    for k, method, rings in ks:
        ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
        mdl = oracle.target_model(fi[10:10 + k.kh, 20:20 + k.kw].copy(), bins, ok,
                                  O.SWIH if method == swg.PLAIN else method, rings)
        reqs.append(swg.MapRequest(k, mdl, method, swg.BHATTACHARYYA, rings))
    single = [t.likelihood_map(r.kernel, r.model, r.method, rings=r.rings) for r in reqs]
    dev = [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda") for r in reqs]
    peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
    t.likelihood_maps(reqs, scores="none", scores_dev=dev, peaks_dev=peaks)
    ctx.synchronize()
    pk = peaks.cpu().numpy()
    for i, (m, p) in enumerate(single):
        assert (dev[i].cpu().numpy() == m).all(), i
        ints = pk[i, :2].view(np.int32)
        assert (int(ints[0]), int(ints[1]), float(pk[i, 2])) == (p[0], p[1], p[4]), i
    maps, pks = t.likelihood_maps(reqs, scores="none")  # peaks only
    assert [tuple(p) for p in pks] == [tuple(p) for _, p in single]


def test_quadratic_tall_image(ctx, oracle):
    """32-bit quadratic planes have no height limit (the 64-bit export keeps
    the 2340-row limit of its y^2 carries): maps of a 40 x 3000 image."""
    img = oracle.random_gray(40, 3000, 12)
    bins = 5
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC)
    k = K(swg.EUCLID_QUAD, 15, 21)
    ok = O.kernel(O.EUCLID_QUAD, 15, 21)
    mdl = oracle.target_model(fi[100:121, 10:25].copy(), bins, ok, O.BRUTE)
    got, pk = t.likelihood_map(k, mdl, swg.SWIH, rows=(2900, 2980))
    want = oracle.likelihood_map(np.ascontiguousarray(fi[2900:3000]), bins, mdl, ok, O.BRUTE)
    assert (got == want).all()
    with pytest.raises(swg.SizeError):
        t.export_i64(0)


def test_bin_range_chain_rebuild_bins(ctx, oracle):
    """One table set walks the bin ranges (swg_tables_rebuild_bins from the
    resident feature image): the chain's last map == the full table's map."""
    import torch
    img = oracle.random_gray(90, 64, 21)
    bins, d = 24, 0.9375
    fi = oracle.quantize_gray8(img, bins)
    for planes, k, method, rings in ((swg.PLANES_DECAY, K(swg.EXP_L1, 11, 11, d), swg.SWIH, 1),
                                     (swg.PLANES_AFFINE, K(swg.MANHATTAN, 9, 13), swg.SWIH, 1),
                                     (swg.PLANES_PLAIN, K(swg.GAUSS_CHEB, 13, 13, 0.5), swg.CAKE, 7)):
        ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
        om = O.CAKE if method == swg.CAKE else (O.BRUTE if k.kind == swg.EXP_L1 else O.SWIH)
        model = oracle.target_model(fi[10:10 + k.kh, 20:20 + k.kw].copy(), bins, ok, om, rings)
        full = (ctx.build_decay(img, d, swg.FMT_GRAY8, bins) if planes == swg.PLANES_DECAY
                else ctx.build(img, swg.FMT_GRAY8, bins, planes))
        want, wpk = full.likelihood_map(k, model, method, rings=rings)
        t = ctx.build_bins(oracle.random_gray(90, 64, 5), 0, 8, swg.FMT_GRAY8, bins, planes,
                           decay=d)  # another frame first: the walk uploads the real one
        shape = t.map_shape(k) + (2,)
        bufs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(2)]
        for rep in range(2):  # two walks: each starts from a fresh upload at range 0
            for c, b0 in enumerate((0, 8, 16)):
                t.rebuild_bins(b0, img if c == 0 else None)
                assert (t.bin_begin, t.bin_end) == (b0, b0 + 8)
                last = c == 2
                r = swg.MapRequest(k, model, method, rings=rings,
                                   partial_in=bufs[(c - 1) % 2] if c else None,
                                   partial_out=None if last else bufs[c % 2])
                maps, pks = t.likelihood_maps([r], scores="host" if last else "none")
            assert (maps[0] == want).all() and pks[0] == wpk, (planes, rep)
    with pytest.raises(swg.OutOfRangeError):
        t.rebuild_bins(20)


def test_cake16_wide_ring0_both_sims(ctx, oracle):
    """257x257 full-ring cake on 16-bit planes: ring 0's box holds >= 2^16
    pixels and is recovered exactly from ring 1 (wide ring 0)."""
    img = oracle.random_gray(300, 270, 31)
    bins = 6
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    k = K(swg.GAUSS_CHEB, 257, 257, 0.5)
    ok = O.kernel(O.GAUSS_CHEB, 257, 257, 0.5)
    model = oracle.target_model(fi[5:262, 20:277].copy(), bins, ok, O.CAKE, 129)
    for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
        want = oracle.likelihood_map(fi, bins, model, ok, O.CAKE, sim, rings=129)
        got, pk = t.likelihood_map(k, model, swg.CAKE, sim, rings=129)
        assert (got == want).all(), sim
        assert pk == oracle.peak(want, 128, 128)


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_random_configurations_all_engines(ctx, oracle, seed):
    """Randomised shapes, bin counts, kernel sizes, row ranges and both
    similarities through every table sweep, against the oracle (bit-exact;
    the exponential map within 1e-4 with an exact peak)."""
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(40, 130)), int(rng.integers(40, 130))
    bins = int(rng.choice([3, 8, 13, 24]))
    img = oracle.random_gray(w, h, seed)
    fi = oracle.quantize_gray8(img, bins)
    d = float(rng.choice([0.75, 0.875, 0.9375]))
    tabs = {swg.PLANES_AFFINE: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_AFFINE),
            swg.PLANES_PLAIN: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN),
            swg.PLANES_QUADRATIC: ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC),
            swg.PLANES_DECAY: ctx.build_decay(img, d, swg.FMT_GRAY8, bins)}
    for trial in range(6):
        kw = 2 * int(rng.integers(0, min(w, h) // 2 - 1)) + 1
        kh = 2 * int(rng.integers(0, min(w, h) // 2 - 1)) + 1
        sq = min(kw, kh)
        cases = [(K(swg.MANHATTAN, kw, kh), swg.SWIH, 1, swg.PLANES_AFFINE, O.SWIH, True),
                 (K(swg.UNIFORM, kw, kh), swg.SWIH, 1, swg.PLANES_PLAIN, O.SWIH, True),
                 (K(swg.GAUSS_CHEB, sq, sq, 0.5), swg.CAKE, sq // 2 + 1, swg.PLANES_PLAIN,
                  O.CAKE, True),
                 (K(swg.GAUSS_CHEB, kw, kh, 0.5), swg.CAKE, min(kw, kh) // 2 + 1,
                  swg.PLANES_AFFINE, O.CAKE, True),
                 (K(swg.EUCLID_QUAD, kw, kh), swg.SWIH, 1, swg.PLANES_QUADRATIC, O.BRUTE, True),
                 (K(swg.EXP_L1, kw, kh, d), swg.SWIH, 1, swg.PLANES_DECAY, O.BRUTE, False),
                 (K(swg.GAUSS_CHEB, kw, kh, 0.5), swg.BRUTE, 1, swg.PLANES_PLAIN, O.BRUTE, True)]
        mh = h - kh + 1
        r0 = int(rng.integers(0, mh))
        rows = (r0, int(rng.integers(r0 + 1, mh + 1)))
        for k, method, rings, planes, om, exact in cases:
            ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
            y0, x0 = int(rng.integers(0, h - k.kh + 1)), int(rng.integers(0, w - k.kw + 1))
            model = oracle.target_model(fi[y0:y0 + k.kh, x0:x0 + k.kw].copy(), bins, ok, om,
                                        rings)
            sim = int(rng.integers(0, 2))
            want = oracle.likelihood_map(fi, bins, model, ok, om, sim, rings=rings, rows=rows)
            got, pk = tabs[planes].likelihood_map(k, model, method, sim, rings, rows=rows)
            if exact:
                assert (got == want).all(), (seed, trial, k.kind, kw, kh, method, sim, rows)
            else:
                np.testing.assert_allclose(got, want, rtol=0, atol=1e-4)
            u, v = pk[0], pk[1] - rows[0]
            assert pk[4] == want.max() and want[v, u] == want.max()
            assert (v, u) == tuple(np.unravel_index(np.argmax(want), want.shape))


def _peer_chain_worker(rank, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        orc = O.Oracle()
        ctx = swg.Context(0)
        img = orc.random_gray(80, 60, 44)
        bins, d = 16, 0.9375
        fi = orc.quantize_gray8(img, bins)
        k = K(swg.EXP_L1, 13, 11, d)
        ok = O.kernel(O.EXP_L1, 13, 11, d)
        model = orc.target_model(fi[20:31, 30:43].copy(), bins, ok, O.BRUTE)
        b0, b1 = (0, 8) if rank == 0 else (8, 16)
        t = ctx.build_bins(img, b0, b1, swg.FMT_GRAY8, bins, swg.PLANES_DECAY, decay=d)
        nbytes = t.map_shape(k)[0] * t.map_shape(k)[1] * 16
        mine = swg.device_alloc(nbytes) if rank == 1 else None
        handles = [None, None]
        dist.all_gather_object(handles, swg.ipc_export(mine) if mine else None)
        token = torch.zeros(1)
        if rank == 0:  # the sweep writes its running sums into rank 1's buffer
            peer = swg.ipc_import(handles[1])
            t.likelihood_maps([swg.MapRequest(k, model, partial_out=peer)], scores="none")
            ctx.synchronize()
            dist.send(token, dst=1)
            q.put((0, True))
        else:
            dist.recv(token, src=0)
            maps, pks = t.likelihood_maps([swg.MapRequest(k, model, partial_in=mine)])
            full = ctx.build_decay(img, d, swg.FMT_GRAY8, bins)
            want, wpk = full.likelihood_map(k, model, swg.SWIH)
            q.put((1, bool((maps[0] == want).all()) and pks[0] == wpk))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_bin_chain_through_peer_memory():
    """Two processes (one per GPU on a multi-GPU box; both on cuda:0 here):
    rank 0's sweep writes its running sums straight into rank 1's buffer
    through an IPC-mapped pointer (swg_ipc_export / swg_ipc_import), rank 1
    finishes the chain; the map equals the single-table map bit for bit."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_peer_chain_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert res[0] and res[1]


# ---------------------------------------------------------------- device boundary rows
@pytest.mark.parametrize("planes", [swg.PLANES_AFFINE, swg.PLANES_QUADRATIC])
def test_device_boundary_row_exchange(ctx, oracle, planes):
    """Row bands built separately; their last record rows exchanged on the
    device (the all-gather simulated by a list) and carried
    (swg_tables_add_carry): every band's 32-bit planes equal the full frame's
    rows, and sweeps on the carried (global-row) tables give the full frame's
    map rows bit for bit."""
    import torch
    from paper_1705_03524_b200 import dist as D
    img = oracle.random_gray(301, 170, 77)
    bins = 12
    full = ctx.build(img, swg.FMT_GRAY8, bins, planes)
    want = [full.export_u32(k) for k in range(3)]
    if planes == swg.PLANES_QUADRATIC:
        want += [(full.export_i64(k) & 0xFFFFFFFF).astype(np.uint32) for k in (3, 4)]
    bands = D.table_bands(170, 3)
    tabs = [ctx.build(np.ascontiguousarray(img[y0:y1]), swg.FMT_GRAY8, bins, planes)
            for y0, y1 in bands]
    lasts = [t.last_row() for t in tabs]
    y0s = [y0 for y0, _ in bands]
    for r, (t, (y0, y1)) in enumerate(zip(tabs, bands)):
        t.add_carry(y0, D.device_carry(lasts, y0s, r).cuda().contiguous())
        for k in range(3):
            assert (t.export_u32(k)[:, :, :] == want[k][:, y0:y1 + 1]).all(), (r, k)
        with pytest.raises(swg.ConfigError):
            t.export_i64(0)
    # maps on the carried tables: map rows of windows inside each band
    kk = K(swg.EUCLID_QUAD if planes == swg.PLANES_QUADRATIC else swg.MANHATTAN, 9, 7)
    fi = oracle.quantize_gray8(img, bins)
    ok = O.kernel(kk.kind, 9, 7)
    mdl = oracle.target_model(fi[40:47, 50:59].copy(), bins, ok,
                              O.BRUTE if planes == swg.PLANES_QUADRATIC else O.SWIH)
    fmap, _ = full.likelihood_map(kk, mdl)
    for t, (y0, y1) in zip(tabs, bands):
        got, _ = t.likelihood_map(kk, mdl)
        assert (got == fmap[y0:y1 - 6]).all()


@pytest.mark.parametrize("kw,kh", [(3, 3), (9, 7), (17, 17), (37, 37), (49, 45), (1, 11)])
def test_affine16_manhattan_exact(ctx, oracle, kw, kh):
    """Manhattan windows of mass < 2^16 on maps of >= 2^20 windows sweep the
    narrow 16-bit {1, x, y} planes (k_sweep_affine16): maps and peaks
    identical to the oracle and to the 32-bit sweep (SWG_AFFINE16=0), on
    affine and quadratic table sets, both similarities, full maps and row
    ranges, and after a rebuild."""
    import os
    w, h = 1200, 1000
    img = oracle.random_gray(w, h, 5 + kw)
    img = ((img.astype(np.uint16) + np.roll(img, 1, 1) + np.roll(img, 1, 0)) // 3).astype(np.uint8)
    bins = 16
    fi = oracle.quantize_gray8(img, bins)
    k = K(swg.MANHATTAN, kw, kh)
    ok = O.kernel(O.MANHATTAN, kw, kh)
    mdl = oracle.target_model(fi[30:30 + kh, 40:40 + kw].copy(), bins, ok)
    assert (w - kw + 1) * (h - kh + 1) >= 1 << 20
    for planes in (swg.PLANES_AFFINE, swg.PLANES_QUADRATIC):
        t = ctx.build(img, swg.FMT_GRAY8, bins, planes)
        for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
            want, wpk, _ = oracle.fast_map(fi, bins, mdl, ok, O.SWIH, sim)
            got, pk = t.likelihood_map(k, mdl, swg.SWIH, sim)
            assert (got == want).all()
            assert pk == wpk
            os.environ["SWG_AFFINE16"] = "0"
            try:
                g32, p32 = t.likelihood_map(k, mdl, swg.SWIH, sim)
            finally:
                del os.environ["SWG_AFFINE16"]
            assert (g32 == got).all() and p32 == pk
        wantb, _, _ = oracle.fast_map(fi, bins, mdl, ok, O.SWIH, O.BHATTACHARYYA)
        rows = (5, 900)
        part, _ = t.likelihood_maps([swg.MapRequest(k, mdl, rows=rows)])
        assert (part[0] == wantb[rows[0]:rows[1]]).all()
        t.rebuild(np.ascontiguousarray(img[::-1]))  # rebuild refreshes the narrow planes
        want2, _, _ = oracle.fast_map(np.ascontiguousarray(fi[::-1]), bins, mdl, ok)
        got2, _ = t.likelihood_map(k, mdl)
        assert (got2 == want2).all()
        t.close()
