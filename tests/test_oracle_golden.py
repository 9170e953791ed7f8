"""CPU: pin the C restatement (oracle/swih_oracle.c) against the reference's
golden vectors (tests/golden, produced by the reference library itself) and,
where the reference library is available, against seeded reference runs."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

K = O.kernel


def test_cross3_known_answers(oracle):
    g = golden("cross3")
    fi = oracle.quantize_gray8(g["image"], 2)
    assert (fi == g["fi"]).all()
    p, x, y = oracle.build_tables(fi, 2)
    assert (p == g["plain"]).all() and (x == g["xramp"]).all() and (y == g["yramp"]).all()
    # test_integral_tables.cpp:53-69: plain(2,2,1)=2, xramp=1, yramp=1
    assert p[1, 2, 2] == 2 and x[1, 2, 2] == 1 and y[1, 2, 2] == 1
    t = (p, x, y)
    man3 = K(O.MANHATTAN, 3, 3)
    assert oracle.swih_query(t, 1, 1, man3).tolist() == g["swih_man3"].tolist() == [7, 8]
    assert oracle.plain_query(t, 1, 1, K(O.UNIFORM, 3, 3)).tolist() == [5, 4]
    assert oracle.brute_counts(fi, 2, 1, 1, man3).tolist() == [7, 8]
    assert (oracle.target_model(fi, 2, man3) == g["model_man3"]).all()
    assert (oracle.target_model(fi, 2, K(O.UNIFORM, 3, 3)) == g["model_uni3"]).all()
    assert (oracle.cake_histogram(t, K(O.CHEBYSHEV, 3, 3), 2, O.RING_MEAN, 1, 1)
            == g["cake_cheb3_r2"]).all()
    assert (oracle.cake_histogram(t, man3, 2, O.RING_MEAN, 1, 1) == g["cake_man3_r2"]).all()
    assert (oracle.cake_histogram(t, man3, 2, O.RING_LEVEL, 1, 1) == g["cake_man3_level"]).all()
    assert oracle.similarity(0, [7 / 15, 8 / 15], [.5, .5]) == g["bhatt_example"][0]


def test_tables_random(oracle):
    g = golden("tables_32x32_s99_b8")
    p, x, y = oracle.build_tables(oracle.quantize_gray8(g["image"], 8), 8)
    assert (p == g["plain"]).all() and (x == g["xramp"]).all() and (y == g["yramp"]).all()


def test_four_corner_rule_vs_direct_loop(oracle):
    # test_integral_tables.cpp:95-110 (seed 99 image, 200 rectangles)
    img = oracle.random_gray(32, 32, 99)
    fi = oracle.quantize_gray8(img, 8)
    p, x, y = oracle.build_tables(fi, 8)
    rng = np.random.default_rng(100)
    yy, xx = np.mgrid[0:32, 0:32]
    for _ in range(200):
        x0 = int(rng.integers(32)); x1 = x0 + int(rng.integers(32 - x0))
        y0 = int(rng.integers(32)); y1 = y0 + int(rng.integers(32 - y0))
        b = int(rng.integers(8))
        m = (fi == b)[y0:y1 + 1, x0:x1 + 1]
        for tab, wgt in ((p, 1), (x, xx), (y, yy)):
            direct = int((m * (wgt if np.isscalar(wgt) else wgt[y0:y1 + 1, x0:x1 + 1])).sum())
            four = tab[b, y1 + 1, x1 + 1] - tab[b, y0, x1 + 1] - tab[b, y1 + 1, x0] + tab[b, y0, x0]
            assert four == direct


def test_clipped_queries(oracle):
    g = golden("clipped_15x11_s8_b4")
    fi = oracle.quantize_gray8(g["image"], 4)
    t = oracle.build_tables(fi, 4)
    k = K(O.MANHATTAN, 7, 5)
    for cy in range(11):
        for cx in range(15):
            assert (oracle.swih_query(t, cx, cy, k, O.CLIPPED) == g["counts"][cy, cx]).all()
            assert (oracle.brute_counts(fi, 4, cx, cy, k, O.CLIPPED) == g["counts"][cy, cx]).all()


@pytest.mark.parametrize("key,method,sim", [("map_bhatt", O.SWIH, O.BHATTACHARYYA),
                                            ("map_inter", O.SWIH, O.INTERSECTION),
                                            ("map_brute", O.BRUTE, O.BHATTACHARYYA)])
def test_maps_bit_exact(oracle, key, method, sim):
    g = golden("map_40x33_s2024_b8_man9x7")
    fi = oracle.quantize_gray8(g["image"], 8)
    k = K(O.MANHATTAN, 9, 7)
    templ = fi[9:16, 12:21].copy()
    model = oracle.target_model(templ, 8, k)
    assert (model == g["model"]).all()
    m = oracle.likelihood_map(fi, 8, model, k, method, sim)
    assert (m == g[key]).all()
    if key != "map_brute":
        assert oracle.peak(m, 4, 3) == tuple(g["peak_" + key[4:]].tolist())


def test_tiled_template_all_methods(oracle):
    g = golden("tiled_9x6")
    fi = oracle.quantize_gray8(g["image"], 2)
    man3 = K(O.MANHATTAN, 3, 3)
    tile = fi[:3, :3].copy()
    for name, meth in (("swih", O.SWIH), ("brute", O.BRUTE), ("cake", O.CAKE), ("plain", O.PLAIN)):
        mdl = oracle.target_model(tile, 2, man3, meth, rings=2)
        assert (mdl == g["model_" + name]).all()
        m = oracle.likelihood_map(fi, 2, mdl, man3, meth, rings=2)
        assert (m == g["map_" + name]).all(), name
        assert abs(m[0, 0] - 1.0) < 1e-12


def test_gaussian_cake_and_brute(oracle):
    g = golden("gauss_48x40_s60_b8_k9")
    fi = oracle.quantize_gray8(g["image"], 8)
    kg = K(O.GAUSS_CHEB, 9, 9, 0.6)
    tfi = fi[10:19, 20:29].copy()
    assert (oracle.target_model(tfi, 8, kg, O.CAKE, rings=5) == g["model_cake"]).all()
    assert (oracle.target_model(tfi, 8, kg, O.BRUTE) == g["model_brute"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model_cake"], kg, O.CAKE, rings=5) == g["map_cake"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model_cake"], kg, O.CAKE, O.INTERSECTION, rings=5)
            == g["map_cake_inter"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model_brute"], kg, O.BRUTE) == g["map_brute"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model_brute"], kg, O.BRUTE, O.INTERSECTION)
            == g["map_brute_inter"]).all()
    # full-ring cake is exact up to rounding vs brute (test_baselines.cpp:104-128)
    assert np.abs(g["map_cake"] - g["map_brute"]).max() < 1e-9


def test_chebyshev(oracle):
    g = golden("cheb_40x36_s5_b8_k7x5")
    fi = oracle.quantize_gray8(g["image"], 8)
    kc = K(O.CHEBYSHEV, 7, 5)
    assert (oracle.target_model(fi[3:8, 4:11].copy(), 8, kc, O.BRUTE) == g["model"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model"], kc, O.BRUTE) == g["map_brute"]).all()
    assert (oracle.likelihood_map(fi, 8, g["model"], kc, O.CAKE, rings=2, rule=O.RING_LEVEL)
            == g["map_cake_level"]).all()


@pytest.mark.parametrize("name,k", [("scene_96x80_man21_b16", 21), ("config1_s3", 33)])
def test_scene_maps_and_peaks(oracle, name, k):
    g = golden(name)
    fi = oracle.quantize_gray8(g["image"], 16)
    kk = K(O.MANHATTAN, k, k)
    m = oracle.likelihood_map(fi, 16, g["model"], kk, threads=8)
    assert (m == g["map"]).all()
    assert oracle.peak(m, kk.kw // 2, kk.kh // 2) == tuple(g["peak"].tolist())
    assert (g["peak"][2], g["peak"][3]) == (g["target"][0], g["target"][1])


def test_peak_tie_rule(oracle):
    g = golden("peak_ties")
    assert oracle.peak(g["scores"], 1, 2) == tuple(g["peak"].tolist()) == (1, 0, 2, 2, 0.9)
    assert oracle.peak(np.full((2, 2), .5), 0, 0)[:2] == (0, 0)


def test_row_band_crop_identity(oracle):
    """Counts do not depend on the crop: a pixel-row band reproduces map rows
    byte for byte (the basis of row-band sharding)."""
    img = oracle.random_gray(64, 70, 12)
    fi = oracle.quantize_gray8(img, 8)
    k = K(O.MANHATTAN, 11, 9)
    model = oracle.target_model(fi[:9, :11].copy(), 8, k)
    full = oracle.likelihood_map(fi, 8, model, k)
    v0, v1 = 17, 40
    band = fi[v0:v1 + k.kh - 1].copy()
    assert (oracle.likelihood_map(band, 8, model, k) == full[v0:v1]).all()
    assert (oracle.likelihood_map(fi, 8, model, k, rows=(v0, v1)) == full[v0:v1]).all()


# ---- against the reference library itself (seeded; this container and any
# box that received oracle/_ref) -------------------------------------------

def test_mt19937_64_matches_std(oracle, ref):
    for seed in (0, 1, 2024, 2**63 + 5):
        assert (oracle.random_gray(17, 9, seed) == ref.random_gray(17, 9, seed)).all()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restatement_vs_reference_random(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(20, 60)), int(rng.integers(20, 60))
    img = ref.random_gray(w, h, seed)
    for bins in (2, 8, 16):
        fi = ref.quantize(img, bins)
        assert (fi == oracle.quantize_gray8(img, bins)).all()
        rt = ref.tables(fi, bins)
        p, x, y = oracle.build_tables(fi, bins)
        assert (rt.export(0) == p).all() and (rt.export(1) == x).all() and (rt.export(2) == y).all()
        for kind, kw, kh, sig in ((O.MANHATTAN, 7, 5, .5), (O.UNIFORM, 9, 9, .5),
                                  (O.GAUSS_CHEB, 7, 7, .5), (O.CHEBYSHEV, 5, 9, .5)):
            k = K(kind, kw, kh, sig)
            templ = img[:kh, :kw].copy()
            for method in (O.SWIH, O.BRUTE, O.CAKE, O.PLAIN):
                if method == O.SWIH and kind not in (O.MANHATTAN, O.UNIFORM):
                    continue
                rings = min(kw, kh) // 2 + 1 if method == O.CAKE else 1
                mdl = ref.target_model(templ, bins, k, method, rings)
                assert (mdl == oracle.target_model(ref.quantize(templ, bins), bins, k, method,
                                                   rings)).all()
                for sim in (0, 1):
                    a, pa = ref.likelihood_map(img, bins, mdl, k, method, sim, rings=rings)
                    b = oracle.likelihood_map(fi, bins, mdl, k, method, sim, rings=rings)
                    assert (a == b).all(), (kind, method, sim)
                    assert oracle.peak(b, k.kw // 2, k.kh // 2) == pa


def test_error_codes_match_reference(oracle, ref):
    img = ref.random_gray(9, 9, 4)
    fi = ref.quantize(img, 2)
    t = oracle.build_tables(fi, 2)
    rt = ref.tables(fi, 2)
    cases = [
        (lambda: oracle.swih_query(t, 1, 4, K(O.MANHATTAN, 5, 5)),
         lambda: rt.swih_query(1, 4, K(O.MANHATTAN, 5, 5))),
        (lambda: oracle.swih_query(t, 4, 9, K(O.MANHATTAN, 3, 3), O.CLIPPED),
         lambda: rt.swih_query(4, 9, K(O.MANHATTAN, 3, 3), O.CLIPPED)),
        (lambda: oracle.swih_query(t, 4, 4, K(O.MANHATTAN, 4, 3)),
         lambda: rt.swih_query(4, 4, K(O.MANHATTAN, 4, 3))),
        (lambda: oracle.swih_query(t, 4, 4, K(O.GAUSS_CHEB, 3, 3)),
         lambda: rt.swih_query(4, 4, K(O.GAUSS_CHEB, 3, 3))),
        (lambda: oracle.cake_plan(K(O.CHEBYSHEV, 3, 3), 3),
         lambda: ref.cake_plan(K(O.CHEBYSHEV, 3, 3), 3)),
    ]
    for a, b in cases:
        with pytest.raises(O.OracleError) as ea:
            a()
        with pytest.raises(O.OracleError) as eb:
            b()
        assert ea.value.code == eb.value.code
